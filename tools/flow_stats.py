"""Print the staged-sweep plan statistics (DSGPU_FLOW_STATS) for a system and
merge factors. Usage: flow_stats.py case k N [M ...]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["DSGPU_FLOW_STATS"] = "1"
from paper_1309_5048_b200 import host, solver
case, k, n = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
s = host.assemble(case, k, n, seed=1234)
for M in (sys.argv[4:] or ["1", "2", "4"]):
    os.environ["DSGPU_MERGE"] = M
    print(f"--- M={M}", file=sys.stderr, flush=True)
    g = solver.GpuStokesSolver(s, "IC0-PCG(A,Q)")
    del g
