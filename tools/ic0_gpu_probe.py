"""Device IC(0) factorization (dsgpu_ic0_factor) vs the native host ic0 on
BASELINE systems: bit-identity and time. One JSON line per config.

  python tools/ic0_gpu_probe.py c2 c4 c5_48 ...
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
from config_probe import CFG  # noqa: E402


def main():
    from paper_1309_5048_b200 import host, solver
    for tag in sys.argv[1:]:
        c = CFG[tag]
        s = host.assemble(c["case"], c["k"], c["n"], dim=c["dim"], seed=c["seed"])
        pm = host.permute_symmetric(s.A, host.rcm_permutation(s.A))
        t0 = time.time()
        H = host.ic0(pm)
        t_host = time.time() - t0
        for flow in os.environ.get("IC0_PROBE_MODES", "1").split(","):
            os.environ["DSGPU_IC0_FLOW"] = flow
            solver.ic0_factor_gpu(pm)  # warm-up (module load, first launches)
            t0 = time.time()
            L, info = solver.ic0_factor_gpu(pm)
            t_gpu = time.time() - t0
            same = (np.array_equal(L.row_ptr, H.row_ptr) and np.array_equal(L.cols, H.cols)
                    and np.array_equal(L.vals.view(np.int64), H.vals.view(np.int64)))
            print(json.dumps(dict(cfg=tag, kernel="dataflow" if flow == "1" else "levels", n=pm.n_rows,
                                  nnz_L=int(L.row_ptr[-1]), levels=info["levels"],
                                  host_ic0_s=round(t_host, 3), gpu_call_s=round(t_gpu, 3),
                                  gpu_device_ms=round(info["device_ms"], 2), bit_identical=bool(same))),
                  flush=True)


if __name__ == "__main__":
    main()
