import os, sys, json
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tools"))
from config_probe import CFG
from paper_1309_5048_b200 import host, solver
for tag in sys.argv[1:]:
    c = CFG[tag]
    s = host.assemble(c["case"], c["k"], c["n"], dim=c["dim"], seed=c["seed"])
    top = solver.prepare_block(s.A, solver.BLOCK_PCG_IC0, ic0_on_gpu=True)
    bot = solver.prepare_block(s.Q_nu, solver.BLOCK_PCG_IC0, ic0_on_gpu=True)
    for L in ("8", "16", "32"):
        os.environ["DSGPU_SPMV_LANES"] = L
        g = solver.GpuStokesSolver(s, "IC0-PCG(A,Q)", top=top, bottom=bot)
        i = g.info(); n = i["n_u"] + i["n_p"]
        t0 = g.time_kernel(0, 50); t3 = g.time_kernel(3, 50)
        print(json.dumps(dict(cfg=tag, lanes=L, lib=os.environ.get("DSGPU_LIB_DIR", "lib")[-8:], saddle_us=round(t0 * 1e3, 1),
                              saddle_GBs=round((12 * i["nnz_K"] + 20 * n) / t0 / 1e6), A_us=round(t3 * 1e3, 1),
                              A_GBs=round((12 * i["nnz_A"] + 20 * i["n_u"]) / t3 / 1e6))), flush=True)
        g.close()
