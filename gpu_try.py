import time, numpy as np, sys
sys.path.insert(0, "/root/repo")
from oracle import PortLib, CSR
from paper_1309_5048_b200 import host, solver
P = PortLib()
def c(m): return CSR(m.n_rows, m.n_cols, m.row_ptr, m.cols, m.vals)
for (k,N,strat,itol) in [(2,8,"Diag(A,Q)",1e-1),(2,16,"IC0-PCG(A)+Diag(Q)",1e-1),(2,16,"IC0-PCG(A,Q)",1e-1),(2,16,"PCG(A,Q)",1e-3),(2,64,"IC0-PCG(A,Q)",1e-1),(2,64,"IC0-PCG(A,Q)",1e-8)]:
    s = host.assemble("psi-mms", k, N)
    o = P.solve_stokes(c(s.A), c(s.B), c(s.Bt), c(s.Q_nu), s.f, strat, 1e-8, itol, Q_filter=c(s.Q))
    g = solver.GpuStokesSolver(s, strat)
    opt = solver.SolverOptions(outer_tol=1e-8, inner_tol=itol)
    sol = g.solve(options=opt)
    t = time.time(); sol = g.solve(options=opt); tw = time.time()-t
    x_o = np.concatenate([o["u"], o["p"]]); x_g = np.concatenate([sol.u, sol.p])
    rel = np.linalg.norm(x_o-x_g)/np.linalg.norm(x_o)
    print(f"k={k} N={N} {strat} itol={itol}: oracle it={o['iterations']} inner={o['mean_inner_top']:.3f}/{o['mean_inner_bottom']:.3f} t={o['wall_seconds']*1e3:.1f}ms | gpu it={sol.report.iterations} conv={sol.report.converged} inner={sol.report.mean_inner_top:.3f}/{sol.report.mean_inner_bottom:.3f} t_kernel={sol.report.wall_seconds*1e3:.2f}ms t_wall={tw*1e3:.2f}ms relL2={rel:.2e} relres_e={sol.report.relres_e:.2e}", flush=True)
    if N == 64 and itol == 1e-1:
        L = g.top.factor
        r = np.random.default_rng(0).standard_normal(s.n_u)
        z_o = P.ic0_solve(c(L), r); z_g = g.apply_ic0(0, r)
        print("  IC apply bitexact:", np.array_equal(z_o, z_g), np.abs(z_o-z_g).max())
        x = np.random.default_rng(1).standard_normal(s.n_u + s.n_p)
        y_g = g.apply(x)
        y_o = np.concatenate([P.spmv(c(s.A), x[:s.n_u]) + P.spmv(c(s.Bt), x[s.n_u:]), P.spmv(c(s.B), x[:s.n_u])])
        print("  saddle rel err", np.abs(y_g-y_o).max()/np.abs(y_o).max())
        for w,nm in [(0,"saddle"),(1,"ic0 A"),(2,"ic0 Q"),(3,"spmv A")]:
            print(f"  kernel {nm}: {g.time_kernel(w, 50)*1e3:.2f} us")
        print("  info", g.info())
