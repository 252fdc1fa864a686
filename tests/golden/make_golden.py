"""Generate the committed golden fixtures from the UNMODIFIED reference.

Run here (where /root/reference exists and oracle/_ref/libdivstokes_ref.so is
built): ``python tests/golden/make_golden.py``. The GPU box never runs this;
tests read the .npz files it writes.

Fixtures (all produced by the reference's own code through oracle/ref_driver):
  c1_psi_k2_n8.npz   psi-MMS, k'=2, 8x8: A, B, Q, Q_nu, f (reference assembly),
                     RCM(A) / RCM(Q_nu), IC(0) factors, one IC(0) apply on a
                     seeded vector, the saddle apply on a seeded vector, and
                     reference solves (u, p, iterations, inner means,
                     histories) for every GPU strategy at outer 1e-8.
  c1_psi_k2_n16.npz  BASELINE config 1 (16x16, IC0-PCG(A)+Diag(Q), 1e-8/1e-1)
                     system + reference solution.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import RefLib  # noqa: E402
from oracle.oracle import STRATEGIES  # noqa: E402


def dump_csr(d, name, m):
    d[name + "_rp"], d[name + "_ci"], d[name + "_v"] = m.rp, m.ci, m.v
    d[name + "_shape"] = np.array([m.n_rows, m.n_cols])


def main():
    R = RefLib()
    rng = np.random.default_rng(2024)
    # --- small system, all strategies
    s = R.assemble("psi-mms", 2, 8)
    d = {}
    for w in ("A", "B", "Bt", "Q", "Q_nu"):
        dump_csr(d, w, s.block(w))
    d["f"] = s.rhs()
    A, Qn = s.block("A"), s.block("Q_nu")
    for tag, M in (("A", A), ("Q", Qn)):
        perm = R.rcm(M)
        L = R.ic0(R.permute(M, perm))
        d["perm_" + tag] = perm
        dump_csr(d, "L_" + tag, L)
        r = rng.standard_normal(M.n_rows)
        d["ic_r_" + tag] = r
        d["ic_z_" + tag] = R.ic0_solve(L, r)
    x = rng.standard_normal(s.n_u + s.n_p)
    d["apply_x"] = x
    d["apply_y"] = s.apply(x)
    for strat in STRATEGIES:
        for itol in (1e-1, 1e-6):
            res = s.solve(strat, 1e-8, itol)
            key = f"{strat}|{itol:g}"
            d["sol_u|" + key] = res["u"]
            d["sol_p|" + key] = res["p"]
            d["sol_meta|" + key] = np.array([res["iterations"], res["converged"],
                                             res["mean_inner_top"], res["mean_inner_bottom"]])
            d["sol_hm|" + key] = res["residual_history"]
            d["sol_he|" + key] = res["euclid_history"]
    np.savez_compressed(os.path.join(HERE, "c1_psi_k2_n8.npz"), **d)
    # --- BASELINE config 1
    s = R.assemble("psi-mms", 2, 16)
    d = {}
    for w in ("A", "B", "Bt", "Q", "Q_nu"):
        dump_csr(d, w, s.block(w))
    d["f"] = s.rhs()
    res = s.solve("IC0-PCG(A)+Diag(Q)", 1e-8, 1e-1)
    d["u"], d["p"] = res["u"], res["p"]
    d["meta"] = np.array([res["iterations"], res["converged"], res["mean_inner_top"],
                          res["mean_inner_bottom"]])
    d["hm"], d["he"] = res["residual_history"], res["euclid_history"]
    np.savez_compressed(os.path.join(HERE, "c1_psi_k2_n16.npz"), **d)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
