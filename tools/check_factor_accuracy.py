"""Accuracy of the memoized operator M = (A_S A_S^T + lam I)^{-1} per factor route against the
oracle's Householder R (M = R^{-1} R^{-T}), on a BASELINE config's first blocks."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2501_11673_b200 as kpp, synth, oracle

name = sys.argv[1] if len(sys.argv) > 1 else "c1"
cfg = synth.CONFIGS[name]
A, b, _ = synth.make_problem(cfg, device="cuda")
An = A.cpu().numpy()
ctxs = {}
for f in (0, 1, 2):
    c = kpp.kpp_setup(A, cfg.s, cfg.lam, 0)
    c.set_option(kpp.OPT_FACTOR, f)
    c.prepare(64)
    ctxs[f] = c
for k in range(6):
    S = ctxs[0].block(k).numpy()
    R = oracle.kpp_factor(An, S, cfg.lam)
    Ri = np.linalg.inv(R)
    Mref = Ri @ Ri.T
    G = An[S] @ An[S].T + cfg.lam * np.eye(cfg.s)
    kap = np.sqrt(np.linalg.cond(G))
    errs = {f: np.linalg.norm(ctxs[f].factor(k).numpy() - Mref) / np.linalg.norm(Mref) for f in ctxs}
    print(f"{name} block {k}: kappa(A_S) {kap:.2e}  u*kappa {kap * 1.1e-16:.1e}  u*kappa^2 {kap**2 * 1.1e-16:.1e}  "
          f"M rel err: cholqr2 {errs[0]:.2e}  gram {errs[1]:.2e}  adaptive {errs[2]:.2e}", flush=True)
