"""Parity of the literal Gram + Cholesky factor route (KPP_OPT_FACTOR=1) vs the CholeskyQR2 route
against the oracle on BASELINE configs, after T iterations (how much accuracy the Gram route loses
at each config's block conditioning)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2501_11673_b200 as kpp, synth, oracle

T = int(sys.argv[2]) if len(sys.argv) > 2 else 200
for name in sys.argv[1].split(","):
    cfg = synth.CONFIGS[name] if name in synth.CONFIGS else None
    A, b, _ = synth.make_problem(cfg, device="cuda")
    An, bn = A.cpu().numpy(), b.cpu().numpy()
    ref = oracle.kpp_run(An, bn, cfg.s, lam=cfg.lam, seed=0, max_iters=T, threads=os.cpu_count())
    out = {}
    for f in (0, 1, 2):
        ctx = kpp.kpp_setup(A, cfg.s, cfg.lam, 0)
        ctx.set_option(kpp.OPT_FACTOR, f)
        x = ctx.solve(b, max_iters=T).x.cpu().numpy()
        out[f] = np.linalg.norm(x - ref.x) / np.linalg.norm(ref.x)
        ctx.destroy()
    print(f"{name}: T={T} rel err vs oracle: cholqr2 {out[0]:.2e}  gram {out[1]:.2e}  adaptive {out[2]:.2e}", flush=True)
