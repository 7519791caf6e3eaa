"""c1 iterate difference vs the oracle at t=200 for every engine / plan (isolates Phase-2 error)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2501_11673_b200 as kpp, synth, oracle
name = sys.argv[1] if len(sys.argv) > 1 else "c1"
T = int(sys.argv[2]) if len(sys.argv) > 2 else 200
cfg = synth.CONFIGS[name]
A, b, _ = synth.make_problem(cfg, device="cuda")
ref = oracle.kpp_run(A.cpu().numpy(), b.cpu().numpy(), cfg.s, lam=cfg.lam, seed=0, max_iters=T, threads=16)
def go(label, **opts):
    ctx = kpp.kpp_setup(A, cfg.s, cfg.lam, 0)
    try:
        for k, v in opts.items():
            ctx.set_option(getattr(kpp, k), v)
    except kpp.KppError as e:
        print(label, "infeasible"); return
    r = ctx.solve(b, max_iters=T)
    x = r.x.cpu().numpy()
    st = ctx.stats()
    print(f"{label:28s} err {np.linalg.norm(x - ref.x) / np.linalg.norm(ref.x):.2e}  rho_hist_diff "
          f"{np.max(np.abs(ctx.rho_history().numpy() - ref.hist_rho)):.1e} plan C={st['cluster']} ygl={st['ygl']}", flush=True)
go("default")
go("graph engine", OPT_ENGINE=1)
for y in (0, 1, 4):
    for C in (1, 2, 4, 8):
        go(f"ygl{y} C{C}", OPT_YGL=y, OPT_CLUSTER=C)
go("streaming", OPT_RESIDENT=0)
go("window 7", OPT_WINDOW=7)
