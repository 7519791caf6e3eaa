"""Measured GPU-vs-oracle parity at BASELINE.json's full sizes (bench.py's instance and launch
configuration): ||x_gpu - x_cpu|| / ||x_cpu|| after T iterations and the largest difference of the
checkpoint residual estimates; K++ with the sketch + LSQR projection on c2/c3 too."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as ora  # noqa: E402
import paper_2501_11673_b200 as kpp  # noqa: E402
import synth  # noqa: E402

ora.build()
rows = []
for name, T, proj, tol in [("c1", 200, 0, 0.0), ("c1", 500, 0, 0.0), ("c2", 200, 0, 0.0), ("c3", 200, 0, 0.0),
                           ("c4", 3, 0, 0.0), ("c5", 200, 0, 0.0), ("c2", 200, 1, 0.0), ("c3", 200, 1, 0.0),
                           ("c3", 100000, 0, 1e-8), ("c5", 100000, 0, 1e-8)]:
    cfg = synth.CONFIGS[name]
    A, b, _ = synth.make_problem(cfg, seed=0, device="cuda")
    ctx = (kpp.cdpp_setup if cfg.kind == "cdpp" else kpp.kpp_setup)(A, cfg.s, cfg.lam, 0)
    if proj:
        ctx.set_option(kpp.OPT_PROJ, 1)
    res = ctx.solve(b, max_iters=T, tol=tol)
    xg = res.x.cpu().numpy()
    hg = res.res_hist.numpy()
    An, bn = A.cpu().numpy(), b.cpu().numpy()
    del A
    ctx.destroy()
    torch.cuda.empty_cache()
    t0 = time.time()
    run = ora.cdpp_run if cfg.kind == "cdpp" else ora.kpp_run
    kw = dict(proj=1, tmax=8) if proj else {}
    ref = run(An, bn, cfg.s, lam=cfg.lam, seed=0, max_iters=T, tol=tol, threads=os.cpu_count() or 1, **kw)
    dt = time.time() - t0
    err = float(np.linalg.norm(xg - ref.x) / np.linalg.norm(ref.x))
    dh = float(np.max(np.abs(hg - ref.hist_res))) if len(hg) and len(hg) == len(ref.hist_res) else float("nan")
    fr = float(np.linalg.norm(An @ xg - bn) / np.linalg.norm(bn)), float(np.linalg.norm(An @ ref.x - bn) / np.linalg.norm(bn))
    label = name + (" LSQR-8" if proj else "") + (f" to {tol:g}" if tol else "")
    stop = f"stop it GPU {res.iters} / oracle {ref.iters}" if tol else f"T={T}"
    hd = f"{dh:.1e}" if dh == dh else "n/a (no checkpoint)"
    print(f"{label:14s} {stop:28s} rel x err {err:.2e}  max |res_hist diff| {hd}  "
          f"rel. residual GPU {fr[0]:.3e} oracle {fr[1]:.3e} (|diff| {abs(fr[0] - fr[1]):.1e})  (oracle {dt:.1f} s)",
          flush=True)
