"""Cross-check of the sketch + LSQR projection against the paper's Fig
lsqr_steps: on the synthetic low-rank K++ systems (m x n = 4096 x 1024, bell
spectrum, effective rank 50 / 100, b ~ N(0, I), block sizes 100 / 200) "with only 8 steps of LSQR,
there is barely any difference between K++ and the alternative using exact projections".

The systems are inconsistent, so the residual estimate (Eq (residual)) converges to a floor near the
least-squares residual; we report, per variant, the estimate at fixed iteration counts and the
least-squares floor min ||Ax - b|| / ||b|| (numpy lstsq) for reference.  GPU solves through the C ABI."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2501_11673_b200 as kpp  # noqa: E402
import synth  # noqa: E402

T = int(os.environ.get("ITERS", "3000"))
lam = 1e-8
for er in (50, 100):
    A, b = synth.make_bell_general(4096, 1024, er, seed=0, device="cuda")
    x_ls = torch.linalg.lstsq(A, b.unsqueeze(1)).solution.squeeze(1)
    floor = float(torch.linalg.vector_norm(A @ x_ls - b) / torch.linalg.vector_norm(b))
    for s in (100, 200):
        rows = []
        for label, proj, tmax in [("Cholesky", 0, 0), ("LSQR-2", 1, 2), ("LSQR-4", 1, 4), ("LSQR-8", 1, 8),
                                  ("Chol,noacc", 0, -1), ("LSQR-8,noacc", 1, -8)]:
            ctx = kpp.kpp_setup(A, s, lam, 0)
            if tmax < 0:  # momentum off (eta = 0): the memoized block Kaczmarz of Table 1 (K++ w/o accel.)
                ctx.set_option(kpp.OPT_ACCEL, 0)
                tmax = -tmax
            if proj:
                ctx.set_option(kpp.OPT_PROJ, 1)
                ctx.set_option(kpp.OPT_TMAX, tmax)
            r = ctx.solve(b, max_iters=T, allow_maxiter=True)
            h = r.res_hist.numpy()
            zeta = (4096 + s - 1) // s
            pick = [max(0, min(len(h), int(t / (2 * zeta))) - 1) for t in (T // 10, T // 4, T // 2, T)]
            true = float(torch.linalg.vector_norm(A @ r.x - b) / torch.linalg.vector_norm(b))
            rows.append((label, [h[i] for i in pick], true))
            ctx.destroy()
        print(f"er={er} s={s} LS floor {floor:.6f}; residual estimate at t = {T // 10}, {T // 4}, {T // 2}, {T}"
              f" and the true residual at t = {T}:")
        for label, vals, true in rows:
            print(f"  K++({label:12s}) " + "  ".join(f"{v:.6f}" for v in vals) + f"   true {true:.6f}")
        sys.stdout.flush()
