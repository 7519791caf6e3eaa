"""c1 parity margin diagnosis: on bench.py's device-generated c1 instance and on the
CPU-generated one the tests use, compare after 200 iterations
  - the GPU (default factor route) and the GPU with CholeskyQR2 for every block,
  - the oracle with every reduction reversed (the oracle's own summation-order noise floor),
  - a numpy re-run of the iteration with the oracle's M = R^-1 R^-T, and with the GPU's memoized M
against the oracle: separates the Phase-1 operator from Phase-2 summation order."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from scipy.linalg import solve_triangular  # noqa: E402

import oracle  # noqa: E402
import paper_2501_11673_b200 as kpp  # noqa: E402
import synth  # noqa: E402

cfg = synth.CONFIGS["c1"]
T = int(sys.argv[1]) if len(sys.argv) > 1 else 200
rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))
for inst in ("device", "cpu"):
    A, b, _ = synth.make_problem(cfg, seed=0, device="cuda" if inst == "device" else "cpu")
    An, bn = A.cpu().numpy(), b.cpu().numpy()
    m, n = An.shape
    s, lam = cfg.s, cfg.lam
    ref = oracle.kpp_run(An, bn, s, lam=lam, seed=0, max_iters=T)
    rev = oracle.kpp_run(An, bn, s, lam=lam, seed=0, max_iters=T, reverse=True)
    gram = oracle.kpp_run(An, bn, s, lam=lam, seed=0, max_iters=T, factor=oracle.GRAM)
    out = {}
    for fac in (-1, 0):
        ctx = kpp.kpp_setup(A.cuda(), s, lam, 0)
        if fac >= 0:
            ctx.set_option(kpp.OPT_FACTOR, fac)
        out[fac] = (ctx.solve(b.cuda(), max_iters=T).x.cpu().numpy(), ctx)
    ctx = out[-1][1]
    C = oracle.kpp_C(m, n, s)
    bid, fresh, nb = oracle.schedule(0, C, T)

    def run(src):
        x = np.zeros(n); mom = np.zeros(n); eta = s / (2.0 * n)
        zeta = -(-m // s); rho = 0.0; rhat = 1.0; E0 = E1 = 0.0; i = 0
        Ms = {}
        for t in range(T):
            k = int(bid[t])
            if k not in Ms:
                S = oracle.fresh_block(0, m, s, k)
                if src == "oracle":
                    X = solve_triangular(oracle.kpp_factor(An, S, lam), np.eye(s))
                    Ms[k] = (S, X @ X.T)
                else:
                    Ms[k] = (S, ctx.factor(k).numpy())
            S, M = Ms[k]
            r = An[S] @ x - bn[S]; y = M @ r; w = An[S].T @ y
            c = (1 - rho) / (1 + rho); mom = c * (mom - w); x = x - w + eta * mom
            e = float(r @ r)
            if t % (2 * zeta) < zeta: E0 += e
            else: E1 += e
            if t % (2 * zeta) == 2 * zeta - 1:
                i += 1
                if E0 > 0: rhat, rho = oracle.rho_update(i, rhat, E0, E1, zeta)
                E0 = E1 = 0.0
        return x

    print(f"c1 {inst} instance, T={T}:")
    print(f"  GPU default route      vs oracle {rel(out[-1][0], ref.x):.2e}")
    print(f"  GPU CholeskyQR2 always vs oracle {rel(out[0][0], ref.x):.2e}")
    print(f"  oracle reversed sums   vs oracle {rel(rev.x, ref.x):.2e}")
    print(f"  oracle Gram route      vs oracle {rel(gram.x, ref.x):.2e}")
    print(f"  numpy iter, oracle M   vs oracle {rel(run('oracle'), ref.x):.2e}")
    print(f"  numpy iter, GPU M      vs oracle {rel(run('gpu'), ref.x):.2e}", flush=True)
