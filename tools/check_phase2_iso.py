"""Isolate Phase-1 vs Phase-2 error on c1: run the iteration in numpy with (a) the oracle's
Householder factors, (b) the GPU's memoized M; both with their own adaptive rho."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from scipy.linalg import solve_triangular
import paper_2501_11673_b200 as kpp, synth, oracle
cfg = synth.CONFIGS["c1"]
A, b, _ = synth.make_problem(cfg); An = A.numpy(); bn = b.numpy()
m, n = An.shape; s = cfg.s; lam = cfg.lam; T = 200
C = oracle.kpp_C(m, n, s)
bid, fresh, nb = oracle.schedule(0, C, T)
ref = oracle.kpp_run(An, bn, s, lam=lam, seed=0, max_iters=T)
ctx = kpp.kpp_setup(A.cuda(), s, lam, 0)
ctx.prepare(T)
def run(src):
    x = np.zeros(n); mom = np.zeros(n); eta = s / (2.0 * n)
    zeta = -(-m // s); rho = 0.0; rhat = 1.0; E0 = E1 = 0.0; i = 0
    Ms = {}
    for t in range(T):
        k = int(bid[t])
        if k not in Ms:
            S = oracle.fresh_block(0, m, s, k)
            if src == "oracle":
                X = solve_triangular(oracle.kpp_factor(An, S, lam), np.eye(s)); Ms[k] = (S, X @ X.T)
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
gpu_x = kpp.kpp_setup(A.cuda(), s, lam, 0).solve(b.cuda(), max_iters=T).x.cpu().numpy()
for src in ("oracle", "gpuM"):
    x = run(src)
    print(src, "numpy iteration err vs oracle", np.linalg.norm(x - ref.x) / np.linalg.norm(ref.x),
          " vs GPU", np.linalg.norm(x - gpu_x) / np.linalg.norm(gpu_x), flush=True)
print("GPU vs oracle", np.linalg.norm(gpu_x - ref.x) / np.linalg.norm(ref.x))
