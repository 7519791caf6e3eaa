"""Helper run in a subprocess by test_gpu_parity.test_gram_i8_opt_in: the int8 tensor-core Gram
(KPP_GRAM_I8=1, read once per process) against the oracle -- M for ragged and full blocks, and a
200-iteration solve of a c2 twin at the parity bar (north_star: 1e-10)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402

import oracle  # noqa: E402
import paper_2501_11673_b200 as kpp  # noqa: E402

assert os.environ.get("KPP_GRAM_I8") == "1"
rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))
oracle.build()
kpp.load_library()
DEV = "cuda:0"
for s in (96, 100, 128):
    m, n, lam = 300, 4100, 1e-8
    A, b, _ = synth.make_problem(synth.twin("c3", m, n, s, k=8))
    ctx = kpp.kpp_setup(A.to(DEV), s, lam, 5)
    ctx.prepare(6)
    An = A.numpy()
    for k in (0, 2):
        S = ctx.block(k).numpy()
        M = ctx.factor(k).numpy()
        Ri = np.linalg.inv(oracle.kpp_factor(An, S, lam))
        G = An[S] @ An[S].T + lam * np.eye(s)
        err, bound = rel(M, Ri @ Ri.T), 200 * 2.2e-16 * np.linalg.cond(G)
        assert err < bound, (s, k, err, bound)
cfg = synth.twin("c2", 1024, 1024, 128)
A, b, _ = synth.make_problem(cfg)
ref = oracle.kpp_run(A.numpy(), b.numpy(), 128, lam=cfg.lam, seed=0, max_iters=200, tol=0.0, threads=8)
ctx = kpp.kpp_setup(A.to(DEV), 128, cfg.lam, 0)
res = ctx.solve(b.to(DEV), None, max_iters=200, tol=0.0)
e = rel(res.x.cpu().numpy(), ref.x)
assert e <= 1e-10, e
assert ctx.stats()["kernel_launches"] > 0
print("gram_i8 ok", os.environ.get("KPP_GRAM_I8_PROD"), e)
