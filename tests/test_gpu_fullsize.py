"""Parity at BASELINE.json's FULL sizes, in the launch configuration bench.py times (default options,
cold solve, default window, the input generated on the device exactly as bench.py does).

- c1, c2, c3, c5: the first 200 iterations against the oracle run on all host cores (the BJ bar,
  ||x_gpu - x_cpu|| / ||x_cpu|| <= 1e-10), plus the checkpoint residual history;
- c4: also 200 iterations (~187 fresh blocks, each a 256 x 131072 Householder QR in the oracle: about
  two minutes on the box's host cores); the same oracle run also checks the Gram + Cholesky route
  without refinement (KPP_OPT_FACTOR=1) at the same bar;
- c3 and c5 run to the 1e-8 estimate (Alg 5 l.15 P:1352 / Alg 3 l.15 P:762): the GPU stops at the
  oracle's checkpoint and the final relative residuals ||Ax - b|| / ||b|| agree within 1e-12 absolute
  (the BJ bar, compared at the oracle's stopping iteration, reading Q15), x within 1e-10;
- every config: the block schedule and the fresh index sets of the solve bit-exact;
- every config: a property of one step that holds at any size (no oracle):
  from x_0 = 0, r_0 = -b_S, m_1 = -w_0 (rho_0 = 0) and x_1 = -(1+eta) w_0, so for K++
  A_S x_1 = (1+eta)(b_S - lam y) with y = (A_S A_S^T + lam I)^{-1} b_S, and for CD++
  (A_SS + lam I) x_1[S] = (1+eta) b_S with x_1 zero outside S.
"""
import os

import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu

DEV = "cuda:0"
rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.fixture(scope="module")
def kpp():
    import paper_2501_11673_b200 as k
    from paper_2501_11673_b200 import build
    build.build()
    k.load_library()
    assert torch.cuda.is_available()
    return k


def setup(kpp, cfg):
    A, b, _ = synth.make_problem(cfg, seed=0, device=DEV)  # bench.py's instance
    ctx = (kpp.cdpp_setup if cfg.kind == "cdpp" else kpp.kpp_setup)(A, cfg.s, cfg.lam, 0)
    return A, b, ctx


@pytest.mark.parametrize("name,T", [("c1", 200), ("c2", 200), ("c3", 200), ("c5", 200), ("c4", 200)])
def test_fullsize_parity(kpp, ora, name, T):
    cfg = synth.CONFIGS[name]
    A, b, ctx = setup(kpp, cfg)
    res = ctx.solve(b, max_iters=T)
    assert res.iters == T
    x_gpu = res.x.cpu().numpy()
    pop = cfg.n if cfg.kind == "cdpp" else cfg.m
    # schedule and fresh index sets, bit-exact (the oracle's schedule is data independent)
    C = ora.cdpp_C(cfg.n, cfg.s) if cfg.kind == "cdpp" else ora.kpp_C(cfg.m, cfg.n, cfg.s)
    bid, fresh, _ = ora.schedule(0, C, T)
    g_bid, g_fresh = ctx.schedule(0, T)
    assert np.array_equal(g_bid.numpy(), bid) and np.array_equal(g_fresh.numpy(), fresh)
    for k in sorted({0, int(bid.max()) // 2, int(bid.max())}):
        assert np.array_equal(ctx.block(k).numpy(), ora.fresh_block(0, pop, cfg.s, k))
    x_gram = None
    if name == "c4":
        # the user's switch for systems like c4 (DESIGN 13 item 2): the literal Gram + Cholesky route
        # without the CholeskyQR2 refinement, against the same oracle run
        ctx.destroy()
        ctx = kpp.kpp_setup(A, cfg.s, cfg.lam, 0)
        ctx.set_option(kpp.OPT_FACTOR, 1)
        res1 = ctx.solve(b, max_iters=T)
        assert res1.iters == T and ctx.stats()["n_refined"] == 0
        x_gram = res1.x.cpu().numpy()
    An, bn = A.cpu().numpy(), b.cpu().numpy()
    del A
    torch.cuda.empty_cache()
    run = ora.cdpp_run if cfg.kind == "cdpp" else ora.kpp_run
    ref = run(An, bn, cfg.s, lam=cfg.lam, seed=0, max_iters=T, threads=os.cpu_count() or 1)
    assert rel(x_gpu, ref.x) <= 1e-10, rel(x_gpu, ref.x)
    if len(ref.hist_res):
        assert np.allclose(res.res_hist.numpy(), ref.hist_res, rtol=1e-6, atol=1e-12)
    if x_gram is not None:
        assert rel(x_gram, ref.x) <= 1e-10, rel(x_gram, ref.x)


@pytest.mark.parametrize("name", ["c3", "c5"])
def test_fullsize_stop_to_tol(kpp, ora, name):
    """Run to the 1e-8 estimate at full size: same stopping checkpoint as the oracle, final relative
    residuals within 1e-12 absolute, x within 1e-10 (BJ bars; Q15)."""
    cfg = synth.CONFIGS[name]
    A, b, ctx = setup(kpp, cfg)
    res = ctx.solve(b, max_iters=100000, tol=1e-8)
    x_gpu = res.x.cpu().numpy()
    An, bn = A.cpu().numpy(), b.cpu().numpy()
    del A
    torch.cuda.empty_cache()
    run = ora.cdpp_run if cfg.kind == "cdpp" else ora.kpp_run
    ref = run(An, bn, cfg.s, lam=cfg.lam, seed=0, max_iters=100000, tol=1e-8, threads=os.cpu_count() or 1)
    assert ref.status == ora.OK and res.status == 0
    assert res.iters == ref.iters, (res.iters, ref.iters)
    nb = np.linalg.norm(bn)
    rg = np.linalg.norm(An @ x_gpu - bn) / nb
    rc = np.linalg.norm(An @ ref.x - bn) / nb
    assert abs(rg - rc) <= 1e-12, (rg, rc)
    assert rel(x_gpu, ref.x) <= 1e-10, rel(x_gpu, ref.x)
    assert np.allclose(res.res_hist.numpy(), ref.hist_res, rtol=1e-6, atol=1e-12)


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4", "c5"])
def test_fullsize_first_step_property(kpp, name):
    cfg = synth.CONFIGS[name]
    A, b, ctx = setup(kpp, cfg)
    x1 = ctx.solve(b, max_iters=1).x
    S = ctx.block(0).to(DEV).long()
    eta = cfg.s / (2.0 * cfg.n)  # P:1340 / P:748
    bS = b[S]
    if cfg.kind == "kpp":
        AS = A[S]
        y = torch.linalg.solve(AS @ AS.T + cfg.lam * torch.eye(cfg.s, dtype=A.dtype, device=DEV), bS)
        lhs = AS @ x1
        # A_S w = r - lam y with r = -b_S, x_1 = -(1+eta) w  =>  A_S x_1 = (1+eta)(b_S - lam y)
        want = (1 + eta) * (bS - cfg.lam * y)
    else:
        ASS = A[S][:, S]
        lhs = (ASS + cfg.lam * torch.eye(cfg.s, dtype=A.dtype, device=DEV)) @ x1[S]
        want = (1 + eta) * bS
        off = x1.clone()
        off[S] = 0
        assert float(off.abs().max()) == 0.0  # CD++ touches only the coordinates in S
    err = float(torch.linalg.vector_norm(lhs - want) / torch.linalg.vector_norm(want))
    assert err <= 1e-9, err


@pytest.mark.parametrize("name", ["c2", "c3"])
def test_fullsize_lsqr_parity(kpp, ora, name):
    """K++ with the sketch + LSQR projection (NEXT-2, bench.py --proj 1) at full size, 200 iterations,
    under the DESIGN.md R5 bar max(1e-10, 4 u kappa(G))."""
    cfg = synth.CONFIGS[name]
    A, b, ctx = setup(kpp, cfg)
    ctx.set_option(kpp.OPT_PROJ, 1)
    T = 200
    res = ctx.solve(b, max_iters=T)
    x_gpu = res.x.cpu().numpy()
    S0 = [ctx.block(k).numpy() for k in range(4)]
    An, bn = A.cpu().numpy(), b.cpu().numpy()
    del A
    torch.cuda.empty_cache()
    ref = ora.kpp_run(An, bn, cfg.s, lam=cfg.lam, seed=0, max_iters=T, proj=1, tmax=8, threads=os.cpu_count() or 1)
    kap = max(np.linalg.cond(ora.sketch_factor(An, S, cfg.lam, 0, 2 * cfg.s)) ** 2 for S in S0)
    bar = max(1e-10, 4 * 2.2e-16 * kap)
    assert rel(x_gpu, ref.x) <= bar, (rel(x_gpu, ref.x), kap)
