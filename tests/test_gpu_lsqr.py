"""GPU parity for K++ with the sketch-and-precondition projection.

Alg 5 with Proj = Alg 6, "K++(LSQR-t_max)" of P:1317-1322: the SRHT
parameters (reading R5) are bit-exact on both sides; the sketch factor R and the iterates agree to
rounding (the GPU memoizes X = R^{-1} and sums in a different order).
"""
import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu

rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))
DEV = "cuda:0"


@pytest.fixture(scope="module")
def kpp():
    import paper_2501_11673_b200 as k
    from paper_2501_11673_b200 import build
    build.build()
    k.load_library()
    assert torch.cuda.is_available()
    return k


def lsqr_ctx(kpp, A, s, lam, seed, tmax=8, tau=0):
    ctx = kpp.kpp_setup(A.to(DEV), s, lam, seed)
    ctx.set_option(kpp.OPT_PROJ, 1)
    ctx.set_option(kpp.OPT_TMAX, tmax)
    if tau:
        ctx.set_option(kpp.OPT_TAU, tau)
    return ctx


def test_sketch_factor(kpp, ora):
    """X = R^{-1} of chol(A_hat A_hat^T + lam I), A_hat = A_S Pi^T (Alg 6 l.3-5)."""
    cfg = synth.twin("c2", 1024, 1000, 96)  # n = 1000: padded to n2 = 1024
    A, b, _ = synth.make_problem(cfg)
    ctx = lsqr_ctx(kpp, A, 96, 1e-8, 7)
    ctx.prepare(20)
    An = A.numpy()
    for k in (0, 3, 11):
        S = ctx.block(k).numpy()
        X = ctx.factor(k).numpy()
        R = ora.sketch_factor(An, S, 1e-8, 7, 2 * 96)
        Ri = np.linalg.inv(R)
        kap = np.linalg.cond(R)
        assert np.allclose(np.tril(X, -1), 0.0)
        assert rel(X, Ri) < 100 * 2.2e-16 * kap * kap, (k, rel(X, Ri), kap)


LSQR_CASES = [synth.twin("c2", 1024, 1024, 128), synth.twin("c3", 2048, 256, 64, k=8),
              synth.twin("c2", 700, 1000, 37), synth.twin("c1", 1024, 512, 32)]


@pytest.mark.parametrize("cfg", LSQR_CASES, ids=[c.name for c in LSQR_CASES])
def test_lsqr_solve_parity(kpp, ora, cfg):
    A, b, _ = synth.make_problem(cfg)
    T = 200
    ref = ora.kpp_run(A.numpy(), b.numpy(), cfg.s, lam=cfg.lam, seed=5, max_iters=T, proj=1, tmax=8)
    ctx = lsqr_ctx(kpp, A, cfg.s, cfg.lam, 5)
    res = ctx.solve(b.to(DEV), max_iters=T)
    assert res.iters == T
    # Alg 6 l.5 factors the sketched Gram matrix: R carries a backward error ~ u kappa(G) on either
    # side (different summation orders), so the bar is max(1e-10, 4 u kappa(G)) (R5)
    An = A.numpy()
    kap = max(np.linalg.cond(ora.sketch_factor(An, ctx.block(k).numpy(), cfg.lam, 5, 2 * cfg.s)) ** 2
              for k in range(4))
    bar = max(1e-10, 4 * 2.2e-16 * kap)
    assert rel(res.x.cpu().numpy(), ref.x) <= bar, (rel(res.x.cpu().numpy(), ref.x), kap)
    assert np.allclose(res.res_hist.numpy(), ref.hist_res, rtol=1e-6, atol=1e-12)
    assert np.allclose(ctx.rho_history().numpy(), ref.hist_rho, rtol=1e-6, atol=1e-12)


@pytest.mark.parametrize("tmax,tau", [(1, 0), (3, 300), (20, 0)])
def test_lsqr_options(kpp, ora, tmax, tau):
    """t_max and the sketch size tau reach both sides."""
    cfg = synth.twin("c2", 512, 512, 64)
    A, b, _ = synth.make_problem(cfg)
    T = 120
    ref = ora.kpp_run(A.numpy(), b.numpy(), 64, lam=cfg.lam, seed=2, max_iters=T, proj=1, tmax=tmax, tau=tau)
    ctx = lsqr_ctx(kpp, A, 64, cfg.lam, 2, tmax=tmax, tau=tau)
    res = ctx.solve(b.to(DEV), max_iters=T)
    # past t_max ~ 16 an LSQR iterate amplifies a perturbation of R by ~1e2 per projection (measured
    # with the oracle: dR/R = 1e-12 -> dw/w = 1e-10 at t = 20), and R itself differs by ~u kappa(G)
    # between the two sides (R5)
    bar = 1e-10 if tmax <= 8 else 1e-6
    assert rel(res.x.cpu().numpy(), ref.x) <= bar


def test_lsqr_tolerance_stop(kpp, ora):
    """Stopping at a checkpoint (Alg 5 l.14-17) happens at the same iteration."""
    cfg = synth.twin("c3", 2048, 256, 64, k=8)
    A, b, _ = synth.make_problem(cfg)
    ref = ora.kpp_run(A.numpy(), b.numpy(), 64, lam=cfg.lam, seed=1, max_iters=20000, tol=1e-6, proj=1)
    ctx = lsqr_ctx(kpp, A, 64, cfg.lam, 1)
    res = ctx.solve(b.to(DEV), max_iters=20000, tol=1e-6)
    assert res.iters == ref.iters
    assert rel(res.x.cpu().numpy(), ref.x) <= 1e-9


def test_lsqr_option_errors(kpp):
    cfg = synth.twin("c5", 256, 256, 32, k=8)
    A, b, _ = synth.make_problem(cfg)
    cd = kpp.cdpp_setup(A.to(DEV), 32, 1e-8, 0)
    with pytest.raises(kpp.KppError):
        cd.set_option(kpp.OPT_PROJ, 1)  # K++ only
    ctx = kpp.kpp_setup(A.to(DEV), 32, 1e-8, 0)
    with pytest.raises(kpp.KppError):
        ctx.set_option(kpp.OPT_PROJ, 2)
    with pytest.raises(kpp.KppError):
        ctx.set_option(kpp.OPT_TMAX, 0)
    ctx.set_option(kpp.OPT_PROJ, 1)
    ctx.solve(b.to(DEV), max_iters=4)
    with pytest.raises(kpp.KppError):
        ctx.set_option(kpp.OPT_TAU, 80)  # the sketch already exists


@pytest.mark.parametrize("cfg", [synth.twin("c3", 1000, 100, 25, k=6), synth.twin("c2", 512, 500, 64)],
                         ids=["tall_ragged", "square_ragged"])
def test_full_kpp_alg5(kpp, ora, cfg):
    """Alg 5 exactly as printed: RHT preprocessing (l.2-3, rows padded to 2^k) AND the
    sketch + LSQR projection (l.10, Alg 6), against the oracle's transcription."""
    A, b, _ = synth.make_problem(cfg)
    T = 200
    ctx = kpp.kpp_setup(A.to(DEV), cfg.s, cfg.lam, 6)
    ctx.enable_rht()
    ctx.set_option(kpp.OPT_PROJ, 1)
    res = ctx.solve(b.to(DEV), max_iters=T)
    ref = ora.kpp_run_rht(A.numpy(), b.numpy(), cfg.s, seed=6, lam=cfg.lam, max_iters=T, proj=1, tmax=8)
    At, _ = ora.rht_rows(A.numpy(), b.numpy(), 6)
    kap = max(np.linalg.cond(ora.sketch_factor(At, ctx.block(k).numpy(), cfg.lam, 6, 2 * cfg.s)) ** 2
              for k in range(4))
    assert rel(res.x.cpu().numpy(), ref.x) <= max(1e-10, 4 * 2.2e-16 * kap)


@pytest.mark.parametrize("s", [1, 2, 33, 64])
def test_lsqr_block_size_edges(kpp, ora, s):
    """Degenerate block sizes for the sketch + LSQR projection: s = 1 (tau = 2), odd s, and s = m
    (every row in one block), on a 64 x 48 system (n padded to 64 for the SRHT)."""
    cfg = synth.twin("c3", 64, 48, s, k=4)
    A, b, _ = synth.make_problem(cfg)
    T = 60
    ref = ora.kpp_run(A.numpy(), b.numpy(), s, lam=cfg.lam, seed=9, max_iters=T, proj=1, tmax=8)
    ctx = lsqr_ctx(kpp, A, s, cfg.lam, 9)
    res = ctx.solve(b.to(DEV), max_iters=T)
    An = A.numpy()
    kap = max(np.linalg.cond(ora.sketch_factor(An, ctx.block(k).numpy(), cfg.lam, 9, min(2 * s, 64))) ** 2
              for k in range(min(3, len(ctx.block(0)))))
    assert rel(res.x.cpu().numpy(), ref.x) <= max(1e-10, 4 * 2.2e-16 * kap)


@pytest.mark.parametrize("opts", [dict(accel=False), dict(memo=False), dict(rho_fixed=0.3), dict(eta=0.01)],
                         ids=["no_accel", "no_memo", "fixed_rho", "eta"])
def test_lsqr_with_options_and_x0(kpp, ora, opts):
    """The LSQR projection under the algorithm options and a start vector, against the oracle."""
    cfg = synth.twin("c2", 256, 200, 32)
    A, b, _ = synth.make_problem(cfg)
    x0 = np.random.default_rng(5).standard_normal(200)
    T = 150
    ref = ora.kpp_run(A.numpy(), b.numpy(), 32, lam=cfg.lam, seed=3, max_iters=T, x0=x0, proj=1, tmax=8, **opts)
    ctx = lsqr_ctx(kpp, A, 32, cfg.lam, 3)
    if "accel" in opts:
        ctx.set_option(kpp.OPT_ACCEL, 0)
    if "memo" in opts:
        ctx.set_option(kpp.OPT_MEMO, 0)
    if "rho_fixed" in opts:
        ctx.set_option(kpp.OPT_RHO_FIXED, opts["rho_fixed"])
    if "eta" in opts:
        ctx.set_option(kpp.OPT_ETA, opts["eta"])
    res = ctx.solve(b.to(DEV), torch.from_numpy(x0).to(DEV), max_iters=T)
    An = A.numpy()
    kap = max(np.linalg.cond(ora.sketch_factor(An, ctx.block(k).numpy(), cfg.lam, 3, 64)) ** 2 for k in range(3))
    assert rel(res.x.cpu().numpy(), ref.x) <= max(1e-10, 4 * 2.2e-16 * kap)
