"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by element.

Bars (BASELINE.json north_star): block schedule bit-exact; ||x_gpu - x_cpu|| / ||x_cpu||
<= 1e-10 after 200 iterations; final relative residuals within 1e-12 absolute.
The oracle uses Householder factors; the GPU uses shifted CholeskyQR2 + the memoized
inverse M = (A_S A_S^T + lam I)^{-1}.
"""
import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu

rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.fixture(scope="module")
def kpp():
    import paper_2501_11673_b200 as k
    from paper_2501_11673_b200 import build
    build.build()
    k.load_library()
    assert torch.cuda.is_available()
    return k


DEV = "cuda:0"


def run_pair(kpp, ora, cfg, T, seed=0, x0=None, tol=0.0, **opts):
    A, b, _ = synth.make_problem(cfg)
    An, bn = A.numpy(), b.numpy()
    s = cfg.s
    if cfg.kind == "cdpp":
        ref = ora.cdpp_run(An, bn, s, lam=cfg.lam, seed=seed, max_iters=T, tol=tol, x0=x0, threads=8)
        ctx = kpp.cdpp_setup(A.to(DEV), s, cfg.lam, seed)
    else:
        ref = ora.kpp_run(An, bn, s, lam=cfg.lam, seed=seed, max_iters=T, tol=tol, x0=x0, threads=8)
        ctx = kpp.kpp_setup(A.to(DEV), s, cfg.lam, seed)
    for k, v in opts.items():
        ctx.set_option(k, v)
    res = ctx.solve(b.to(DEV), None if x0 is None else torch.from_numpy(x0).to(DEV), max_iters=T, tol=tol)
    return An, bn, ref, res, ctx


# ----------------------------------------------------------------- schedule
@pytest.mark.parametrize("m,n,s,T", [(256, 256, 32, 500), (8192, 8192, 128, 200000), (65536, 65536, 512, 50000)])
def test_schedule_bit_exact(kpp, ora, m, n, s, T):
    nc = min(n, 8192)  # only the schedule is used; C depends on min(m, n)
    ctx = kpp.kpp_setup(torch.zeros(m, nc, dtype=torch.float64, device=DEV), s, 1e-8, 7)
    bid, fresh = ctx.schedule(0, T)
    C = ora.kpp_C(m, nc, s)
    rb, rf, nb = ora.schedule(7, C, T)
    assert np.array_equal(bid.numpy(), rb) and np.array_equal(fresh.numpy(), rf)
    # windows starting mid-stream agree too
    bid2, fresh2 = ctx.schedule(T // 3, T // 5)
    assert np.array_equal(bid2.numpy(), rb[T // 3: T // 3 + T // 5])
    # fresh index sets, bit-exact
    for k in list(range(min(nb, 50))) + [nb - 1]:
        assert np.array_equal(ctx.block(k).numpy(), ora.fresh_block(7, m, s, k)), k


def test_philox_against_curand(ora):
    """Both Philox implementations against the toolkit's curand_Philox4x32_10 (test-only)."""
    from torch.utils.cpp_extension import load_inline
    src = r"""
#include <curand_philox4x32_x.h>
__global__ void k(const uint4* c, const uint2* key, uint4* o, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) o[i] = curand_Philox4x32_10(c[i], key[i]);
}
torch::Tensor run(torch::Tensor c, torch::Tensor key) {
  auto o = torch::empty_like(c);
  int n = c.size(0);
  k<<<(n + 127) / 128, 128>>>((const uint4*)c.data_ptr(), (const uint2*)key.data_ptr(), (uint4*)o.data_ptr(), n);
  return o;
}
"""
    try:
        mod = load_inline("philox_kat", cpp_sources="torch::Tensor run(torch::Tensor c, torch::Tensor key);",
                          cuda_sources=src, functions=["run"],
                          extra_cuda_cflags=["-gencode", "arch=compute_100a,code=sm_100a"])
    except Exception as e:  # pragma: no cover - toolchain problem, not a parity failure
        pytest.skip(f"inline extension unavailable: {e}")
    rng = np.random.default_rng(0)
    c = rng.integers(0, 2**32, size=(256, 4), dtype=np.uint64).astype(np.uint32)
    kk = rng.integers(0, 2**32, size=(256, 2), dtype=np.uint64).astype(np.uint32)
    out = mod.run(torch.from_numpy(c.view(np.int32)).to(DEV), torch.from_numpy(kk.view(np.int32)).to(DEV))
    out = out.cpu().numpy().view(np.uint32)
    for i in range(256):
        assert np.array_equal(out[i], ora.philox(c[i], kk[i]))


# ----------------------------------------------------------------- Phase-1 operator
@pytest.mark.parametrize("factor", [0, 1, 2])
def test_factor_operator(kpp, ora, factor):
    """M_k = (A_S A_S^T + lam I)^{-1} from the GPU against the oracle's Householder R
    (M = R^{-1} R^{-T}); error bound ~ u kappa(G)."""
    cfg = synth.twin("c2", 1024, 1024, 128)
    A, b, _ = synth.make_problem(cfg)
    ctx = kpp.kpp_setup(A.to(DEV), 128, 1e-8, 3)
    ctx.set_option(kpp.OPT_FACTOR, factor)
    ctx.prepare(20)
    An = A.numpy()
    for k in (0, 5, 13):
        S = ctx.block(k).numpy()
        assert np.array_equal(S, ora.fresh_block(3, 1024, 128, k))
        M = ctx.factor(k).numpy()
        R = ora.kpp_factor(An, S, 1e-8)
        Ri = np.linalg.inv(R)
        Mref = Ri @ Ri.T
        G = An[S] @ An[S].T + 1e-8 * np.eye(128)
        kap = np.linalg.cond(G)
        assert rel(M, Mref) < 200 * 2.2e-16 * kap, (k, rel(M, Mref), kap)
        assert np.allclose(M, M.T, rtol=0, atol=1e-12 * np.abs(M).max())


@pytest.mark.parametrize("s", [31, 33, 64, 65, 96, 100, 128, 129, 200, 256])
@pytest.mark.parametrize("factor", [1, 2])
def test_factor_operator_ragged(kpp, ora, s, factor):
    """The Gram products' tile edges: 64-row upper-only tiles, the diagonal warp tiles whose
    fragments below the diagonal are skipped, and a split-K whose last 4096-column chunk is ragged
    (n = 4100: the TMA Gram's last stage is 12 columns past n, zero-filled). s = 96 .. 256 run the
    TMA-ring Gram (one CTA per block and chunk up to s = 128, two above; rows past s ragged at 100,
    129, 200). M against the oracle's Householder factor, same bound as above."""
    m, n, lam = 300, 4100, 1e-8
    cfg = synth.twin("c3", m, n, s, k=8)
    A, b, _ = synth.make_problem(cfg)
    ctx = kpp.kpp_setup(A.to(DEV), s, lam, 5)
    ctx.set_option(kpp.OPT_FACTOR, factor)
    ctx.prepare(6)
    An = A.numpy()
    for k in (0, 2):
        S = ctx.block(k).numpy()
        M = ctx.factor(k).numpy()
        Ri = np.linalg.inv(ora.kpp_factor(An, S, lam))
        G = An[S] @ An[S].T + lam * np.eye(s)
        assert rel(M, Ri @ Ri.T) < 200 * 2.2e-16 * np.linalg.cond(G), (s, k, rel(M, Ri @ Ri.T))
        assert np.allclose(M, M.T, rtol=0, atol=1e-12 * np.abs(M).max())


@pytest.mark.parametrize("s,n", [(64, 130), (128, 130), (64, 4100), (128, 4100), (192, 4100), (256, 4100)])
def test_factor_cholqr2_trmm(kpp, ora, s, n):
    """CholeskyQR2 for every block (OPT_FACTOR 0), whose Q1 = X1^T A_S runs on the TMA-ring stripe
    kernel (trmm_tma.cu, s a multiple of 64): 64-column stripes with a ragged last one (n = 130: two
    full stripes and 2 columns, s <= n; n = 4100: 4 columns), the triangle's boxes skipped per stage, pairs of
    row blocks per warp (s = 64: one pair, 256: four).  M against the oracle's Householder factor,
    the bound of test_factor_operator."""
    m, lam = 300, 1e-8
    cfg = synth.twin("c3", m, n, s, k=8)
    A, b, _ = synth.make_problem(cfg)
    ctx = kpp.kpp_setup(A.to(DEV), s, lam, 5)
    ctx.set_option(kpp.OPT_FACTOR, 0)
    ctx.prepare(6)
    An = A.numpy()
    for k in (0, 3):
        S = ctx.block(k).numpy()
        M = ctx.factor(k).numpy()
        Ri = np.linalg.inv(ora.kpp_factor(An, S, lam))
        G = An[S] @ An[S].T + lam * np.eye(s)
        assert rel(M, Ri @ Ri.T) < 200 * 2.2e-16 * np.linalg.cond(G), (s, n, k, rel(M, Ri @ Ri.T))
        assert np.allclose(M, M.T, rtol=0, atol=1e-12 * np.abs(M).max())


@pytest.mark.parametrize("prod", [0, 1, 2])
def test_gram_i8_opt_in(prod):
    """The opt-in int8 tensor-core Gram (gram_i8.cu, tcgen05.mma.kind::i8 on exact 7-digit splittings
    of A, KPP_GRAM_I8=1; read once per process, hence the subprocess) with each operand producer
    (0 TMA gather4, 1 TMA multicast across a cluster pair, 2 cp.async): M against the oracle's
    Householder factor at s = 96, 100 (ragged), 128 with n = 4100 (ragged K), and a c2 twin solve at
    the 1e-10 parity bar after 200 iterations."""
    import os
    import subprocess
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    env = dict(os.environ, KPP_GRAM_I8="1", KPP_GRAM_I8_PROD=str(prod))
    r = subprocess.run([sys.executable, os.path.join(here, "gram_i8_check.py")], env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0 and "gram_i8 ok" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]


@pytest.mark.parametrize("s", [33, 100])
def test_cdpp_factor_operator_ragged(kpp, ora, s):
    cfg = synth.twin("c5", 700, 700, s, k=25)
    A, b, _ = synth.make_problem(cfg)
    ctx = kpp.cdpp_setup(A.to(DEV), s, 1e-8, 2)
    ctx.prepare(4)
    An = A.numpy()
    for k in (0, 1):
        S = ctx.block(k).numpy()
        Ri = np.linalg.inv(ora.cdpp_factor(An, S, 1e-8))
        assert rel(ctx.factor(k).numpy(), Ri @ Ri.T) < 1e-10


def test_cdpp_factor_operator(kpp, ora):
    cfg = synth.twin("c5", 1024, 1024, 128, k=25)
    A, b, _ = synth.make_problem(cfg)
    ctx = kpp.cdpp_setup(A.to(DEV), 128, 1e-8, 1)
    ctx.prepare(10)
    An = A.numpy()
    for k in (0, 4):
        S = ctx.block(k).numpy()
        M = ctx.factor(k).numpy()
        R = ora.cdpp_factor(An, S, 1e-8)
        Ri = np.linalg.inv(R)
        assert rel(M, Ri @ Ri.T) < 1e-11


# ----------------------------------------------------------------- end-to-end parity
def test_persistent_plan(kpp):
    """c2/c3-sized blocks run resident (slab in shared memory) with clusters; c4/c5 stream."""
    for cfg, resident in [(synth.CONFIGS["c2"], 1), (synth.twin("c3", 4096, 4096, 256), 1),
                          (synth.twin("c4", 256, 131072, 256), 0)]:
        A = torch.zeros(cfg.m, cfg.n, dtype=torch.float64, device=DEV)
        ctx = kpp.kpp_setup(A, cfg.s, 1e-8, 0)
        st = ctx.stats()
        assert st["resident"] == resident, (cfg.name, st)
        assert st["grid_ctas"] >= 0.75 * torch.cuda.get_device_properties(0).multi_processor_count
        print(cfg.name, st)


def test_c1_parity_200(kpp, ora):
    """BASELINE configs[0] at its exact size: x after 200 iterations within 1e-10."""
    _, _, ref, res, _ = run_pair(kpp, ora, synth.CONFIGS["c1"], 200)
    assert res.iters == 200
    assert rel(res.x.cpu().numpy(), ref.x) <= 1e-10


def test_c1_final_residual_500(kpp, ora):
    """configs[0]: 500 iterations; final relative residuals within 1e-12 absolute; history agrees."""
    An, bn, ref, res, ctx = run_pair(kpp, ora, synth.CONFIGS["c1"], 500)
    xg = res.x.cpu().numpy()
    rg = np.linalg.norm(An @ xg - bn) / np.linalg.norm(bn)
    rc = np.linalg.norm(An @ ref.x - bn) / np.linalg.norm(bn)
    assert abs(rg - rc) <= 1e-12
    assert np.allclose(res.res_hist.numpy(), ref.hist_res, rtol=1e-6, atol=0)
    assert np.allclose(ctx.rho_history().numpy(), ref.hist_rho, rtol=1e-6, atol=1e-12)


TWINS = [
    synth.twin("c2", 2048, 2048, 128, k=64),       # square, spiked bulk
    synth.twin("c3", 8192, 512, 256),              # over-determined
    synth.twin("c4", 512, 8192, 256),              # under-determined
    synth.twin("c3", 1000, 777, 50, k=8),          # ragged: nothing a multiple of a tile
    synth.twin("c4", 300, 5003, 37, k=8),          # ragged under-determined
    synth.twin("c5", 2048, 2048, 512, k=100),      # CD++ at the real block size
    synth.twin("c5", 1001, 1001, 77, k=16),        # CD++ ragged
]


@pytest.mark.parametrize("cfg", TWINS, ids=[c.name for c in TWINS])
def test_twin_parity_200(kpp, ora, cfg):
    _, _, ref, res, _ = run_pair(kpp, ora, cfg, 200)
    assert res.iters == 200
    assert rel(res.x.cpu().numpy(), ref.x) <= 1e-10


@pytest.mark.parametrize("cfg", [synth.twin("c3", 4096, 512, 64, k=16), synth.twin("c5", 1024, 1024, 128, k=25)],
                         ids=["kpp", "cdpp"])
def test_engines_agree(kpp, ora, cfg):
    """Persistent kernel and step-kernel graph (the multi-GPU engine at P=1) both match the oracle."""
    A, b, _ = synth.make_problem(cfg)
    ref = (ora.cdpp_run if cfg.kind == "cdpp" else ora.kpp_run)(A.numpy(), b.numpy(), cfg.s, max_iters=300, threads=8)
    outs = []
    for eng in (0, 1, 2):
        ctx = (kpp.cdpp_setup if cfg.kind == "cdpp" else kpp.kpp_setup)(A.to(DEV), cfg.s, 1e-8, 0)
        ctx.set_option(kpp.OPT_ENGINE, eng)
        outs.append(ctx.solve(b.to(DEV), max_iters=300).x.cpu().numpy())
        assert ctx.stats()["engine"] == eng
        assert rel(outs[-1], ref.x) <= 1e-10, eng
    assert rel(outs[0], outs[1]) <= 1e-10
    assert rel(outs[0], outs[2]) <= 1e-10


@pytest.mark.parametrize("cfg", TWINS, ids=[c.name for c in TWINS])
def test_fused_exchange_engine(kpp, ora, cfg):
    """Engine 2 (dist.cu: grid reduce + peer-buffer exchange + replicated solve in one persistent
    kernel; the multi-GPU default) on one GPU, self-mapped, against the oracle; a second solve on the
    same context re-arms the tags and gives the same bits."""
    A, b, _ = synth.make_problem(cfg)
    T = 200
    if cfg.kind == "cdpp":
        ctx = kpp.cdpp_setup(A.to(DEV), cfg.s, cfg.lam, 0)
        ref = ora.cdpp_run(A.numpy(), b.numpy(), cfg.s, lam=cfg.lam, seed=0, max_iters=T, threads=8)
    else:
        ctx = kpp.kpp_setup(A.to(DEV), cfg.s, cfg.lam, 0)
        ref = ora.kpp_run(A.numpy(), b.numpy(), cfg.s, lam=cfg.lam, seed=0, max_iters=T, threads=8)
    ctx.set_option(kpp.OPT_ENGINE, 2)
    ctx.set_option(kpp.OPT_WINDOW, 64)  # several launches per solve
    res = ctx.solve(b.to(DEV), max_iters=T)
    assert ctx.stats()["engine"] == 2
    assert rel(res.x.cpu().numpy(), ref.x) <= 1e-10
    assert np.allclose(res.res_hist.numpy(), ref.hist_res, rtol=1e-6, atol=1e-12)
    x1 = res.x.clone()
    assert torch.equal(ctx.solve(b.to(DEV), max_iters=T).x, x1)
    # a start vector and the tolerance stop (checkpoint logic inside the fused kernel)
    x0 = np.random.default_rng(3).standard_normal(A.shape[1])
    run = ora.cdpp_run if cfg.kind == "cdpp" else ora.kpp_run
    ref2 = run(A.numpy(), b.numpy(), cfg.s, lam=cfg.lam, seed=0, max_iters=3000, tol=0.05, x0=x0, threads=8)
    res2 = ctx.solve(b.to(DEV), torch.from_numpy(x0).to(DEV), max_iters=3000, tol=0.05)
    assert res2.iters == ref2.iters
    assert rel(res2.x.cpu().numpy(), ref2.x) <= 1e-10


def test_deterministic_and_warm_cache(kpp):
    """Same inputs -> same bits; a second solve on the same context reuses the memo cache."""
    cfg = synth.twin("c2", 1024, 1024, 64, k=16)
    A, b, _ = synth.make_problem(cfg)
    ctx = kpp.kpp_setup(A.to(DEV), 64, 1e-8, 0)
    x1 = ctx.solve(b.to(DEV), max_iters=400).x.clone()
    nf1 = ctx.stats()["n_fresh_last"]
    x2 = ctx.solve(b.to(DEV), max_iters=400).x.clone()
    assert ctx.stats()["n_fresh_last"] == 0 and nf1 > 0
    assert torch.equal(x1, x2)
    ctx2 = kpp.kpp_setup(A.to(DEV), 64, 1e-8, 0)
    ctx2.set_option(kpp.OPT_WINDOW, 37)  # window boundaries do not change the result
    assert torch.equal(ctx2.solve(b.to(DEV), max_iters=400).x, x1)


def test_host_buffers_equal_device_buffers(kpp):
    cfg = synth.twin("c3", 2048, 256, 32)
    A, b, _ = synth.make_problem(cfg)
    ctx = kpp.kpp_setup(A.to(DEV), 32, 1e-8, 0)
    xd = ctx.solve(b.to(DEV), max_iters=100).x.cpu()
    xh = ctx.solve(b.pin_memory(), max_iters=100, x_out=torch.empty(256, dtype=torch.float64).pin_memory()).x
    assert torch.equal(xd, xh)


def test_stop_matches_oracle(kpp, ora):
    """Tolerance stop (Alg 5 l.15): same stopping checkpoint as the oracle on a case whose
    estimate crosses the threshold with margin; x within the parity bar there."""
    cfg = synth.twin("c3", 4096, 256, 64, k=8)
    An, bn, ref, res, _ = run_pair(kpp, ora, cfg, 20000, tol=1e-6)
    assert ref.status == ora.OK and res.status == 0
    assert res.iters == ref.iters
    assert rel(res.x.cpu().numpy(), ref.x) <= 1e-10


def test_x0_and_options(kpp, ora):
    """x0 given; momentum off; memoization off; fixed rho -- each against the oracle."""
    cfg = synth.twin("c3", 2048, 300, 40, k=8)
    A, b, _ = synth.make_problem(cfg)
    An, bn = A.numpy(), b.numpy()
    x0 = np.random.default_rng(1).standard_normal(300)
    cases = [
        (dict(), dict()),
        (dict(accel=False), {kpp.OPT_ACCEL: 0}),
        (dict(memo=False), {kpp.OPT_MEMO: 0}),
        (dict(rho_fixed=0.2), {kpp.OPT_RHO_FIXED: 0.2}),
        (dict(eta=0.05), {kpp.OPT_ETA: 0.05}),
    ]
    for okw, gopts in cases:
        ref = ora.kpp_run(An, bn, 40, lam=1e-8, seed=2, max_iters=150, x0=x0, **okw)
        ctx = kpp.kpp_setup(A.to(DEV), 40, 1e-8, 2)
        for k, v in gopts.items():
            ctx.set_option(k, v)
        res = ctx.solve(b.to(DEV), torch.from_numpy(x0).to(DEV), max_iters=150)
        assert rel(res.x.cpu().numpy(), ref.x) <= 1e-10, okw


def test_edge_cases(kpp, ora):
    # s = m (one full block), s = 1, max_iters = 0
    rng = np.random.default_rng(5)
    A = rng.standard_normal((48, 64))
    b = rng.standard_normal(48)
    for s in (48, 1, 7):
        ref = ora.kpp_run(A, b, s, lam=1e-8, seed=0, max_iters=60)
        ctx = kpp.kpp_setup(torch.from_numpy(A).to(DEV), s, 1e-8, 0)
        res = ctx.solve(torch.from_numpy(b).to(DEV), max_iters=60)
        assert rel(res.x.cpu().numpy(), ref.x) <= 1e-10, s
    res = ctx.solve(torch.from_numpy(b).to(DEV), max_iters=0)
    assert res.iters == 0 and float(res.x.abs().max()) == 0.0
    # identity, full block, lam = 0, no momentum: exact in one step
    I = torch.eye(64, dtype=torch.float64, device=DEV)
    bb = torch.from_numpy(rng.standard_normal(64)).to(DEV)
    ctx = kpp.kpp_setup(I, 64, 0.0, 0)
    ctx.set_option(kpp.OPT_ACCEL, 0)
    assert torch.allclose(ctx.solve(bb, max_iters=1).x, bb, rtol=1e-15, atol=1e-15)


def test_errors(kpp):
    A = torch.ones(4, 4, dtype=torch.float64, device=DEV)
    with pytest.raises(kpp.KppError) as e:
        kpp.kpp_setup(A, 5)
    assert e.value.status == kpp.EINVAL
    ctx = kpp.kpp_setup(A, 2, 0.0, 0)  # rank-1 rows, lam = 0 -> not positive definite
    with pytest.raises(kpp.KppError) as e:
        ctx.solve(torch.ones(4, dtype=torch.float64, device=DEV), max_iters=5)
    assert e.value.status == kpp.ENOTPD
    B = torch.full((8, 8), float("nan"), dtype=torch.float64, device=DEV)
    ctx = kpp.kpp_setup(torch.eye(8, dtype=torch.float64, device=DEV), 4, 1e-8, 0)
    with pytest.raises(kpp.KppError) as e:
        ctx.solve(torch.full((8,), float("inf"), dtype=torch.float64, device=DEV), max_iters=4)
    assert e.value.status == kpp.EDIVERGED
    del B


def test_cdpp_identity_and_scalar(kpp, ora):
    rng = np.random.default_rng(6)
    X = rng.standard_normal((40, 40))
    A = X @ X.T + np.eye(40)
    A = (A + A.T) / 2
    b = rng.standard_normal(40)
    x0 = rng.standard_normal(40)
    ref = ora.cdpp_run(A, b, 1, lam=0.0, seed=4, max_iters=30, x0=x0, accel=False)
    ctx = kpp.cdpp_setup(torch.from_numpy(A).to(DEV), 1, 0.0, 4)
    ctx.set_option(kpp.OPT_ACCEL, 0)
    res = ctx.solve(torch.from_numpy(b).to(DEV), torch.from_numpy(x0).to(DEV), max_iters=30)
    assert rel(res.x.cpu().numpy(), ref.x) <= 1e-12


PLAN_CASES = [(cfg, y, C) for cfg in (synth.twin("c2", 2048, 2048, 128, k=64), synth.twin("c3", 1000, 778, 50, k=8))
              for y in (0, 1, 4) for C in (0, 2, 8)]


@pytest.mark.parametrize("cfg,ygl,cluster", PLAN_CASES,
                         ids=[f"{c.name}-ygl{y}-C{cc}" for c, y, cc in PLAN_CASES])
def test_launch_plans_parity(kpp, ora, cfg, ygl, cluster):
    """Every placement of y = M r (per cluster / once per GPU / per cluster from partial sums) and
    several cluster sizes give the oracle's iterates."""
    A, b, _ = synth.make_problem(cfg)
    ctx = kpp.kpp_setup(A.to(DEV), cfg.s, cfg.lam, 0)
    try:
        ctx.set_option(kpp.OPT_CLUSTER, cluster)
        ctx.set_option(kpp.OPT_YGL, ygl)
    except kpp.KppError:
        pytest.skip("no feasible plan for this combination")
    st = ctx.stats()
    assert st["ygl"] == ygl
    ref = ora.kpp_run(A.numpy(), b.numpy(), cfg.s, lam=cfg.lam, seed=0, max_iters=300, threads=8)
    res = ctx.solve(b.to(DEV), max_iters=300)
    assert rel(res.x.cpu().numpy(), ref.x) <= 1e-10
    # early stop inside a window (drains in-flight copies) and a second, warm solve
    res2 = ctx.solve(b.to(DEV), max_iters=300, tol=0.5)
    assert res2.iters < 300
    res3 = ctx.solve(b.to(DEV), max_iters=300)
    assert np.array_equal(res3.x.cpu().numpy(), res.x.cpu().numpy())


REASSOC_CASES = [synth.twin("c5", 2048, 2048, 512, k=100), synth.twin("c5", 1001, 1001, 77, k=16),
                 synth.twin("c5", 4096, 4096, 256, k=50)]


@pytest.mark.parametrize("cfg", REASSOC_CASES, ids=[c.name for c in REASSOC_CASES])
@pytest.mark.parametrize("cluster", [0, 2, 8])
def test_cdpp_reassociated_parity(kpp, ora, cfg, cluster):
    """CD++ with the re-associated residual (the c5 streaming kernel), forced on
    small systems: iterates within 1e-10 of the oracle, early stop, x0, warm second solve."""
    A, b, _ = synth.make_problem(cfg)
    ctx = kpp.cdpp_setup(A.to(DEV), cfg.s, cfg.lam, 0)
    ctx.set_option(kpp.OPT_CLUSTER, cluster)
    ctx.set_option(kpp.OPT_REASSOC, 2)
    assert ctx.stats()["reassoc"] == 1
    ref = ora.cdpp_run(A.numpy(), b.numpy(), cfg.s, lam=cfg.lam, seed=0, max_iters=300, threads=8)
    res = ctx.solve(b.to(DEV), max_iters=300)
    assert res.iters == 300
    assert rel(res.x.cpu().numpy(), ref.x) <= 1e-10
    assert np.allclose(res.res_hist.numpy(), ref.hist_res, rtol=1e-6, atol=1e-12)
    # windows of 7 iterations: the pipeline restarts at every launch
    ctx.set_option(kpp.OPT_WINDOW, 7)
    res_w = ctx.solve(b.to(DEV), max_iters=300)
    assert rel(res_w.x.cpu().numpy(), ref.x) <= 1e-10
    # stop at the oracle's iteration
    ref2 = ora.cdpp_run(A.numpy(), b.numpy(), cfg.s, lam=cfg.lam, seed=0, max_iters=3000, tol=0.05, threads=8)
    res2 = ctx.solve(b.to(DEV), max_iters=3000, tol=0.05)
    assert res2.iters == ref2.iters
    assert rel(res2.x.cpu().numpy(), ref2.x) <= 1e-10
    x0 = np.random.default_rng(1).standard_normal(A.shape[1])
    ref3 = ora.cdpp_run(A.numpy(), b.numpy(), cfg.s, lam=cfg.lam, seed=0, max_iters=100, x0=x0, threads=8)
    res3 = ctx.solve(b.to(DEV), torch.from_numpy(x0).to(DEV), max_iters=100)
    assert rel(res3.x.cpu().numpy(), ref3.x) <= 1e-10


@pytest.mark.parametrize("cfg,expect", [(synth.twin("c2", 2048, 2048, 128, k=64), "some"),
                                        (synth.twin("c3", 8192, 512, 256), "all")],
                         ids=["c2twin", "c3twin"])
def test_adaptive_refinement(kpp, ora, cfg, expect):
    """Default factor route: Gram + Cholesky, second CholeskyQR pass only for ill-conditioned blocks
    (estimated 4 u kappa(A_S)^2 > 3e-11).  Iterates within 1e-10 of the oracle either way; the spiked
    over-determined twin (kappa ~ 3e3) refines every block."""
    A, b, _ = synth.make_problem(cfg)
    ctx = kpp.kpp_setup(A.to(DEV), cfg.s, cfg.lam, 0)
    ref = ora.kpp_run(A.numpy(), b.numpy(), cfg.s, lam=cfg.lam, seed=0, max_iters=200, threads=8)
    ctx.reset_stats()
    res = ctx.solve(b.to(DEV), max_iters=200)
    st = ctx.stats()
    assert rel(res.x.cpu().numpy(), ref.x) <= 1e-10
    if expect == "all":
        assert st["n_refined"] == st["n_fresh_last"] > 0
    else:
        assert 0 <= st["n_refined"] <= st["n_fresh_last"]
    # the refined blocks' operators equal the always-CholeskyQR2 route closely
    ctx2 = kpp.kpp_setup(A.to(DEV), cfg.s, cfg.lam, 0)
    ctx2.set_option(kpp.OPT_FACTOR, 0)
    res2 = ctx2.solve(b.to(DEV), max_iters=200)
    assert rel(res.x.cpu().numpy(), res2.x.cpu().numpy()) <= 1e-10


@pytest.mark.parametrize("cfg", [synth.twin("c3", 4096, 512, 64, k=16), synth.twin("c5", 1024, 1024, 128, k=25)],
                         ids=["kpp", "cdpp"])
def test_dist_path_single_rank(kpp, ora, cfg):
    """The column-sharded entry points (kpp_setup_dist / cdpp_setup_dist) with a one-rank NCCL
    communicator: graph engine with the per-iteration allreduce and the per-fresh-block Gram /
    principal-block allreduce inside, against the oracle."""
    A, b, _ = synth.make_problem(cfg)
    uid = kpp.kpp_get_unique_id()
    n = A.shape[1]
    if cfg.kind == "cdpp":
        ctx = kpp.cdpp_setup_dist(A.to(DEV), n, 0, n, cfg.s, cfg.lam, 0, uid, 0, 1)
        ref = ora.cdpp_run(A.numpy(), b.numpy(), cfg.s, lam=cfg.lam, seed=0, max_iters=300, threads=8)
    else:
        ctx = kpp.kpp_setup_dist(A.to(DEV), A.shape[0], n, 0, n, cfg.s, cfg.lam, 0, uid, 0, 1)
        ref = ora.kpp_run(A.numpy(), b.numpy(), cfg.s, lam=cfg.lam, seed=0, max_iters=300, threads=8)
    ctx.set_option(kpp.OPT_ENGINE, 1)  # one rank would otherwise run the persistent kernel
    assert ctx.stats()["xchg"] == 1  # the fused peer exchange (self-mapped with one rank)
    res2 = ctx.solve(b.to(DEV), max_iters=300)
    assert ctx.stats()["engine"] == 1
    ctx.set_option(kpp.OPT_ENGINE, 2)  # the multi-rank default: fused-exchange persistent kernel
    res_e2 = ctx.solve(b.to(DEV), max_iters=300)
    assert ctx.stats()["engine"] == 2
    assert rel(res_e2.x.cpu().numpy(), ref.x) <= 1e-10
    assert rel(res_e2.x.cpu().numpy(), res2.x.cpu().numpy()) <= 1e-12
    ctx.set_option(kpp.OPT_ENGINE, 1)
    res = ctx.solve(b.to(DEV), max_iters=300)
    assert res.iters == 300
    assert rel(res.x.cpu().numpy(), ref.x) <= 1e-10
    assert np.allclose(res.res_hist.numpy(), ref.hist_res, rtol=1e-6, atol=1e-12)
    # the same solve with the NCCL allreduce between kernels: identical bits (rank-order sums)
    x_peer = res.x.clone()
    res2 = ctx.solve(b.to(DEV), max_iters=300)  # a second solve re-arms the tags
    assert torch.equal(res2.x, x_peer)
    ctx.set_option(kpp.OPT_XCHG, 0)
    assert ctx.stats()["xchg"] == 0
    res3 = ctx.solve(b.to(DEV), max_iters=300)
    assert torch.equal(res3.x, x_peer)
    ctx.destroy()


# ----------------------------------------------------------------- RHT preprocessing (NEXT-1)
RHT_CASES = [synth.twin("c3", 1024, 128, 32, k=8), synth.twin("c3", 1000, 100, 25, k=6),
             synth.twin("c5", 512, 512, 64, k=16), synth.twin("c5", 300, 300, 37, k=10)]


@pytest.mark.parametrize("cfg", RHT_CASES, ids=[c.name for c in RHT_CASES])
def test_rht_transform_parity(kpp, ora, cfg):
    """The transformed matrix (H D A or H D A_pad D H) element by element against the oracle."""
    A, b, _ = synth.make_problem(cfg)
    if cfg.kind == "cdpp":
        ctx = kpp.cdpp_setup(A.to(DEV), cfg.s, cfg.lam, 11)
        ref, _ = ora.rht_sym(A.numpy(), b.numpy(), 11)
    else:
        ctx = kpp.kpp_setup(A.to(DEV), cfg.s, cfg.lam, 11)
        ref, _ = ora.rht_rows(A.numpy(), b.numpy(), 11)
    ctx.enable_rht()
    got = ctx.rht_matrix().numpy()
    assert got.shape == ref.shape
    assert np.allclose(got, ref, rtol=0, atol=1e-13 * np.abs(ref).max() * np.log2(ref.shape[0]))


@pytest.mark.parametrize("cfg", RHT_CASES, ids=[c.name for c in RHT_CASES])
def test_rht_solve_parity(kpp, ora, cfg):
    """Alg 5 / Alg 3 with their preprocessing lines (and CD++'s back-rotation): GPU vs oracle."""
    A, b, _ = synth.make_problem(cfg)
    T = 300
    if cfg.kind == "cdpp":
        ctx = kpp.cdpp_setup(A.to(DEV), cfg.s, cfg.lam, 4)
        ref = ora.cdpp_run_rht(A.numpy(), b.numpy(), cfg.s, seed=4, lam=cfg.lam, max_iters=T, threads=8)
    else:
        ctx = kpp.kpp_setup(A.to(DEV), cfg.s, cfg.lam, 4)
        ref = ora.kpp_run_rht(A.numpy(), b.numpy(), cfg.s, seed=4, lam=cfg.lam, max_iters=T, threads=8)
    ctx.enable_rht()
    res = ctx.solve(b.to(DEV), max_iters=T)
    assert res.x.shape[0] == A.shape[1]
    assert rel(res.x.cpu().numpy(), ref.x) <= 1e-10
    assert np.allclose(res.res_hist.numpy(), ref.hist_res, rtol=1e-6, atol=1e-12)
    if cfg.kind == "cdpp":  # x0 goes through Q
        x0 = np.random.default_rng(2).standard_normal(A.shape[1])
        ref0 = ora.cdpp_run_rht(A.numpy(), b.numpy(), cfg.s, seed=4, lam=cfg.lam, max_iters=50, x0=x0, threads=8)
        res0 = ctx.solve(b.to(DEV), torch.from_numpy(x0).to(DEV), max_iters=50)
        assert rel(res0.x.cpu().numpy(), ref0.x) <= 1e-10


def test_rht_dist_kpp(kpp, ora):
    """K++ RHT on a column-sharded context (one rank): the slab transform + the fused-exchange engine
    against the oracle's transformed solve; CD++ column-sharded RHT is refused."""
    cfg = synth.twin("c3", 1000, 100, 25, k=6)
    A, b, _ = synth.make_problem(cfg)
    uid = kpp.kpp_get_unique_id()
    ctx = kpp.kpp_setup_dist(A.to(DEV), A.shape[0], A.shape[1], 0, A.shape[1], cfg.s, cfg.lam, 4, uid, 0, 1)
    ctx.enable_rht()
    ctx.set_option(kpp.OPT_ENGINE, 2)
    res = ctx.solve(b.to(DEV), max_iters=300)
    ref = ora.kpp_run_rht(A.numpy(), b.numpy(), cfg.s, seed=4, lam=cfg.lam, max_iters=300, threads=8)
    assert rel(res.x.cpu().numpy(), ref.x) <= 1e-10
    ctx.destroy()
    c5 = synth.twin("c5", 300, 300, 37, k=10)
    A5, b5, _ = synth.make_problem(c5)
    cd = kpp.cdpp_setup_dist(A5.to(DEV), 300, 0, 300, 37, c5.lam, 4, kpp.kpp_get_unique_id(), 0, 1)
    cd.enable_rht()  # one rank holds the whole matrix: allowed
    cd.destroy()


MAX_CASES = [synth.twin("c3", 2048, 1100, 1024, k=8), synth.twin("c4", 1030, 3000, 1023, k=8),
             synth.twin("c5", 1100, 1100, 1024, k=16), synth.twin("c5", 1100, 1100, 1023, k=16)]


@pytest.mark.parametrize("cfg", MAX_CASES, ids=[c.name for c in MAX_CASES])
def test_max_block_size(kpp, ora, cfg):
    """The largest block the ABI accepts (s = 1024) and an odd neighbour (1023): blocked and one-CTA
    factorisations, slices of a whole CTA's row range in the exchange."""
    A, b, _ = synth.make_problem(cfg)
    T = 40
    if cfg.kind == "cdpp":
        ctx = kpp.cdpp_setup(A.to(DEV), cfg.s, cfg.lam, 0)
        ref = ora.cdpp_run(A.numpy(), b.numpy(), cfg.s, lam=cfg.lam, seed=0, max_iters=T, threads=8)
    else:
        ctx = kpp.kpp_setup(A.to(DEV), cfg.s, cfg.lam, 0)
        ref = ora.kpp_run(A.numpy(), b.numpy(), cfg.s, lam=cfg.lam, seed=0, max_iters=T, threads=8)
    res = ctx.solve(b.to(DEV), max_iters=T)
    assert rel(res.x.cpu().numpy(), ref.x) <= 1e-10


@pytest.mark.parametrize("mode", ["default", "engine2", "lsqr"])
@pytest.mark.parametrize("pad", [3, 4])
@pytest.mark.parametrize("cfg", [synth.twin("c3", 1000, 777, 50, k=8), synth.twin("c5", 301, 301, 37, k=10)],
                         ids=["kpp", "cdpp"])
def test_padded_leading_dimension(kpp, ora, cfg, pad, mode):
    """The C ABI with lda > n (A as the left part of a wider row-major buffer; odd lda disables the
    16-byte paths: TMA, vector loads, the pipelined GEMM) against the oracle."""
    import ctypes
    A, b, _ = synth.make_problem(cfg)
    m, n = A.shape
    buf = torch.full((m, n + pad), float("nan"), dtype=torch.float64, device=DEV)  # padding poisoned
    buf[:, :n] = A.to(DEV)
    L = kpp.load_library()
    h = ctypes.c_void_p()
    if cfg.kind == "cdpp":
        st = L.cdpp_setup(ctypes.byref(h), ctypes.c_void_p(buf.data_ptr()), n, n + pad, cfg.s, cfg.lam, 0)
    else:
        st = L.kpp_setup(ctypes.byref(h), ctypes.c_void_p(buf.data_ptr()), m, n, n + pad, cfg.s, cfg.lam, 0)
    assert st == kpp.OK
    if mode == "lsqr" and cfg.kind == "cdpp":
        L.kpp_destroy(h)
        pytest.skip("sketch + LSQR is a K++ projection")
    if mode == "engine2":
        assert L.kpp_set_option(h, kpp.OPT_ENGINE, 2.0) == kpp.OK
    if mode == "lsqr":
        assert L.kpp_set_option(h, kpp.OPT_PROJ, 1.0) == kpp.OK
    T = 200
    bd = b.to(DEV)
    x = torch.zeros(n, dtype=torch.float64, device=DEV)
    iters = ctypes.c_int64()
    st = L.kpp_solve(h, ctypes.c_void_p(bd.data_ptr()), None, T, 0.0, ctypes.c_void_p(x.data_ptr()), None, 0,
                     None, ctypes.byref(iters))
    assert st in (kpp.OK, kpp.EMAXITER) and iters.value == T
    run = ora.cdpp_run if cfg.kind == "cdpp" else ora.kpp_run
    kw = dict(proj=1, tmax=8) if mode == "lsqr" else {}
    ref = run(A.numpy(), b.numpy(), cfg.s, lam=cfg.lam, seed=0, max_iters=T, threads=8, **kw)
    assert rel(x.cpu().numpy(), ref.x) <= 1e-10
    L.kpp_destroy(h)


@pytest.mark.parametrize("engine", [0, 1, 2])
@pytest.mark.parametrize("cfg,s", [(synth.twin("c3", 96, 40, 1, k=4), 1), (synth.twin("c3", 96, 40, 96, k=4), 96),
                                   (synth.twin("c5", 70, 70, 1, k=4), 1), (synth.twin("c5", 70, 70, 70, k=4), 70)],
                         ids=["kpp_s1", "kpp_sm", "cdpp_s1", "cdpp_sn"])
def test_block_size_extremes_engines(kpp, ora, cfg, s, engine):
    """s = 1 and s = m (K++) / n (CD++) on the persistent and fused-exchange engines, with RHT for
    s = 1 (padding of a non-power-of-2 size)."""
    A, b, _ = synth.make_problem(cfg)
    T = 120
    setup = kpp.cdpp_setup if cfg.kind == "cdpp" else kpp.kpp_setup
    run = ora.cdpp_run if cfg.kind == "cdpp" else ora.kpp_run
    ctx = setup(A.to(DEV), s, cfg.lam, 2)
    ctx.set_option(kpp.OPT_ENGINE, engine)
    res = ctx.solve(b.to(DEV), max_iters=T)
    ref = run(A.numpy(), b.numpy(), s, lam=cfg.lam, seed=2, max_iters=T, threads=8)
    assert rel(res.x.cpu().numpy(), ref.x) <= 1e-10
    if s == 1:
        ctx2 = setup(A.to(DEV), s, cfg.lam, 2)
        ctx2.set_option(kpp.OPT_ENGINE, engine)
        ctx2.enable_rht()
        res2 = ctx2.solve(b.to(DEV), max_iters=T)
        runr = ora.cdpp_run_rht if cfg.kind == "cdpp" else ora.kpp_run_rht
        ref2 = runr(A.numpy(), b.numpy(), s, seed=2, lam=cfg.lam, max_iters=T, threads=8)
        assert rel(res2.x.cpu().numpy(), ref2.x) <= 1e-10


@pytest.mark.parametrize("mode", ["engine0", "engine1", "engine2", "lsqr"])
def test_zero_rhs(kpp, ora, mode):
    """b = 0 from x0 = 0: every residual is zero, x stays 0 and the solve stops at the first checkpoint
    (E1 = 0 <= tol^2 ||b||^2 = 0), as in the oracle."""
    A = torch.from_numpy(np.random.default_rng(8).standard_normal((96, 50)))
    b = torch.zeros(96, dtype=torch.float64)
    ctx = kpp.kpp_setup(A.to(DEV), 12, 1e-8, 0)
    if mode == "lsqr":
        ctx.set_option(kpp.OPT_PROJ, 1)
    else:
        ctx.set_option(kpp.OPT_ENGINE, int(mode[-1]))
    res = ctx.solve(b.to(DEV), max_iters=1000)
    ref = ora.kpp_run(A.numpy(), b.numpy(), 12, lam=1e-8, seed=0, max_iters=1000, proj=1 if mode == "lsqr" else 0)
    assert res.iters == ref.iters == 2 * 8  # zeta = ceil(96 / 12)
    assert float(res.x.abs().max()) == 0.0


@pytest.mark.parametrize("engine", [0, 1, 2])
@pytest.mark.parametrize("kind", ["kpp", "cdpp"])
def test_window_checkpoint_closed_form_gpu(kpp, kind, engine):
    """Alg 5 l.13-18 / Alg 3 l.14-20 on the GPU against the hand-derived closed form (no oracle):
    A = I_64, s = n (zeta = 1), lam = 0, x0 = 0, eta = 1/2: hist_res[0] = 0.5 exactly,
    rho_1 = 1 - (omega_1 + (1 - omega_1)/4) = 0.286122647, then the scalar recursion
    (tests/closed_forms.py) for the next checkpoints; every engine."""
    from closed_forms import full_block_window_trace
    b = torch.from_numpy(np.random.default_rng(21).standard_normal(64))
    A = torch.eye(64, dtype=torch.float64, device=DEV)
    ctx = (kpp.kpp_setup if kind == "kpp" else kpp.cdpp_setup)(A, 64, 0.0, 0)
    ctx.set_option(kpp.OPT_ENGINE, engine)
    res = ctx.solve(b.to(DEV), max_iters=8)
    hr, hp = full_block_window_trace(0.5, 4)
    assert res.iters == 8 and len(res.res_hist) == 4
    assert abs(float(res.res_hist[0]) - 0.5) < 1e-15
    rh = ctx.rho_history().numpy()
    assert abs(rh[0] - 0.286122647) < 1e-9
    np.testing.assert_allclose(res.res_hist.numpy(), hr, rtol=1e-10, atol=0)
    np.testing.assert_allclose(rh, hp, rtol=1e-10, atol=1e-15)
    # KPP_OPT_RHO0 / KPP_OPT_RHO_MAX (closed form with rho_0 = 0.6, the clamp 0.25 active)
    ctx.set_option(kpp.OPT_RHO0, 0.6)
    ctx.set_option(kpp.OPT_RHO_MAX, 0.25)
    res = ctx.solve(b.to(DEV), max_iters=8)
    hr, hp = full_block_window_trace(0.5, 4, rho0=0.6, rho_max=0.25)
    np.testing.assert_allclose(res.res_hist.numpy(), hr, rtol=1e-10, atol=0)
    np.testing.assert_allclose(ctx.rho_history().numpy(), hp, rtol=1e-10, atol=1e-15)
    with pytest.raises(kpp.KppError):
        ctx.set_option(kpp.OPT_RHO_MAX, 1.0)
    with pytest.raises(kpp.KppError):
        ctx.set_option(kpp.OPT_RHO0, -0.1)


VR_TWINS = [synth.twin("c3", 8192, 512, 256), synth.twin("c4", 512, 8192, 256),
            synth.twin("c5", 2048, 2048, 512, k=100), synth.twin("c4", 300, 5003, 37, k=8)]


@pytest.mark.parametrize("P", [2, 3, 4, 8])
@pytest.mark.parametrize("cfg", VR_TWINS, ids=[c.name for c in VR_TWINS])
def test_emulated_ranks_exchange(kpp, ora, cfg, P):
    """SURVEY 8(e) per-iteration exchange with P > 1 ranks, emulated on one GPU inside one cooperative
    launch (B200_PROFILING.md: ranks whose kernels wait on one another are emulated as one kernel over
    all ranks' data): rank v owns columns [v n/P, (v+1) n/P), reduces them over its own grid, publishes
    its tagged partial into EVERY rank's receive buffer and sums the P partials in rank order.  Against
    the oracle at the BJ bar after 200 iterations, the checkpoint history, a start vector with the
    tolerance stop at the oracle's iteration, and bit-identical repeats (the rank-order sum is
    deterministic)."""
    A, b, _ = synth.make_problem(cfg)
    run = ora.cdpp_run if cfg.kind == "cdpp" else ora.kpp_run
    ctx = (kpp.cdpp_setup if cfg.kind == "cdpp" else kpp.kpp_setup)(A.to(DEV), cfg.s, cfg.lam, 0)
    ctx.set_option(kpp.OPT_ENGINE, 2)
    ctx.set_option(kpp.OPT_VRANKS, P)
    ctx.set_option(kpp.OPT_WINDOW, 64)
    T = 200
    ref = run(A.numpy(), b.numpy(), cfg.s, lam=cfg.lam, seed=0, max_iters=T, threads=8)
    res = ctx.solve(b.to(DEV), max_iters=T)
    assert ctx.stats()["engine"] == 2
    assert rel(res.x.cpu().numpy(), ref.x) <= 1e-10
    assert np.allclose(res.res_hist.numpy(), ref.hist_res, rtol=1e-6, atol=1e-12)
    x1 = res.x.clone()
    assert torch.equal(ctx.solve(b.to(DEV), max_iters=T).x, x1)
    x0 = np.random.default_rng(3).standard_normal(A.shape[1])
    ref2 = run(A.numpy(), b.numpy(), cfg.s, lam=cfg.lam, seed=0, max_iters=3000, tol=0.05, x0=x0, threads=8)
    res2 = ctx.solve(b.to(DEV), torch.from_numpy(x0).to(DEV), max_iters=3000, tol=0.05)
    assert res2.iters == ref2.iters
    assert rel(res2.x.cpu().numpy(), ref2.x) <= 1e-10


def test_emulated_ranks_options(kpp):
    A = torch.zeros(64, 64, dtype=torch.float64, device=DEV)
    ctx = kpp.kpp_setup(A, 8, 1e-8, 0)
    for bad in (0, 9, 2.5):
        with pytest.raises(kpp.KppError):
            ctx.set_option(kpp.OPT_VRANKS, bad)
    ctx.set_option(kpp.OPT_VRANKS, 8)


@pytest.mark.parametrize("rht", [False, True], ids=["plain", "rht"])
@pytest.mark.parametrize("er", [25, 200])
def test_bell_psd_parity(kpp, ora, er, rht):
    """NEXT-3: the paper's CD++ test systems, App F P:1302-1306 -- A = Phi Phi^T + 0.001 I,
    n = 4096, bell singular-value profile of effective rank er, b ~ N(0, I), s = 200 --
    GPU against the oracle after 200 iterations at the BJ bar, with and without the randomized Hadamard
    preprocessing (Alg 3 l.2-3 and the back-rotation of l.16: "Full CD++")."""
    A, b = synth.make_bell_psd(4096, effective_rank=er, phi=1e-3, seed=0)
    s, lam, T = 200, 1e-8, 200
    ctx = kpp.cdpp_setup(A.to(DEV), s, lam, 0)
    if rht:
        ctx.enable_rht()
        ref = ora.cdpp_run_rht(A.numpy(), b.numpy(), s, seed=0, lam=lam, max_iters=T, threads=8)
    else:
        ref = ora.cdpp_run(A.numpy(), b.numpy(), s, lam=lam, seed=0, max_iters=T, threads=8)
    res = ctx.solve(b.to(DEV), max_iters=T)
    assert rel(res.x.cpu().numpy(), ref.x) <= 1e-10
    assert np.allclose(res.res_hist.numpy(), ref.hist_res, rtol=1e-6, atol=1e-12)


@pytest.mark.parametrize("accel", [True, False], ids=["momentum", "no_momentum"])
def test_bell_general_parity(kpp, ora, accel):
    """NEXT-3: the paper's K++ system of Fig lsqr_steps (App F): 4096 x 1024 with
    the bell profile (effective rank 50), b ~ N(0, I) (inconsistent), s = 100; GPU against the oracle
    after 200 iterations at the BJ bar, momentum on and off (Table 1 ablation toggle)."""
    A, b = synth.make_bell_general(4096, 1024, effective_rank=50, seed=0)
    s, lam, T = 100, 1e-8, 200
    ctx = kpp.kpp_setup(A.to(DEV), s, lam, 0)
    ctx.set_option(kpp.OPT_ACCEL, 1 if accel else 0)
    ref = ora.kpp_run(A.numpy(), b.numpy(), s, lam=lam, seed=0, max_iters=T, accel=accel, threads=8)
    res = ctx.solve(b.to(DEV), max_iters=T)
    assert rel(res.x.cpu().numpy(), ref.x) <= 1e-10
    assert np.allclose(res.res_hist.numpy(), ref.hist_res, rtol=1e-6, atol=1e-12)


CS_TWINS = [synth.twin("c5", 2048, 2048, 512, k=100), synth.twin("c5", 1001, 1001, 77, k=16),
            synth.twin("c5", 4096, 4096, 256, k=100)]


@pytest.mark.parametrize("P", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("cfg", CS_TWINS, ids=[c.name for c in CS_TWINS])
def test_cdpp_stream_rank_stage(kpp, ora, cfg, P):
    """The CD++ re-associated streaming kernel (row 7) with the rank stage of the column-sharded
    exchange (row 9: the dense pass of t+1 hides the exchange of t), P ranks emulated in
    one cooperative launch: rank v owns columns [v n/P, (v+1) n/P), reduces them over its own clusters,
    publishes its partial of the s-vector into every rank's receive buffer and sums the P partials in
    rank order.  Against the oracle at the BJ bar after 200 iterations, the checkpoint history, the
    tolerance stop with a start vector, and bit-identical repeats."""
    A, b, _ = synth.make_problem(cfg)
    ctx = kpp.cdpp_setup(A.to(DEV), cfg.s, cfg.lam, 0)
    ctx.set_option(kpp.OPT_REASSOC, 2)  # the streaming kernel even where the slab would fit on chip
    ctx.set_option(kpp.OPT_VRANKS, P)
    ctx.set_option(kpp.OPT_WINDOW, 64)
    T = 200
    ref = ora.cdpp_run(A.numpy(), b.numpy(), cfg.s, lam=cfg.lam, seed=0, max_iters=T, threads=8)
    res = ctx.solve(b.to(DEV), max_iters=T)
    st = ctx.stats()
    assert st["engine"] == 0 and st["reassoc"] == 1
    assert rel(res.x.cpu().numpy(), ref.x) <= 1e-10
    assert np.allclose(res.res_hist.numpy(), ref.hist_res, rtol=1e-6, atol=1e-12)
    x1 = res.x.clone()
    assert torch.equal(ctx.solve(b.to(DEV), max_iters=T).x, x1)
    x0 = np.random.default_rng(5).standard_normal(A.shape[1])
    ref2 = ora.cdpp_run(A.numpy(), b.numpy(), cfg.s, lam=cfg.lam, seed=0, max_iters=3000, tol=0.05, x0=x0, threads=8)
    res2 = ctx.solve(b.to(DEV), torch.from_numpy(x0).to(DEV), max_iters=3000, tol=0.05)
    assert res2.iters == ref2.iters
    assert rel(res2.x.cpu().numpy(), ref2.x) <= 1e-10


def test_cdpp_stream_dist_context(kpp, ora):
    """cdpp_setup_dist at one rank (self-mapped receive buffer, one-rank NCCL communicator): the
    automatic engine is the streaming kernel with its rank stage (system-scope peer stores)."""
    cfg = synth.twin("c5", 2048, 2048, 512, k=100)
    A, b, _ = synth.make_problem(cfg)
    n = A.shape[1]
    ctx = kpp.cdpp_setup_dist(A.to(DEV), n, 0, n, cfg.s, cfg.lam, 0, kpp.kpp_get_unique_id(), 0, 1)
    ctx.set_option(kpp.OPT_REASSOC, 2)
    ctx.set_option(kpp.OPT_WINDOW, 64)
    ref = ora.cdpp_run(A.numpy(), b.numpy(), cfg.s, lam=cfg.lam, seed=0, max_iters=200, threads=8)
    res = ctx.solve(b.to(DEV), max_iters=200)
    st = ctx.stats()
    assert st["engine"] == 0 and st["reassoc"] == 1 and st["xchg"] == 1
    assert rel(res.x.cpu().numpy(), ref.x) <= 1e-10
    assert torch.equal(ctx.solve(b.to(DEV), max_iters=200).x, res.x)
    ctx.destroy()


PK_TWINS = VR_TWINS + [synth.twin("c2", 2048, 2048, 128, k=64)]


@pytest.mark.parametrize("P", [2, 3, 4, 8])
@pytest.mark.parametrize("cfg", PK_TWINS, ids=[c.name for c in PK_TWINS])
def test_persistent_rank_stage(kpp, ora, cfg, P):
    """The rank stage of the column-sharded exchange inside the persistent cluster kernel (engine 0:
    TMA slabs, DSMEM cluster reduction, L2 exchange, then the P rank partials through every rank's
    receive buffer, rank-order sums), P ranks emulated in one cooperative launch; the c2-shaped twin
    leaves its one-GPU lean plan for the generic kernel.  Against the oracle (200 iterations at the BJ
    bar, checkpoint history, tolerance stop from x0, bit-identical repeat)."""
    A, b, _ = synth.make_problem(cfg)
    run = ora.cdpp_run if cfg.kind == "cdpp" else ora.kpp_run
    ctx = (kpp.cdpp_setup if cfg.kind == "cdpp" else kpp.kpp_setup)(A.to(DEV), cfg.s, cfg.lam, 0)
    ctx.set_option(kpp.OPT_ENGINE, 0)
    if cfg.kind == "cdpp":
        ctx.set_option(kpp.OPT_REASSOC, 0)  # the generic kernel (the streaming one has its own test)
    ctx.set_option(kpp.OPT_VRANKS, P)
    ctx.set_option(kpp.OPT_WINDOW, 64)
    T = 200
    ref = run(A.numpy(), b.numpy(), cfg.s, lam=cfg.lam, seed=0, max_iters=T, threads=8)
    res = ctx.solve(b.to(DEV), max_iters=T)
    assert ctx.stats()["engine"] == 0
    assert rel(res.x.cpu().numpy(), ref.x) <= 1e-10
    assert np.allclose(res.res_hist.numpy(), ref.hist_res, rtol=1e-6, atol=1e-12)
    x1 = res.x.clone()
    assert torch.equal(ctx.solve(b.to(DEV), max_iters=T).x, x1)
    x0 = np.random.default_rng(3).standard_normal(A.shape[1])
    ref2 = run(A.numpy(), b.numpy(), cfg.s, lam=cfg.lam, seed=0, max_iters=3000, tol=0.05, x0=x0, threads=8)
    res2 = ctx.solve(b.to(DEV), torch.from_numpy(x0).to(DEV), max_iters=3000, tol=0.05)
    assert res2.iters == ref2.iters
    assert rel(res2.x.cpu().numpy(), ref2.x) <= 1e-10


def test_persistent_dist_context(kpp, ora):
    """kpp_setup_dist at one rank (self-mapped receive buffer): the automatic engine of a column-sharded
    K++ context is the persistent kernel with its rank stage (the generic kernel: a one-GPU context of
    this shape would run the lean one)."""
    cfg = synth.twin("c3", 8192, 512, 256)
    A, b, _ = synth.make_problem(cfg)
    n = A.shape[1]
    ctx = kpp.kpp_setup_dist(A.to(DEV), A.shape[0], n, 0, n, cfg.s, cfg.lam, 0, kpp.kpp_get_unique_id(), 0, 1)
    ctx.set_option(kpp.OPT_WINDOW, 64)
    ref = ora.kpp_run(A.numpy(), b.numpy(), cfg.s, lam=cfg.lam, seed=0, max_iters=200, threads=8)
    res = ctx.solve(b.to(DEV), max_iters=200)
    st = ctx.stats()
    assert st["engine"] == 0 and st["xchg"] == 1
    assert rel(res.x.cpu().numpy(), ref.x) <= 1e-10
    assert torch.equal(ctx.solve(b.to(DEV), max_iters=200).x, res.x)
    ctx.destroy()


LEAN_CASES = [synth.twin("c3", 8192, 512, 256), synth.twin("c3", 6000, 1000, 200, k=16),
              synth.twin("c3", 4096, 300, 126, k=8), synth.twin("c2", 700, 700, 32, k=8)]


@pytest.mark.parametrize("cfg", LEAN_CASES, ids=[c.name for c in LEAN_CASES])
def test_lean_kernel_shapes(kpp, ora, cfg):
    """The lean register-tile kernel at its shape limits -- slices of 64 rows with one M-row buffer
    (s = 256, 200), ragged s and n, short windows (several launches), the tolerance stop from x0 (the
    early-exit drain of the in-flight slab / M-row copies) -- against the oracle at the BJ bar, and a
    repeated solve bit-identical."""
    A, b, _ = synth.make_problem(cfg)
    ctx = kpp.kpp_setup(A.to(DEV), cfg.s, cfg.lam, 0)
    ctx.set_option(kpp.OPT_WINDOW, 96)
    ref = ora.kpp_run(A.numpy(), b.numpy(), cfg.s, lam=cfg.lam, seed=0, max_iters=200, threads=8)
    res = ctx.solve(b.to(DEV), max_iters=200)
    assert rel(res.x.cpu().numpy(), ref.x) <= 1e-10
    assert np.allclose(res.res_hist.numpy(), ref.hist_res, rtol=1e-6, atol=1e-12)
    x0 = np.random.default_rng(7).standard_normal(A.shape[1])
    ref2 = ora.kpp_run(A.numpy(), b.numpy(), cfg.s, lam=cfg.lam, seed=0, max_iters=5000, tol=0.02, x0=x0, threads=8)
    res2 = ctx.solve(b.to(DEV), torch.from_numpy(x0).to(DEV), max_iters=5000, tol=0.02)
    assert res2.iters == ref2.iters and res2.status == ref2.status
    assert rel(res2.x.cpu().numpy(), ref2.x) <= 1e-10
    # the same solve again: the drained copies left no stale phase behind
    res3 = ctx.solve(b.to(DEV), torch.from_numpy(x0).to(DEV), max_iters=5000, tol=0.02)
    assert torch.equal(res3.x, res2.x)


@pytest.mark.parametrize("s", [2, 4, 6, 30, 66])
def test_lean_kernel_small_slices(kpp, ora, s):
    """The lean kernel with slices of 0-1 rows on some CTAs of a cluster (s < cluster size x ...),
    slices that do not fill a warp and ones just above 32 / 64 rows per cluster: against the oracle."""
    cfg = synth.twin("c2", 600, 600, s, k=8)
    A, b, _ = synth.make_problem(cfg)
    ctx = kpp.kpp_setup(A.to(DEV), s, cfg.lam, 1)
    ref = ora.kpp_run(A.numpy(), b.numpy(), s, lam=cfg.lam, seed=1, max_iters=150, threads=8)
    res = ctx.solve(b.to(DEV), max_iters=150)
    assert rel(res.x.cpu().numpy(), ref.x) <= 1e-10
    assert np.allclose(res.res_hist.numpy(), ref.hist_res, rtol=1e-6, atol=1e-12)
