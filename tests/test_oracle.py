"""Pins for the CPU oracle (oracle/) against what the paper and mathematics fix.

No GPU.  Each test names the passage (P:n = PAPER.md line n) or closed form it checks.
The oracle is never compared with itself through a re-typed formula: pins use closed
forms, library routines (LAPACK via numpy), textbook special cases, published
known-answer vectors, or an independent formulation (three-sequence form, classical
block Kaczmarz, the CD++ -> K++ reduction).
"""
import math
import os

import numpy as np
import pytest
import torch

import synth
from closed_forms import full_block_window_trace as _full_block_window_trace

GOLD = os.path.join(os.path.dirname(__file__), "golden")
rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))


def _rng(seed=0):
    return np.random.default_rng(seed)


# ----------------------------------------------------------------- Philox / schedule
def test_philox_known_answers(ora):
    """Random123 / SC'11 known-answer vectors for Philox-4x32-10."""
    rows = [l.split() for l in open(os.path.join(GOLD, "philox4x32_10_kat.txt")) if not l.startswith("#")]
    assert len(rows) == 3
    for r in rows:
        v = [int(h, 16) for h in r]
        out = ora.philox(v[0:4], v[4:6])
        assert [int(o) for o in out] == v[6:10]


@pytest.mark.parametrize("pop,s", [(1, 1), (7, 7), (10, 3), (256, 32), (1000, 50), (65536, 512), (131072, 256)])
def test_fresh_block_valid(ora, pop, s):
    """S ~ ([pop] choose s): s distinct indices in [0,pop), sorted (Q6)."""
    for k in range(5):
        S = ora.fresh_block(123, pop, s, k)
        assert S.size == s and S.min() >= 0 and S.max() < pop
        assert np.all(np.diff(S) > 0)
    if s == pop:
        assert np.array_equal(ora.fresh_block(1, pop, s, 0), np.arange(pop))


def test_fresh_block_uniform_subsets(ora):
    """Every s-subset is equally likely (partial Fisher-Yates): chi-square over all
    C(6,3)=20 subsets from 20000 independent blocks."""
    from itertools import combinations
    subsets = {c: 0 for c in combinations(range(6), 3)}
    N = 20000
    for k in range(N):
        subsets[tuple(int(v) for v in ora.fresh_block(7, 6, 3, k))] += 1
    exp = N / 20
    chi2 = sum((c - exp) ** 2 / exp for c in subsets.values())
    assert chi2 < 43.8  # chi-square(19) 0.999 quantile


def test_schedule_structure(ora):
    """t=0 fresh (Q4); memo off => always fresh; reuse ids index earlier blocks (Q7)."""
    C = ora.kpp_C(256, 256, 32)
    assert abs(C - (256 / 32) * math.log(256)) < 1e-12
    assert abs(ora.cdpp_C(65536, 512) - 128 * math.log(65536)) < 1e-9
    bid, fresh, nb = ora.schedule(0, C, 5000)
    assert fresh[0] == 1 and bid[0] == 0
    cnt = np.cumsum(fresh)
    assert cnt[-1] == nb
    for t in range(1, 5000):
        if fresh[t]:
            assert bid[t] == cnt[t - 1]
        else:
            assert 0 <= bid[t] < cnt[t - 1]
    # the first floor(C) iterations have p = 1 (min{1, C/t})
    assert fresh[: int(C)].all()
    bid0, fresh0, nb0 = ora.schedule(0, C, 300, memo=False)
    assert fresh0.all() and np.array_equal(bid0, np.arange(300)) and nb0 == 300


def test_schedule_fresh_rate(ora):
    """E[#fresh by T] = 1 + sum_{t=1}^{T-1} min(1, C/t) ~ C(1 + ln(T/C)).
    Mean over 40 seeds within 3 standard errors of the exact expectation."""
    C, T = 44.36, 3000
    expect = 1 + sum(min(1.0, C / t) for t in range(1, T))
    var = sum(min(1.0, C / t) * (1 - min(1.0, C / t)) for t in range(1, T))
    counts = [ora.schedule(seed, C, T)[2] for seed in range(40)]
    se = math.sqrt(var / 40)
    assert abs(np.mean(counts) - expect) < 3.5 * se
    assert abs(expect - C * (1 + math.log(T / C))) / expect < 0.05


def test_reuse_uniform(ora):
    """Reuse draws are uniform over the blocks created so far (Q7): after the fresh
    phase, block ids among reuse iterations of [2000, 60000) with C=20 are ~uniform."""
    bid, fresh, nb = ora.schedule(3, 20.0, 60000)
    sel = (~fresh.astype(bool)) & (np.arange(60000) >= 2000)
    nb_at = np.cumsum(fresh)
    # probability integral transform: (bid + U)/nb_before ~ Uniform(0,1)
    u = (bid[sel] + 0.5) / nb_at[sel]
    hist, _ = np.histogram(u, bins=10, range=(0, 1))
    exp = sel.sum() / 10
    assert np.max(np.abs(hist - exp)) < 5 * math.sqrt(exp)


# ----------------------------------------------------------------- factors
def test_factor_spec_example(ora):
    """chol([[4,2],[2,5]]) = [[2,1],[0,2]] (SPEC dense-linalg cholesky example)."""
    G = np.array([[4.0, 2.0], [2.0, 5.0]])
    R_cd = ora.cdpp_factor(G, np.array([0, 1]), 0.0)
    assert np.allclose(R_cd, [[2, 1], [0, 2]], atol=1e-15)
    # rows (2,0), (1,2) have Gram [[4,2],[2,5]]
    AS = np.array([[2.0, 0.0], [1.0, 2.0]])
    for mode in (ora.HOUSEHOLDER, ora.GRAM):
        R = ora.kpp_factor(AS, np.array([0, 1]), 0.0, mode)
        assert np.allclose(R, [[2, 1], [0, 2]], atol=1e-14)


@pytest.mark.parametrize("mode", ["householder", "gram"])
def test_factor_matches_lapack(ora, mode):
    """R^T R = A_S A_S^T + lam I and R = LAPACK dpotrf (numpy) on a well-conditioned block."""
    rng = _rng(1)
    A = rng.standard_normal((40, 300))
    S = np.array(sorted(rng.choice(40, 12, replace=False)), dtype=np.int32)
    lam = 0.37
    G = A[S] @ A[S].T + lam * np.eye(12)
    R = ora.kpp_factor(A, S, lam, ora.HOUSEHOLDER if mode == "householder" else ora.GRAM)
    assert np.allclose(np.triu(R), R)
    assert np.all(np.diag(R) > 0)
    assert np.linalg.norm(R.T @ R - G) / np.linalg.norm(G) < 1e-14
    Rl = np.linalg.cholesky(G).T
    assert np.linalg.norm(R - Rl) / np.linalg.norm(Rl) < 1e-13


def test_cdpp_factor_matches_lapack(ora):
    rng = _rng(2)
    X = rng.standard_normal((30, 30))
    A = X @ X.T + np.eye(30)
    A = (A + A.T) / 2
    S = np.array([1, 4, 5, 9, 20, 29], dtype=np.int32)
    R = ora.cdpp_factor(A, S, 1e-3)
    Rl = np.linalg.cholesky(A[np.ix_(S, S)] + 1e-3 * np.eye(6)).T
    assert np.linalg.norm(R - Rl) / np.linalg.norm(Rl) < 1e-14


def test_factor_not_pd(ora):
    """lam = 0 with a rank-deficient block -> non-positive pivot (Q13)."""
    A = np.array([[1.0, 1.0], [1.0, 1.0]])
    with pytest.raises(RuntimeError):
        ora.cdpp_factor(A, np.array([0, 1]), 0.0)


# ----------------------------------------------------------------- projection / momentum
def test_projection_hand_example(ora):
    """SPEC regularized_projection example: A_S=[[1,0],[0,1],[1,1]], x=(1,1), b_S=0, lam=1.
    Normal equations by hand: (A_S A_S^T + I) z = (1,1,2) => z=(1/4,1/4,1/2), w = A_S^T z
    = (3/4, 3/4); one accel-off step gives x1 = x - w = (1/4, 1/4)."""
    A = np.array([[1.0, 0.0], [0.0, 1.0], [1.0, 1.0]])
    res = ora.kpp_run(A, np.zeros(3), 3, lam=1.0, max_iters=1, x0=np.ones(2), accel=False)
    assert np.allclose(res.x, [0.25, 0.25], atol=1e-15)


def test_exact_projection_lambda0(ora):
    """lam=0, eta=0: x_{t+1} = x_t - A_S^+(A_S x_t - b_S) solves A_S x = b_S."""
    rng = _rng(3)
    A = rng.standard_normal((64, 48))
    b = rng.standard_normal(64)
    x0 = rng.standard_normal(48)
    for T in (1, 2, 5):
        res = ora.kpp_run(A, b, 16, lam=0.0, max_iters=T, x0=x0, accel=False, seed=5)
        bid, fresh, _ = ora.schedule(5, ora.kpp_C(64, 48, 16), T)
        S = ora.fresh_block(5, 64, 16, int(bid[T - 1]))
        assert np.linalg.norm(A[S] @ res.x - b[S]) <= 1e-12 * np.linalg.norm(b[S])


def test_orthonormal_rows(ora):
    """lam=0 and orthonormal rows: w = A_S^T r (SPEC projection example 1)."""
    rng = _rng(4)
    Q, _ = np.linalg.qr(rng.standard_normal((40, 40)))
    A = Q[:10]  # 10 x 40, orthonormal rows
    b = rng.standard_normal(10)
    x0 = rng.standard_normal(40)
    res = ora.kpp_run(A, b, 10, lam=0.0, max_iters=1, x0=x0, accel=False)
    expect = x0 - A.T @ (A @ x0 - b)
    assert rel(res.x, expect) < 1e-14


def test_large_lambda_shrinks(ora):
    """lam -> 1e12: ||w|| <= 1e-9 ||r|| ||A_S|| (SPEC projection example 2)."""
    rng = _rng(5)
    A = rng.standard_normal((20, 30))
    b = rng.standard_normal(20)
    x0 = rng.standard_normal(30)
    res = ora.kpp_run(A, b, 20, lam=1e12, max_iters=1, x0=x0, accel=False)
    w = x0 - res.x
    r = A @ x0 - b
    assert np.linalg.norm(w) <= 1e-9 * np.linalg.norm(r) * np.linalg.norm(A, 2)


def test_momentum_first_step(ora):
    """rho=0, m_0=0: m_1 = -w_0, x_1 = x_0 - (1+eta) w_0 (Eq (momentum))."""
    rng = _rng(6)
    A = rng.standard_normal((50, 40))
    b = rng.standard_normal(50)
    x0 = rng.standard_normal(40)
    plain = ora.kpp_run(A, b, 10, max_iters=1, x0=x0, accel=False)
    w0 = x0 - plain.x
    acc = ora.kpp_run(A, b, 10, max_iters=1, x0=x0, accel=True)
    eta = 10 / (2 * 40)
    assert rel(acc.x, x0 - (1 + eta) * w0) < 1e-14


def test_rho_one_is_plain_kaczmarz(ora):
    """rho=1 => (1-rho)/(1+rho)=0, m=0: the accelerated update is the plain one (SPEC)."""
    rng = _rng(7)
    A = rng.standard_normal((60, 30))
    b = rng.standard_normal(60)
    a = ora.kpp_run(A, b, 10, max_iters=40, rho_fixed=1.0, accel=True)
    p = ora.kpp_run(A, b, 10, max_iters=40, accel=False)
    assert np.array_equal(a.x, p.x)


def test_three_sequence_equivalence(ora):
    """Lemma equivalence (proof P:1036-1057): the (x,y,v) recursion of
    Eq (alg:main_analyze) with beta = 1-rho, gamma = 1 + eta/rho - eta, alpha = rho/(1+rho),
    v_0 = y_0 = x_0, driven by the same blocks, reproduces the momentum iterates.
    Independent formulation; projections by numpy lstsq on the regularized system."""
    rng = _rng(8)
    m, n, s, lam = 64, 32, 8, 1e-3
    A = rng.standard_normal((m, n))
    b = A @ rng.standard_normal(n)
    rho, eta = 0.3, 0.2
    alpha, beta, gamma = rho / (1 + rho), 1 - rho, 1 + eta / rho - eta
    T = 100
    bid, fresh, nb = ora.schedule(11, ora.kpp_C(m, n, s), T)
    blocks = [ora.fresh_block(11, m, s, k) for k in range(nb)]
    x0 = rng.standard_normal(n)
    y = x0.copy(); v = x0.copy()
    xs = []
    for t in range(T):
        x = alpha * v + (1 - alpha) * y
        xs.append(x)
        S = blocks[bid[t]]
        AS = A[S]
        w = AS.T @ np.linalg.solve(AS @ AS.T + lam * np.eye(s), AS @ x - b[S])
        y_new = x - w
        v = beta * v + (1 - beta) * x - gamma * w
        y = y_new
    xs.append(alpha * v + (1 - alpha) * y)
    for T_chk in (1, 10, 50, 100):
        res = ora.kpp_run(A, b, s, lam=lam, seed=11, max_iters=T_chk, x0=x0, rho_fixed=rho, eta=eta)
        assert rel(res.x, xs[T_chk]) < 1e-10, T_chk


def test_adaptive_rho_example(ora):
    """Eq (weighted) P:728-733 worked example (tests/golden/adaptive_rho_example.txt)."""
    row = [l.split() for l in open(os.path.join(GOLD, "adaptive_rho_example.txt")) if not l.startswith("#")][0]
    i, rprev, E0, E1, zeta = int(row[0]), float(row[1]), float(row[2]), float(row[3]), int(row[4])
    omega, rhat_x, rho_x = map(float, row[5:8])
    assert abs(math.exp(-math.log(2) ** 2) - omega) < 1e-9  # a_0/a_1 = 1/2^{ln 2}
    rh, rho = ora.rho_update(i, rprev, E0, E1, zeta)
    assert abs(rh - rhat_x) < 1e-9 and abs(rho - rho_x) < 1e-9


def test_adaptive_rho_limits(ora):
    """Ratio 1 at every checkpoint is the fixed point r_hat=1 => rho=0; ratio > 1 clamps to 0;
    omega_i = a_{i-1}/a_i with a_i = (i+1)^{ln(i+1)}."""
    rh = 1.0
    for i in range(1, 30):
        rh, rho = ora.rho_update(i, rh, 2.0, 2.0, 8)
        assert rh == pytest.approx(1.0, abs=1e-15) and rho == pytest.approx(0.0, abs=1e-15)
    rh, rho = ora.rho_update(3, 0.5, 1.0, 4.0, 4)
    assert rho == 0.0
    # omega_i from the literal definition, a few i (no overflow at these sizes)
    for i in (1, 2, 5, 20):
        a = lambda j: (j + 1) ** math.log(j + 1)
        om = a(i - 1) / a(i)
        rh, _ = ora.rho_update(i, 0.0, 1.0, 0.5, 4)  # r_hat = (1 - omega) * 0.5
        assert rh == pytest.approx((1 - om) * 0.5, rel=1e-12)
    # tiny ratio -> rho clamped at 0.99
    _, rho = ora.rho_update(1, 1e-300, 1.0, 1e-300, 1)
    assert rho == 0.99


def test_zero_residual_stops_at_first_checkpoint(ora):
    """x0 = x* on a consistent system: every r_t = 0, E1 = 0 <= eps^2 ||b||^2 at the first
    checkpoint t = 2 zeta - 1 (Alg 5 l.15)."""
    rng = _rng(9)
    A = rng.standard_normal((96, 40))
    xs = rng.standard_normal(40)
    b = A @ xs
    res = ora.kpp_run(A, b, 16, max_iters=1000, tol=1e-8, x0=xs)
    zeta = 96 // 16
    assert res.status == ora.OK and res.iters == 2 * zeta
    assert res.hist_res[0] < 1e-14  # zero up to the rounding of b = A x*


def test_window_checkpoint_closed_form(ora):
    """Alg 5 l.13-18 / Alg 3 l.14-20 wiring pinned by a closed form (not by the oracle):
    A = I_64, s = n (zeta = 1), lam = 0, x0 = 0, eta = s/(2n) = 1/2.  First checkpoint:
    hist_res[0] = eta = 0.5 exactly (r_1 = eta b) and rho_1 = 1 - (omega_1 + (1 - omega_1) eta^2)
    with omega_1 = e^{-(ln 2)^2}, i.e. 0.286122647; second checkpoint hist_res[1] = c_1 / 8 with
    c_1 = (1 - rho_1)/(1 + rho_1), and rho_2 from r_hat_2 = omega_2 r_hat_1 + (1 - omega_2) c_1^2 / 4.  Swapping E0/E1 or feeding the wrong checkpoint index to
    omega fails here."""
    om1 = math.exp(-math.log(2) ** 2)
    rho1 = 1.0 - (om1 + (1.0 - om1) * 0.25)
    assert abs(rho1 - 0.286122647) < 1e-9
    c1 = (1 - rho1) / (1 + rho1)
    b = _rng(21).standard_normal(64)
    hr, hp = _full_block_window_trace(0.5, 6)
    # the hand-derived values of the first two checkpoints, restated
    assert hr[0] == 0.5 and abs(hp[0] - rho1) < 1e-15
    assert abs(hr[1] - 0.125 * c1) < 1e-15
    om2 = math.exp(math.log(2) ** 2 - math.log(3) ** 2)
    rhat1 = 1.0 - rho1
    rho2 = min(max(1.0 - (om2 * rhat1 + (1 - om2) * 0.25 * c1 * c1), 0.0), 0.99)
    assert abs(hp[1] - rho2) < 1e-15
    for run in (ora.kpp_run, ora.cdpp_run):
        # 4 checkpoints: the residual falls to ~1e-5 (later ones reach the rounding floor)
        res = run(np.eye(64), b, 64, lam=0.0, max_iters=8)
        hr, hp = hr[:4], hp[:4]
        assert res.iters == 8 and len(res.hist_res) == 4
        assert abs(res.hist_res[0] - 0.5) < 1e-15
        assert abs(res.hist_rho[0] - 0.286122647) < 1e-9
        # rounding: alpha_t - 1 cancels to ~1e-5, so ~1e-11 relative at the 4th checkpoint
        np.testing.assert_allclose(res.hist_res, hr, rtol=1e-10, atol=0)
        np.testing.assert_allclose(res.hist_rho, hp, rtol=1e-10, atol=1e-15)


@pytest.mark.parametrize("rho0,rho_max", [(0.3, 0.99), (0.0, 0.2), (0.6, 0.25)])
def test_window_rho0_rho_max_closed_form(ora, rho0, rho_max):
    """The options rho_0 (Alg 5 l.4 P:1340 fixes 0) and the upper clamp of Q9 (0.99) on the same
    closed form: with rho_max = 0.2 the first update (0.286) is clamped."""
    b = _rng(24).standard_normal(64)
    hr, hp = _full_block_window_trace(0.5, 4, rho0=rho0, rho_max=rho_max)
    if rho0 > 0:
        c0 = (1 - rho0) / (1 + rho0)  # first checkpoint with rho_0: r_1 = eta c_0 b
        assert abs(hr[0] - 0.5 * c0) < 1e-15
    if rho_max < 0.286:
        assert hp[0] == rho_max
    for run in (ora.kpp_run, ora.cdpp_run):
        res = run(np.eye(64), b, 64, lam=0.0, max_iters=8, rho0=rho0, rho_max=rho_max)
        np.testing.assert_allclose(res.hist_res, hr, rtol=1e-10, atol=0)
        np.testing.assert_allclose(res.hist_rho, hp, rtol=1e-10, atol=1e-15)


def test_window_checkpoint_closed_form_general(ora):
    """Same reduction on a general full-row-rank A (32 x 80, s = m = 32, eta = s/(2n) = 0.2):
    hist_res[0] = eta for any A; the whole checkpoint trajectory follows the scalar recursion.
    The final iterate is alpha_T x_mn with x_mn the min-norm solution by LAPACK."""
    rng = _rng(22)
    A = rng.standard_normal((32, 80))
    b = rng.standard_normal(32)
    eta = 32 / (2 * 80)
    n_chk = 4  # residual ~1e-4 at the 4th checkpoint: E1/E0 still far above rounding
    hr, hp = _full_block_window_trace(eta, n_chk)
    res = ora.kpp_run(A, b, 32, lam=0.0, max_iters=2 * n_chk)
    assert abs(res.hist_res[0] - eta) < 1e-12
    np.testing.assert_allclose(res.hist_res, hr, rtol=1e-9, atol=1e-14)
    np.testing.assert_allclose(res.hist_rho, hp, rtol=1e-9, atol=1e-12)
    # x_T = alpha_T x_mn: recompute alpha_T with the same recursion
    alpha, mu, rho = 0.0, 0.0, 0.0
    for t in range(2 * n_chk):
        if t >= 2 and t % 2 == 0:
            rho = hp[t // 2 - 1]
        c = (1 - rho) / (1 + rho)
        mu = c * (mu - (alpha - 1.0))
        alpha = 1.0 + eta * mu
    x_mn = A.T @ np.linalg.solve(A @ A.T, b)
    assert rel(res.x, alpha * x_mn) < 1e-10


def test_window_estimator_partition_identity(ora):
    """SPEC's partition identity for Eq (residual): when the blocks of a window partition
    the row set (here s = m, zeta = 1: one block = all rows) the window sum E equals ||A x - b||^2
    of the iterate the block residual was taken at.  With x0 given and accel off, E0 of the first
    checkpoint is ||A x0 - b||^2 and hist_res[0]^2 ||b||^2 = E1 = ||A x1 - b||^2 with
    x1 = x0 - A^T (A A^T)^{-1} (A x0 - b) = the projection of x0, so E1 = 0 up to rounding; with
    lam > 0 the residual of the regularised step is lam (A A^T + lam I)^{-1} (A x0 - b)."""
    rng = _rng(23)
    A = rng.standard_normal((24, 60))
    b = rng.standard_normal(24)
    x0 = rng.standard_normal(60)
    lam = 0.5
    G = A @ A.T + lam * np.eye(24)
    r0 = A @ x0 - b
    x1 = x0 - A.T @ np.linalg.solve(G, r0)
    res = ora.kpp_run(A, b, 24, lam=lam, max_iters=2, accel=False, x0=x0)
    bb = float(b @ b)
    r1 = A @ x1 - b
    assert abs(res.hist_res[0] ** 2 * bb - float(r1 @ r1)) < 1e-10 * float(r1 @ r1)
    np.testing.assert_allclose(r1, lam * np.linalg.solve(G, r0), rtol=1e-10, atol=1e-12)


# ----------------------------------------------------------------- end-to-end limits
def test_identity_full_block(ora):
    """A = I, s = n, lam = 0, no momentum: one exact projection solves the system (SPEC)."""
    b = _rng(10).standard_normal(64)
    res = ora.kpp_run(np.eye(64), b, 64, lam=0.0, max_iters=2, accel=False)
    assert rel(res.x, b) < 1e-15
    res = ora.cdpp_run(np.eye(64), b, 64, lam=0.0, max_iters=2, accel=False)
    assert rel(res.x, b) < 1e-15


def test_square_converges_to_dense_lu(ora):
    """Tiny well-conditioned square system: iterates -> numpy.linalg.solve (LAPACK getrf)."""
    rng = _rng(11)
    n = 48
    A = rng.standard_normal((n, n)) / math.sqrt(n) + 3 * np.eye(n)
    b = rng.standard_normal(n)
    res = ora.kpp_run(A, b, 12, max_iters=20000, tol=1e-14)
    assert rel(res.x, np.linalg.solve(A, b)) < 1e-11


def test_underdetermined_min_norm(ora):
    """Under-determined consistent system from x0 = 0: the limit is the min-norm
    solution A^T (A A^T)^{-1} b."""
    rng = _rng(12)
    A = rng.standard_normal((24, 96))
    b = rng.standard_normal(24)
    res = ora.kpp_run(A, b, 6, max_iters=40000, tol=1e-14)
    xmn = A.T @ np.linalg.solve(A @ A.T, b)
    assert rel(res.x, xmn) < 1e-9


def test_overdetermined_consistent(ora):
    rng = _rng(13)
    A = rng.standard_normal((200, 20))
    xs = rng.standard_normal(20)
    res = ora.kpp_run(A, A @ xs, 10, max_iters=20000, tol=1e-14)
    assert rel(res.x, xs) < 1e-11


def test_classical_block_kaczmarz(ora):
    """Momentum off + memoization off + lam = 0 is classical randomized block Kaczmarz
    (P:814-823): x <- x - pinv(A_S)(A_S x - b_S) with block k = t."""
    rng = _rng(14)
    m, n, s = 80, 50, 10
    A = rng.standard_normal((m, n))
    b = rng.standard_normal(m)
    x = np.zeros(n)
    for t in range(30):
        S = ora.fresh_block(21, m, s, t)
        x = x - np.linalg.pinv(A[S]) @ (A[S] @ x - b[S])
    res = ora.kpp_run(A, b, s, lam=0.0, seed=21, max_iters=30, accel=False, memo=False)
    assert rel(res.x, x) < 1e-10


def test_synthetic_c1_converges(ora):
    """c1 (BASELINE configs[0]) decreases the residual by > 1e3 in 500 iterations."""
    A, b, xs = synth.make_problem("c1")
    A, b = A.numpy(), b.numpy()
    res = ora.kpp_run(A, b, 32, max_iters=500)
    assert np.linalg.norm(A @ res.x - b) / np.linalg.norm(b) < 1e-3
    assert res.nfresh > 44


def test_noise_floor_c1(ora):
    """Documents the parity floor: the oracle against itself with every sum reversed stays
    well under the 1e-10 bar with Householder factors, while the literal Gram route does not
    (u kappa(A_S)^2) -- the reason the product uses CholeskyQR2."""
    A, b, _ = synth.make_problem("c1")
    A, b = A.numpy(), b.numpy()
    h = ora.kpp_run(A, b, 32, max_iters=200)
    hr = ora.kpp_run(A, b, 32, max_iters=200, reverse=True)
    assert rel(hr.x, h.x) < 3e-11
    g = ora.kpp_run(A, b, 32, max_iters=200, factor=ora.GRAM)
    gr = ora.kpp_run(A, b, 32, max_iters=200, factor=ora.GRAM, reverse=True)
    assert rel(gr.x, g.x) > 3e-11


def test_threads_do_not_change_results(ora):
    A, b, _ = synth.make_problem(synth.twin("c3", 2048, 256, 32))
    A, b = A.numpy(), b.numpy()
    r1 = ora.kpp_run(A, b, 32, max_iters=60)
    r4 = ora.kpp_run(A, b, 32, max_iters=60, threads=4)
    assert np.array_equal(r1.x, r4.x)


# ----------------------------------------------------------------- CD++
def test_cdpp_scalar_coordinate_step(ora):
    """S={i}, lam=0: classical coordinate descent x_i <- x_i - (A_i x - b_i)/A_ii (SPEC cd_step)."""
    rng = _rng(15)
    X = rng.standard_normal((20, 20))
    A = X @ X.T + np.eye(20)
    A = (A + A.T) / 2
    b = rng.standard_normal(20)
    x0 = rng.standard_normal(20)
    res = ora.cdpp_run(A, b, 1, lam=0.0, seed=4, max_iters=1, x0=x0, accel=False)
    i = int(ora.fresh_block(4, 20, 1, 0)[0])
    expect = x0.copy()
    expect[i] -= (A[i] @ x0 - b[i]) / A[i, i]
    assert rel(res.x, expect) < 1e-15


def test_cdpp_reduces_to_kpp(ora):
    """CD++ on A = Phi Phi^T is K++ on Phi z = b with z_t = Phi^T x_t (Eq (implicit)
    P:631-636, Thm t:cd++ proof), same schedule/eta/zeta; <= 1e-9 over 50 iterations."""
    rng = _rng(16)
    n, s = 32, 4
    Phi = rng.standard_normal((n, n)) / math.sqrt(n) + np.eye(n)
    A = Phi @ Phi.T
    A = (A + A.T) / 2
    b = rng.standard_normal(n)
    x0 = rng.standard_normal(n)
    for T in (1, 10, 50):
        c = ora.cdpp_run(A, b, s, lam=1e-6, seed=2, max_iters=T, x0=x0)
        k = ora.kpp_run(Phi, b, s, lam=1e-6, seed=2, max_iters=T, x0=Phi.T @ x0)
        assert np.linalg.norm(k.x - Phi.T @ c.x) / np.linalg.norm(k.x) < 1e-9, T


def test_cdpp_converges_psd(ora):
    """c5 recipe at n=512 (block 64 > 16 spikes, as s=512 > 100 spikes at full size)."""
    cfg = synth.twin("c5", 512, 512, 64, k=16)
    A, b, _ = synth.make_problem(cfg)
    A, b = A.numpy(), b.numpy()
    assert np.array_equal(A, A.T)
    res = ora.cdpp_run(A, b, 64, max_iters=20000, tol=1e-8)
    assert res.status == ora.OK
    assert np.linalg.norm(A @ res.x - b) / np.linalg.norm(b) < 1e-7


# ----------------------------------------------------------------- RHT
def _sylvester(n):
    H = np.array([[1.0]])
    while H.shape[0] < n:
        H = np.block([[H, H], [H, -H]])
    return H


def test_fht_examples(ora):
    """(1,2) -> (3,-1); e_1 (n=4) -> (1,1,1,1); H^2 = n I."""
    assert np.array_equal(ora.fht([1.0, 2.0]), [3.0, -1.0])
    assert np.array_equal(ora.fht([1.0, 0.0, 0.0, 0.0]), [1.0, 1.0, 1.0, 1.0])
    v = np.random.default_rng(0).standard_normal(64)
    assert np.allclose(ora.fht(ora.fht(v)), 64 * v, rtol=0, atol=1e-12 * 64 * np.abs(v).max())


@pytest.mark.parametrize("n", [2, 8, 32, 256])
def test_fht_matches_dense_sylvester(ora, n):
    """Def E.1: H_{2h} = [[H_h, H_h], [H_h, -H_h]] built densely, independent of the butterflies."""
    H = _sylvester(n)
    X = np.random.default_rng(n).standard_normal((n, 3))
    got = np.stack([ora.fht(X[:, j]) for j in range(3)], axis=1)
    assert np.allclose(got, H @ X, rtol=0, atol=1e-12 * n)


def test_rht_signs(ora):
    d = ora.rht_signs(7, 4096)
    assert set(np.unique(d)) == {-1, 1}
    assert abs(int(d.sum())) < 4 * np.sqrt(4096)          # Rademacher balance
    assert np.array_equal(d, ora.rht_signs(7, 4096))     # deterministic
    assert not np.array_equal(d, ora.rht_signs(8, 4096))
    # the convention: lowest bit of word (i mod 4) of philox((i/4, 0, 3, 0), key)
    for i in (0, 1, 5, 4095):
        w = ora.philox([i // 4, 0, 3, 0], [7, 0])
        assert d[i] == (-1 if (w[i % 4] & 1) else 1)


@pytest.mark.parametrize("m,n", [(64, 16), (100, 20), (37, 37)])
def test_rht_rows_isometry_and_solution(ora, m, n):
    """Q = H D with D = diag(d)/sqrt(m2): Q^T Q = I, so Q A has A's singular values and the
    transformed system has A's solutions."""
    rng = np.random.default_rng(m)
    A = rng.standard_normal((m, n))
    x = rng.standard_normal(n)
    b = A @ x
    At, bt = ora.rht_rows(A, b, 3)
    m2 = ora.next_pow2(m)
    assert At.shape == (m2, n)
    H = _sylvester(m2)
    D = np.diag(np.concatenate([ora.rht_signs(3, m).astype(float), np.zeros(m2 - m)])) / np.sqrt(m2)
    Apad = np.vstack([A, np.zeros((m2 - m, n))])
    assert np.allclose(At, H @ D @ Apad, rtol=0, atol=1e-13 * np.abs(A).max() * np.log2(m2) * 4)
    assert np.allclose(np.linalg.svd(At, compute_uv=False), np.linalg.svd(A, compute_uv=False), rtol=1e-12)
    xs = np.linalg.lstsq(At, bt, rcond=None)[0]
    assert np.allclose(xs, x, rtol=0, atol=1e-10)


@pytest.mark.parametrize("n", [16, 24])
def test_rht_sym_conjugation(ora, n):
    """Alg 3 l.3: H D A D H = Q A_pad Q^T is symmetric with the spectrum of A_pad (unit padded diagonal)."""
    rng = np.random.default_rng(n)
    G = rng.standard_normal((n, n))
    A = G @ G.T + np.eye(n)
    b = rng.standard_normal(n)
    At, bt = ora.rht_sym(A, b, 5)
    n2 = ora.next_pow2(n)
    Apad = np.eye(n2)
    Apad[:n, :n] = A
    Q = _sylvester(n2) @ np.diag(np.concatenate([ora.rht_signs(5, n2).astype(float)])) / np.sqrt(n2)
    assert np.allclose(At, Q @ Apad @ Q.T, rtol=0, atol=1e-12 * np.abs(A).max())
    assert np.allclose(At, At.T, rtol=0, atol=1e-12 * np.abs(A).max())
    assert np.allclose(np.linalg.eigvalsh(At), np.linalg.eigvalsh(Apad), rtol=1e-11)
    # back-rotation (Alg 3 l.16): x = D H xt solves A x = b when xt solves the transformed system
    xt = np.linalg.solve(At, bt)
    x = ora.rht_vec(xt, n, n2, 5, False)
    assert np.allclose(A @ x, b, rtol=0, atol=1e-9 * np.abs(b).max())
    # forward then backward is the identity (Q^T Q = I)
    v = rng.standard_normal(n)
    assert np.allclose(ora.rht_vec(ora.rht_vec(v, n, n2, 5, True), n, n2, 5, False), v, rtol=0, atol=1e-13)


def test_spec_symfht_2x2(ora):
    """H [[1,2],[2,3]] H = [[8,-2],[-2,0]] (the unscaled two-sided transform)."""
    A = np.array([[1.0, 2.0], [2.0, 3.0]])
    HA = np.stack([ora.fht(A[:, j]) for j in range(2)], axis=1)
    HAH = np.stack([ora.fht(HA[i, :]) for i in range(2)], axis=0)
    assert np.array_equal(HAH, [[8.0, -2.0], [-2.0, 0.0]])


def test_kpp_rht_converges(ora):
    """Alg 5 with preprocessing (l.2-3): still converges to the solution of the original system."""
    cfg = synth.twin("c3", 1000, 100, 25, k=6)   # over-determined consistent; m padded to 1024
    A, b, xs = synth.make_problem(cfg)
    r = ora.kpp_run_rht(A.numpy(), b.numpy(), 25, seed=0, max_iters=20000, tol=1e-10)
    assert r.status == ora.OK
    assert np.linalg.norm(r.x - xs.numpy()) / np.linalg.norm(xs.numpy()) < 1e-7


def test_cdpp_rht_converges(ora):
    """Alg 3 with SymFHT preprocessing and the back-rotation (l.2-3, l.16), ragged n (padding)."""
    cfg = synth.twin("c5", 200, 200, 32, k=10)
    A, b, _ = synth.make_problem(cfg)
    An, bn = A.numpy(), b.numpy()
    r = ora.cdpp_run_rht(An, bn, 32, seed=1, max_iters=20000, tol=1e-11)
    assert np.linalg.norm(An @ r.x - bn) / np.linalg.norm(bn) < 1e-8


def test_bell_spectrum_generator():
    """NEXT-3 workload: sigma_0 = 1 at er=25, ts=0.01 (SPEC S:229 example); A = Phi Phi^T + phi I has
    eigenvalues sigma_i^2 + phi; bitwise symmetric."""
    prof = synth.bell_profile(64, 25, 0.01)
    assert abs(float(prof[0]) - 1.0) < 1e-15
    assert bool(torch.all(prof[1:] < prof[:-1]))
    A, b = synth.make_bell_psd(64, 8, seed=3)
    A = A.numpy()
    assert np.array_equal(A, A.T)
    ev = np.sort(np.linalg.eigvalsh(A))[::-1]
    want = np.sort(synth.bell_profile(64, 8).numpy() ** 2 + 1e-3)[::-1]
    assert np.allclose(ev, want, rtol=0, atol=1e-12)


def test_bell_general_generator():
    """K++ bell-spectrum systems (App F): the singular values of A are the profile."""
    A, b = synth.make_bell_general(256, 64, 10, seed=5)
    sv = np.linalg.svd(A.numpy(), compute_uv=False)
    want = np.sort(synth.bell_profile(64, 10).numpy())[::-1]
    assert np.allclose(sv, want, rtol=0, atol=1e-13)
    assert A.shape == (256, 64) and b.shape == (256,)


# ----------------------------------------------------------------- sketch + LSQR (NEXT-2)
def test_srht_full_sketch_is_orthogonal(ora):
    """tau = n2 (T = every index): Pi = H D/sqrt(n2) is orthogonal, so A_hat A_hat^T = A_S A_S^T."""
    rng = np.random.default_rng(0)
    A = rng.standard_normal((40, 64))
    S = np.arange(0, 40, 4, dtype=np.int32)
    R = ora.sketch_factor(A, S, 1e-8, 3, 64)
    G = A[S] @ A[S].T + 1e-8 * np.eye(len(S))
    assert np.allclose(R.T @ R, G, rtol=0, atol=1e-12 * np.abs(G).max())
    d, T = ora.srht(3, 64, 64)
    assert np.array_equal(T, np.arange(64)) and set(np.unique(d)) <= {-1.0, 1.0}


def test_srht_subspace_embedding(ora):
    """Lemma l:inner: the preconditioned system is well conditioned; for a Gaussian A_S
    (d_lambda = s) the singular values of the subsampled orthogonal sketch concentrate in
    [1 - sqrt(s/tau), 1 + sqrt(s/tau)] (Marchenko-Pastur), i.e. kappa ~ 5.8 at tau = 2s, 2.4 at 4s."""
    rng = np.random.default_rng(1)
    A = rng.standard_normal((256, 1000))
    s = 32
    S = np.sort(rng.choice(256, s, replace=False)).astype(np.int32)
    lam = 1e-8
    for tau in (2 * s, 4 * s):
        R = ora.sketch_factor(A, S, lam, 5, tau)
        Maug = np.linalg.solve(R.T, np.hstack([A[S], np.sqrt(lam) * np.eye(s)]))
        sv = np.linalg.svd(Maug, compute_uv=False)
        q = np.sqrt(s / tau)
        assert sv[0] / sv[-1] < 1.5 * (1 + q) / (1 - q)


def test_lsqr_converges_to_exact_projection(ora):
    """Alg 6 with many LSQR steps = the exact regularised projection A_S^T (A_S A_S^T + lam I)^{-1} r;
    8 steps are already close for tau = 2s."""
    rng = np.random.default_rng(2)
    A = rng.standard_normal((300, 500))
    s = 40
    S = np.sort(rng.choice(300, s, replace=False)).astype(np.int32)
    lam = 1e-6
    r = rng.standard_normal(s)
    w_exact = A[S].T @ np.linalg.solve(A[S] @ A[S].T + lam * np.eye(s), r)
    R = ora.sketch_factor(A, S, lam, 7, 2 * s)
    w40 = ora.lsqr_proj(A, S, lam, R, r, 40)
    assert np.linalg.norm(w40 - w_exact) / np.linalg.norm(w_exact) < 1e-10
    # 8 steps at kappa ~ 5.8 (flat Gaussian spectrum, d_lambda = s): error ~ ((k-1)/(k+1))^8 ~ 6e-2
    errs = [np.linalg.norm(ora.lsqr_proj(A, S, lam, R, r, t) - w_exact) / np.linalg.norm(w_exact)
            for t in (2, 4, 8, 16)]
    assert all(b2 < a2 for a2, b2 in zip(errs, errs[1:])) and errs[2] < 6e-2


def test_kpp_lsqr_matches_exact_with_many_steps(ora):
    """Alg 5 + Alg 6 with t_max large reproduces K++(Cholesky); with t_max = 8 it still converges."""
    cfg = synth.twin("c3", 1024, 128, 32, k=8)
    A, b, xs = synth.make_problem(cfg)
    An, bn = A.numpy(), b.numpy()
    ex = ora.kpp_run(An, bn, 32, seed=0, max_iters=150, rho_fixed=0.2)
    ls = ora.kpp_run(An, bn, 32, seed=0, max_iters=150, rho_fixed=0.2, proj=1, tmax=60)
    assert np.linalg.norm(ls.x - ex.x) / np.linalg.norm(ex.x) < 1e-9
    l8 = ora.kpp_run(An, bn, 32, seed=0, max_iters=6000, proj=1, tmax=8, tol=1e-8)
    assert l8.status == ora.OK
    assert np.linalg.norm(l8.x - xs.numpy()) / np.linalg.norm(xs.numpy()) < 1e-6
