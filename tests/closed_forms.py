"""Closed forms derived by hand from the paper (no oracle, no CUDA path): shared by the oracle
pins (tests/test_oracle.py) and the GPU tests that check the same special cases."""
import math

import numpy as np


def full_block_window_trace(eta, n_chk, rho0=0.0, rho_max=0.99):
    """Hand reduction of Alg 5 l.9-18 / Alg 3 l.10-20 when the block is
    the whole row set (s = m, so zeta = 1, E0 = ||r_{2i}||^2, E1 = ||r_{2i+1}||^2) and lam = 0,
    x0 = 0, A of full row rank.  Then every projection is onto the full solution set:
    with x_t = alpha_t x_mn, m_t = mu_t x_mn (x_mn = A^T (A A^T)^{-1} b) one has
    r_t = (alpha_t - 1) b, w_t = (alpha_t - 1) x_mn, and the momentum recursion (Eq (momentum)
    P:114-124) collapses to scalars:  mu_{t+1} = c_t (mu_t - (alpha_t - 1)),
    alpha_{t+1} = 1 + eta mu_{t+1},  ||r_t||^2 = (alpha_t - 1)^2 ||b||^2.
    Checkpoint i (after t = 2i - 1): hist_res = sqrt(E1 / ||b||^2) = |alpha_{2i-1} - 1|;
    Eq (weighted) P:728-733 with omega_i = a_{i-1}/a_i, a_j = (j+1)^{ln(j+1)} (Q8), r_hat_0 = 1,
    rho_i = clamp(1 - r_hat_i^{1/zeta}, 0, 0.99) (Q9), zeta = 1.  The rho in force at t is the
    one set at the last checkpoint strictly before t (Q11); rho_0 = 0 (Alg 5 l.4 P:1340) unless given."""
    a = lambda j: math.exp(math.log(j + 1) ** 2)
    alpha, mu, rho, rhat = 0.0, 0.0, rho0, 1.0
    E = [0.0, 0.0]
    res, rhos = [], []
    for t in range(2 * n_chk):
        e = (alpha - 1.0) ** 2  # in units of ||b||^2
        c = (1.0 - rho) / (1.0 + rho)
        mu = c * (mu - (alpha - 1.0))
        alpha = 1.0 + eta * mu
        E[t % 2] += e
        if t % 2 == 1:
            i = t // 2 + 1
            res.append(math.sqrt(E[1]))
            if E[0] > 0:
                om = a(i - 1) / a(i)
                rhat = om * rhat + (1.0 - om) * (E[1] / E[0])
                rho = min(max(1.0 - rhat, 0.0), rho_max)
            rhos.append(rho)
            E = [0.0, 0.0]
    return np.array(res), np.array(rhos)
