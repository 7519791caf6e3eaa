// kpp_oracle.cpp -- TEST INFRASTRUCTURE ONLY (see kpp_oracle.h).
//
// A plain sequential CPU transcription of the paper's algorithms, in the paper's
// order and notation.  No blocking, no fusion, no reordering: each loop below is
// one line of Alg 5 or Alg 3.  Only tests/, smoke() and
// bench.py's cpu_baseline use it; the CUDA product shares no code with it.
#include "kpp_oracle.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>
#ifdef _OPENMP
#include <omp.h>
#endif

namespace {

// ---------------------------------------------------------------- Philox-4x32-10
// Salmon, Moraes, Dror, Shaw, "Parallel random numbers: as easy as 1, 2, 3" (SC'11).
// The paper is silent on the RNG (Q4-Q7); this generator is the binding convention.
const uint32_t PH_M0 = 0xD2511F53u, PH_M1 = 0xCD9E8D57u;
const uint32_t PH_W0 = 0x9E3779B9u, PH_W1 = 0xBB67AE85u;

void philox(const uint32_t in[4], const uint32_t key[2], uint32_t out[4]) {
  uint32_t c0 = in[0], c1 = in[1], c2 = in[2], c3 = in[3];
  uint32_t k0 = key[0], k1 = key[1];
  for (int round = 0; round < 10; ++round) {
    if (round > 0) { k0 += PH_W0; k1 += PH_W1; }
    uint64_t p0 = (uint64_t)PH_M0 * (uint64_t)c0;
    uint64_t p1 = (uint64_t)PH_M1 * (uint64_t)c2;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c1 ^ k0;
    uint32_t n1 = lo1;
    uint32_t n2 = hi0 ^ c3 ^ k1;
    uint32_t n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

void seed_key(uint64_t seed, uint32_t key[2]) {
  key[0] = (uint32_t)(seed & 0xffffffffu);
  key[1] = (uint32_t)(seed >> 32);
}

// Decision stream for iteration t: counter (lo32 t, hi32 t, 1, 0).
// word0 -> Bernoulli draw, word1 -> reuse draw (Q4, Q7).
void decision_words(uint64_t seed, int64_t t, uint32_t out[4]) {
  uint32_t key[2];
  seed_key(seed, key);
  uint64_t ut = (uint64_t)t;
  uint32_t ctr[4] = {(uint32_t)(ut & 0xffffffffu), (uint32_t)(ut >> 32), 1u, 0u};
  philox(ctr, key, out);
}

// Is the block at iteration t fresh?  Bernoulli(min{1, C/t}) with p_0 = 1 (Q4):
// Alg 5 line 6 / Alg 3 line 6.  u = word0 * 2^-32 exactly.
bool is_fresh(uint64_t seed, double C, int32_t memo, int64_t t, uint32_t* word1) {
  uint32_t w[4];
  decision_words(seed, t, w);
  *word1 = w[1];
  if (t == 0 || !memo) return true;
  double p = std::min(1.0, C / (double)t);
  double u = (double)w[0] * 0x1p-32;
  return u < p;
}

// Reuse: S ~ uniform over the nb blocks drawn before t (Q7).
int64_t reuse_index(uint32_t word1, int64_t nb) {
  return (int64_t)(((uint64_t)word1 * (uint64_t)nb) >> 32);
}

// Fresh block k: S ~ ([pop] choose s), sampled by a partial Fisher-Yates shuffle of
// the array [0..pop) (Q6); draw i uses word (i mod 4) of counter (i/4, lo32 k, 2, hi32 k).
void fresh_block(uint64_t seed, int64_t pop, int32_t s, int64_t k, int32_t* S) {
  std::vector<int32_t> perm((size_t)pop);
  for (int64_t i = 0; i < pop; ++i) perm[(size_t)i] = (int32_t)i;
  uint32_t key[2];
  seed_key(seed, key);
  uint64_t uk = (uint64_t)k;
  uint32_t w[4] = {0, 0, 0, 0};
  for (int32_t i = 0; i < s; ++i) {
    if (i % 4 == 0) {
      uint32_t ctr[4] = {(uint32_t)(i / 4), (uint32_t)(uk & 0xffffffffu), 2u, (uint32_t)(uk >> 32)};
      philox(ctr, key, w);
    }
    uint32_t u = w[i % 4];
    int64_t j = i + (int64_t)(((uint64_t)u * (uint64_t)(pop - i)) >> 32);
    std::swap(perm[(size_t)i], perm[(size_t)j]);
  }
  for (int32_t i = 0; i < s; ++i) S[i] = perm[(size_t)i];
  std::sort(S, S + s);
}

// ---------------------------------------------------------------- small dense algebra
struct Par {
  int threads;
  bool rev;
};

// Cholesky, upper: R^T R = G (row-major s x s).  Column-by-column (textbook).
int cholesky_upper(const std::vector<double>& G, int32_t s, bool rev, double* R) {
  std::fill(R, R + (size_t)s * s, 0.0);
  for (int32_t j = 0; j < s; ++j) {
    double acc = 0.0;
    for (int32_t q = 0; q < j; ++q) {
      int32_t k = rev ? (j - 1 - q) : q;
      acc += R[(size_t)k * s + j] * R[(size_t)k * s + j];
    }
    double d = G[(size_t)j * s + j] - acc;
    if (!(d > 0.0)) return ORA_ENOTPD;
    double rjj = std::sqrt(d);
    R[(size_t)j * s + j] = rjj;
    for (int32_t l = j + 1; l < s; ++l) {
      double a = 0.0;
      for (int32_t q = 0; q < j; ++q) {
        int32_t k = rev ? (j - 1 - q) : q;
        a += R[(size_t)k * s + j] * R[(size_t)k * s + l];
      }
      R[(size_t)j * s + l] = (G[(size_t)j * s + l] - a) / rjj;
    }
  }
  return ORA_OK;
}

// Householder QR of M = [A_S^T ; sqrt(lam) I_s]  ((n+s) x s), returning the upper
// factor with positive diagonal.  R^T R = M^T M = A_S A_S^T + lam I exactly in real
// arithmetic, i.e. R = chol(A_S A_S^T + lam I), computed backward-stably (Q18).
int householder_factor(const double* A, int64_t lda, int64_t n, const int32_t* S, int32_t s,
                       double lam, const Par& par, double* R) {
  const int64_t L = n + s;
  std::vector<double> M((size_t)L * s);  // column-major: column c at M[c*L]
  for (int32_t c = 0; c < s; ++c) {
    double* col = &M[(size_t)c * L];
    const double* arow = A + (size_t)S[c] * lda;
    for (int64_t i = 0; i < n; ++i) col[i] = arow[i];
    for (int32_t i = 0; i < s; ++i) col[n + i] = (i == c) ? std::sqrt(lam) : 0.0;
  }
  std::fill(R, R + (size_t)s * s, 0.0);
  for (int32_t j = 0; j < s; ++j) {
    double* v = &M[(size_t)j * L];
    const int64_t len = L - j;
    double nrm2 = 0.0;
    for (int64_t q = 0; q < len; ++q) {
      int64_t i = par.rev ? (L - 1 - q) : (j + q);
      nrm2 += v[i] * v[i];
    }
    double nrm = std::sqrt(nrm2);
    if (!(nrm > 0.0)) return ORA_ENOTPD;
    double alpha = (v[j] >= 0.0) ? -nrm : nrm;
    v[j] -= alpha;  // v[j:] is now the Householder vector u
    double uu = 0.0;
    for (int64_t q = 0; q < len; ++q) {
      int64_t i = par.rev ? (L - 1 - q) : (j + q);
      uu += v[i] * v[i];
    }
    R[(size_t)j * s + j] = alpha;
#pragma omp parallel for schedule(static) num_threads(par.threads) if (par.threads > 1)
    for (int32_t c = j + 1; c < s; ++c) {
      double* col = &M[(size_t)c * L];
      double d = 0.0;
      for (int64_t q = 0; q < len; ++q) {
        int64_t i = par.rev ? (L - 1 - q) : (j + q);
        d += v[i] * col[i];
      }
      double f = 2.0 * d / uu;
      for (int64_t i = j; i < L; ++i) col[i] -= f * v[i];
      R[(size_t)j * s + c] = col[j];
    }
  }
  // sign fix: rows with negative diagonal are negated (Q R = (Q D)(D R), D = diag(+-1))
  for (int32_t j = 0; j < s; ++j) {
    if (R[(size_t)j * s + j] < 0.0)
      for (int32_t c = j; c < s; ++c) R[(size_t)j * s + c] = -R[(size_t)j * s + c];
  }
  return ORA_OK;
}

int gram_factor(const double* A, int64_t lda, int64_t n, const int32_t* S, int32_t s, double lam,
                const Par& par, double* R) {
  std::vector<double> G((size_t)s * s);
#pragma omp parallel for schedule(static) num_threads(par.threads) if (par.threads > 1)
  for (int32_t k = 0; k < s; ++k) {
    for (int32_t l = 0; l < s; ++l) {
      const double* ak = A + (size_t)S[k] * lda;
      const double* al = A + (size_t)S[l] * lda;
      double g = 0.0;
      for (int64_t q = 0; q < n; ++q) {
        int64_t j = par.rev ? (n - 1 - q) : q;
        g += ak[j] * al[j];
      }
      G[(size_t)k * s + l] = g + ((k == l) ? lam : 0.0);
    }
  }
  return cholesky_upper(G, s, par.rev, R);
}

int cdpp_factor(const double* A, int64_t lda, const int32_t* S, int32_t s, double lam,
                const Par& par, double* R) {
  std::vector<double> G((size_t)s * s);
  for (int32_t k = 0; k < s; ++k)
    for (int32_t l = 0; l < s; ++l)
      G[(size_t)k * s + l] = A[(size_t)S[k] * lda + S[l]] + ((k == l) ? lam : 0.0);
  return cholesky_upper(G, s, par.rev, R);
}

// y = (R^T R)^{-1} r by forward substitution R^T z = r then back substitution R y = z.
void chol_solve(const double* R, int32_t s, const double* r, bool rev, double* y) {
  std::vector<double> z((size_t)s);
  for (int32_t k = 0; k < s; ++k) {
    double a = 0.0;
    for (int32_t q = 0; q < k; ++q) {
      int32_t l = rev ? (k - 1 - q) : q;
      a += R[(size_t)l * s + k] * z[(size_t)l];
    }
    z[(size_t)k] = (r[k] - a) / R[(size_t)k * s + k];
  }
  for (int32_t k = s - 1; k >= 0; --k) {
    double a = 0.0;
    for (int32_t q = 0; q < s - 1 - k; ++q) {
      int32_t l = rev ? (k + 1 + q) : (s - 1 - q);
      a += R[(size_t)k * s + l] * y[l];
    }
    y[k] = (z[(size_t)k] - a) / R[(size_t)k * s + k];
  }
}

// Adaptive rho, Eq (weighted) P:728-733 with omega_i = a_{i-1}/a_i, a_i = (i+1)^{ln(i+1)} (Q8),
// rho = 1 - rhat^{1/zeta}, clamped to [0, 0.99] (Q9).
// a_{i-1}/a_i = exp(ln(i)^2 - ln(i+1)^2)  (same value; avoids overflow of a_i).
void rho_update(int64_t i, double rhat_prev, double E0, double E1, int64_t zeta, double* rhat,
                double* rho, double rho_max = 0.99) {
  double li = std::log((double)i), li1 = std::log((double)(i + 1));
  double omega = std::exp(li * li - li1 * li1);
  double rh = omega * rhat_prev + (1.0 - omega) * (E1 / E0);
  double rr = 1.0 - std::pow(rh, 1.0 / (double)zeta);
  if (rr < 0.0) rr = 0.0;
  if (rr > rho_max) rr = rho_max;
  *rhat = rh;
  *rho = rr;
}

struct Block {
  std::vector<int32_t> S;
  std::vector<double> R;
};

// ---------------------------------------------------------------- sketch + LSQR (NEXT-2)
int64_t next_pow2_(int64_t n) {
  int64_t p = 1;
  while (p < n) p <<= 1;
  return p;
}

void fht_inplace(double* v, int64_t n) {  // Sylvester order, half-sizes 1, 2, 4, ... (Def E.1)
  for (int64_t h = 1; h < n; h <<= 1)
    for (int64_t i0 = 0; i0 < n; i0 += 2 * h)
      for (int64_t i = i0; i < i0 + h; ++i) {
        const double a = v[i], b = v[i + h];
        v[i] = a + b;
        v[i + h] = a - b;
      }
}

// SRHT parameters (reading R5): d_j = +-1 (stream 4: word (j mod 4) of counter (lo32(j/4),
// hi32(j/4), 4, 0), lowest bit), T = sorted first tau entries of a partial Fisher-Yates shuffle of
// [0, n2) drawing word (i mod 4) of counter (i/4, 0, 5, 0).
void srht_params(uint64_t seed, int64_t n2, int32_t tau, std::vector<double>& d, std::vector<int32_t>& T) {
  uint32_t key[2];
  seed_key(seed, key);
  d.assign((size_t)n2, 0.0);
  for (int64_t j = 0; j < n2; ++j) {
    const uint64_t c = (uint64_t)j >> 2;
    uint32_t ctr[4] = {(uint32_t)(c & 0xffffffffu), (uint32_t)(c >> 32), 4u, 0u}, w[4];
    philox(ctr, key, w);
    d[(size_t)j] = (w[j & 3] & 1u) ? -1.0 : 1.0;
  }
  std::vector<int32_t> perm((size_t)n2);
  for (int64_t i = 0; i < n2; ++i) perm[(size_t)i] = (int32_t)i;
  uint32_t w[4] = {0, 0, 0, 0};
  for (int32_t i = 0; i < tau; ++i) {
    if (i % 4 == 0) {
      uint32_t ctr[4] = {(uint32_t)(i / 4), 0u, 5u, 0u};
      philox(ctr, key, w);
    }
    const int64_t j = i + (int64_t)(((uint64_t)w[i % 4] * (uint64_t)(n2 - i)) >> 32);
    std::swap(perm[(size_t)i], perm[(size_t)j]);
  }
  T.assign(perm.begin(), perm.begin() + tau);
  std::sort(T.begin(), T.end());
}

// Alg 6 l.3-4: A_hat = A_S Pi^T, Pi = sqrt(n2/tau) I_T H diag(d)/sqrt(n2) = I_T H diag(d)/sqrt(tau);
// R = chol(A_hat A_hat^T + lam I).
int sketch_factor(const double* A, int64_t lda, int64_t n, const int32_t* S, int32_t s, double lam, uint64_t seed,
                  int32_t tau, double* R) {
  const int64_t n2 = next_pow2_(n);
  if (tau < 1 || tau > n2) return ORA_EINVAL;  // T is tau distinct rows of the n2-point transform
  std::vector<double> d;
  std::vector<int32_t> T;
  srht_params(seed, n2, tau, d, T);
  std::vector<double> Ah((size_t)s * tau), v((size_t)n2);
  const double sc = 1.0 / std::sqrt((double)tau);
  for (int32_t k = 0; k < s; ++k) {
    for (int64_t j = 0; j < n2; ++j) v[(size_t)j] = j < n ? d[(size_t)j] * A[(size_t)S[k] * lda + j] : 0.0;
    fht_inplace(v.data(), n2);
    for (int32_t q = 0; q < tau; ++q) Ah[(size_t)k * tau + q] = sc * v[(size_t)T[(size_t)q]];
  }
  std::vector<double> G((size_t)s * s);
  for (int32_t k = 0; k < s; ++k)
    for (int32_t l = 0; l < s; ++l) {
      double a = 0.0;
      for (int32_t q = 0; q < tau; ++q) a += Ah[(size_t)k * tau + q] * Ah[(size_t)l * tau + q];
      G[(size_t)k * s + l] = a + ((k == l) ? lam : 0.0);
    }
  return cholesky_upper(G, s, false, R);
}

// z = R^{-T} v (forward substitution), z = R^{-1} v (back substitution); R upper s x s
void solve_rt(const double* R, int32_t s, const double* v, double* z) {
  for (int32_t k = 0; k < s; ++k) {
    double a = v[k];
    for (int32_t l = 0; l < k; ++l) a -= R[(size_t)l * s + k] * z[l];
    z[k] = a / R[(size_t)k * s + k];
  }
}
void solve_r(const double* R, int32_t s, const double* v, double* z) {
  for (int32_t k = s - 1; k >= 0; --k) {
    double a = v[k];
    for (int32_t l = k + 1; l < s; ++l) a -= R[(size_t)k * s + l] * z[l];
    z[k] = a / R[(size_t)k * s + k];
  }
}

// Alg 6 l.6-8: LSQR (Paige & Saunders 1982, Algorithm LSQR) on M z = R^{-T} r with
// M = R^{-T} [A_S, sqrt(lam) I] (implicit), z0 = 0, exactly tmax steps; returns w = z[0:n].
// Degenerate steps (a zero beta or alpha) leave the normalised vector at 0.
void lsqr_proj(const double* A, int64_t lda, int64_t n, const int32_t* S, int32_t s, double lam, const double* R,
               const double* r, int32_t tmax, double* wout) {
  const double sl = std::sqrt(lam);
  std::vector<double> u((size_t)s), t1((size_t)s), t2((size_t)s), vn((size_t)n), vs((size_t)s),
      xn((size_t)n, 0.0), xs((size_t)s, 0.0), wn((size_t)n), ws((size_t)s);
  // [on; os] = M^T uu = [A_S^T R^{-1} uu; sqrt(lam) R^{-1} uu]
  auto matvec_t = [&](const std::vector<double>& uu, std::vector<double>& on, std::vector<double>& os) {
    solve_r(R, s, uu.data(), t1.data());
    for (int64_t j = 0; j < n; ++j) {
      double acc = 0.0;
      for (int32_t k = 0; k < s; ++k) acc += A[(size_t)S[k] * lda + j] * t1[(size_t)k];
      on[(size_t)j] = acc;
    }
    for (int32_t k = 0; k < s; ++k) os[(size_t)k] = sl * t1[(size_t)k];
  };
  // out = M [zn; zs] = R^{-T} (A_S zn + sqrt(lam) zs)
  auto matvec = [&](const std::vector<double>& zn, const std::vector<double>& zs, std::vector<double>& out) {
    for (int32_t k = 0; k < s; ++k) {
      double acc = 0.0;
      for (int64_t j = 0; j < n; ++j) acc += A[(size_t)S[k] * lda + j] * zn[(size_t)j];
      t2[(size_t)k] = acc + sl * zs[(size_t)k];
    }
    solve_rt(R, s, t2.data(), out.data());
  };
  auto nrm = [](const std::vector<double>& a, const std::vector<double>* b2) {
    double q = 0.0;
    for (double v : a) q += v * v;
    if (b2)
      for (double v : *b2) q += v * v;
    return std::sqrt(q);
  };
  auto scale = [](std::vector<double>& a, double d) {
    for (double& v : a) v = d > 0.0 ? v / d : 0.0;
  };
  // beta_1 u_1 = b,  alpha_1 v_1 = M^T u_1,  w_1 = v_1,  phibar_1 = beta_1,  rhobar_1 = alpha_1
  std::vector<double> rr(r, r + s);
  solve_rt(R, s, rr.data(), u.data());
  double beta = nrm(u, nullptr);
  scale(u, beta);
  matvec_t(u, vn, vs);
  double alpha = nrm(vn, &vs);
  scale(vn, alpha);
  scale(vs, alpha);
  wn = vn;
  ws = vs;
  double phibar = beta, rhobar = alpha;
  std::vector<double> mv((size_t)s), qn((size_t)n), qs((size_t)s);
  for (int32_t it = 0; it < tmax; ++it) {
    // beta u = M v - alpha u
    matvec(vn, vs, mv);
    for (int32_t k = 0; k < s; ++k) u[(size_t)k] = mv[(size_t)k] - alpha * u[(size_t)k];
    beta = nrm(u, nullptr);
    scale(u, beta);
    // alpha v = M^T u - beta v
    matvec_t(u, qn, qs);
    for (int64_t j = 0; j < n; ++j) vn[(size_t)j] = qn[(size_t)j] - beta * vn[(size_t)j];
    for (int32_t k = 0; k < s; ++k) vs[(size_t)k] = qs[(size_t)k] - beta * vs[(size_t)k];
    alpha = nrm(vn, &vs);
    scale(vn, alpha);
    scale(vs, alpha);
    // plane rotation
    const double rho = std::sqrt(rhobar * rhobar + beta * beta);
    const double c = rho > 0.0 ? rhobar / rho : 1.0, sn = rho > 0.0 ? beta / rho : 0.0;
    const double theta = sn * alpha;
    rhobar = -c * alpha;
    const double phi = c * phibar;
    phibar = sn * phibar;
    // x = x + (phi/rho) w;  w = v - (theta/rho) w
    const double f1 = rho > 0.0 ? phi / rho : 0.0, f2 = rho > 0.0 ? theta / rho : 0.0;
    for (int64_t j = 0; j < n; ++j) {
      xn[(size_t)j] += f1 * wn[(size_t)j];
      wn[(size_t)j] = vn[(size_t)j] - f2 * wn[(size_t)j];
    }
    for (int32_t k = 0; k < s; ++k) {
      xs[(size_t)k] += f1 * ws[(size_t)k];
      ws[(size_t)k] = vs[(size_t)k] - f2 * ws[(size_t)k];
    }
  }
  for (int64_t j = 0; j < n; ++j) wout[j] = xn[(size_t)j];
}

// The shared outer loop of Alg 5 / Alg 3 (lines 5-18).  `cd` selects CD++.
int run(bool cd, const double* A, int64_t m, int64_t n, int64_t lda, const double* b,
        const double* x0, int32_t s, double lam, uint64_t seed, int64_t max_iters, double tol,
        const ora_opts* opt_in, double* x_out, double* hist_res, double* hist_rho,
        int64_t hist_cap, int64_t* n_hist, int64_t* iters_out, int64_t* nfresh_out) {
  ora_opts opt = {1, 1, -1.0, -1.0, ORA_FACTOR_HOUSEHOLDER, 0, 1, 0, 8, 0, 0.0, 0.99, nullptr};
  if (opt_in) opt = *opt_in;
  const int64_t pop = cd ? n : m;  // sampling population: rows (K++) or coordinates (CD++)
  if (s < 1 || s > pop || lam < 0.0 || tol < 0.0 || max_iters < 0 || lda < n) return ORA_EINVAL;
  Par par{opt.threads < 1 ? 1 : opt.threads, opt.reverse != 0};

  // Initialisation (Alg 5 l.4 P:1340 / Alg 3 l.4 P:748)
  const double C = cd ? ora_cdpp_C(n, s) : ora_kpp_C(m, n, s);
  const int64_t zeta = (pop + s - 1) / s;
  const double eta = opt.accel ? (opt.eta_override >= 0.0 ? opt.eta_override : (double)s / (2.0 * (double)n)) : 0.0;
  double rho = opt.rho_fixed >= 0.0 ? opt.rho_fixed : opt.rho0;  // rho_0 (Alg 5 l.4 P:1340: 0)
  double rhat = 1.0, E0 = 0.0, E1 = 0.0;
  int64_t ichk = 0, nh = 0;
  std::vector<double> x((size_t)n), mom((size_t)n, 0.0), w((size_t)n, 0.0);
  for (int64_t j = 0; j < n; ++j) x[(size_t)j] = x0 ? x0[j] : 0.0;
  double bb = 0.0;
  for (int64_t q = 0; q < pop; ++q) {
    int64_t j = par.rev ? (pop - 1 - q) : q;
    bb += b[j] * b[j];
  }
  std::vector<Block> cache;
  int64_t nfresh = 0;
  std::vector<double> r((size_t)s), y((size_t)s);
  Block scratch;
  int status = ORA_EMAXITER;
  const double t_run0 = omp_get_wtime();
  double t_factor = 0.0;
  int64_t t = 0;
  for (; t < max_iters; ++t) {
    // line 6-8: block selection with memoization
    uint32_t word1;
    const Block* blk;
    if (is_fresh(seed, C, opt.memo, t, &word1)) {
      Block nbk;
      nbk.S.resize((size_t)s);
      nbk.R.resize((size_t)s * s);
      fresh_block(seed, pop, s, opt.memo ? nfresh : t, nbk.S.data());
      const double tf0 = omp_get_wtime();
      int rc;
      const bool lsqr = !cd && opt.proj == 1;
      // tau = 2s (Alg 5 l.4), at most the padded dimension n2 (R5)
      const int32_t tau = opt.tau > 0 ? opt.tau : (int32_t)std::min<int64_t>(2 * (int64_t)s, next_pow2_(n));
      if (cd)
        rc = cdpp_factor(A, lda, nbk.S.data(), s, lam, par, nbk.R.data());
      else if (lsqr)
        rc = sketch_factor(A, lda, n, nbk.S.data(), s, lam, seed, tau, nbk.R.data());  // Alg 6 l.2-5
      else if (opt.factor == ORA_FACTOR_GRAM)
        rc = gram_factor(A, lda, n, nbk.S.data(), s, lam, par, nbk.R.data());
      else
        rc = householder_factor(A, lda, n, nbk.S.data(), s, lam, par, nbk.R.data());
      t_factor += omp_get_wtime() - tf0;
      if (rc != ORA_OK) { status = rc; break; }
      ++nfresh;
      if (opt.memo) {
        cache.push_back(std::move(nbk));
        blk = &cache.back();
      } else {
        scratch = std::move(nbk);
        blk = &scratch;
      }
    } else {
      blk = &cache[(size_t)reuse_index(word1, (int64_t)cache.size())];
    }
    const int32_t* S = blk->S.data();
    // line 9 / 10: r_t = A_S x_t - b_S
#pragma omp parallel for schedule(static) num_threads(par.threads) if (par.threads > 1)
    for (int32_t k = 0; k < s; ++k) {
      const double* arow = A + (size_t)S[k] * lda;
      double a = 0.0;
      for (int64_t q = 0; q < n; ++q) {
        int64_t j = par.rev ? (n - 1 - q) : q;
        a += arow[j] * x[(size_t)j];
      }
      r[(size_t)k] = a - b[S[k]];
    }
    // line 10 / 11: y = (A_S A_S^T + lam I)^{-1} r (K++) or (A_SS + lam I)^{-1} r (CD++)
    if (!cd && opt.proj == 1) {
      // Alg 5 l.10 with Proj = Alg 6: w_t from tmax LSQR steps on the preconditioned system
      lsqr_proj(A, lda, n, S, s, lam, blk->R.data(), r.data(), opt.tmax, w.data());
    } else {
      chol_solve(blk->R.data(), s, r.data(), par.rev, y.data());
    }
    // w_t = A_S^T y (K++, Eq (bk)) or I_S^T y (CD++, Alg 3 l.11)
    if (!cd && opt.proj == 1) {
      // w already holds the LSQR solution
    } else if (cd) {
      std::fill(w.begin(), w.end(), 0.0);
      for (int32_t k = 0; k < s; ++k) w[(size_t)S[k]] = y[(size_t)k];
    } else {
#pragma omp parallel for schedule(static) num_threads(par.threads) if (par.threads > 1)
      for (int64_t j = 0; j < n; ++j) {
        double a = 0.0;
        for (int32_t q = 0; q < s; ++q) {
          int32_t k = par.rev ? (s - 1 - q) : q;
          a += A[(size_t)S[k] * lda + j] * y[(size_t)k];
        }
        w[(size_t)j] = a;
      }
    }
    // lines 11-12: m_{t+1} = (1-rho)/(1+rho) (m_t - w_t);  x_{t+1} = x_t - w_t + eta m_{t+1}
    const double c = (1.0 - rho) / (1.0 + rho);
    for (int64_t j = 0; j < n; ++j) {
      mom[(size_t)j] = c * (mom[(size_t)j] - w[(size_t)j]);
      x[(size_t)j] = x[(size_t)j] - w[(size_t)j] + eta * mom[(size_t)j];
    }
    // line 13: window accumulation of ||r_t||^2 (Eq (residual), Q10)
    double e = 0.0;
    for (int32_t q = 0; q < s; ++q) {
      int32_t k = par.rev ? (s - 1 - q) : q;
      e += r[(size_t)k] * r[(size_t)k];
    }
    if (!std::isfinite(e)) { status = ORA_EDIVERGED; ++t; break; }
    if (t % (2 * zeta) < zeta) E0 += e; else E1 += e;
    // lines 14-18: checkpoint
    if (t % (2 * zeta) == 2 * zeta - 1) {
      ++ichk;
      bool stop = E1 <= tol * tol * bb;
      if (!stop && opt.rho_fixed < 0.0 && E0 > 0.0) rho_update(ichk, rhat, E0, E1, zeta, &rhat, &rho, opt.rho_max);
      if (nh < hist_cap) {
        if (hist_res) hist_res[nh] = std::sqrt(E1 / bb);
        if (hist_rho) hist_rho[nh] = rho;
      }
      ++nh;
      E0 = E1 = 0.0;
      if (stop) { status = ORA_OK; ++t; break; }
    }
  }
  for (int64_t j = 0; j < n; ++j) x_out[j] = x[(size_t)j];
  if (opt.timing) {
    opt.timing[0] = omp_get_wtime() - t_run0;
    opt.timing[1] = t_factor;
    opt.timing[2] = (double)nfresh;
  }
  if (n_hist) *n_hist = nh;
  if (iters_out) *iters_out = t;
  if (nfresh_out) *nfresh_out = nfresh;
  return status;
}

// ---------------------------------------------------------------- RHT
// Def 1.1: Q = H D, D = diag(d)/sqrt(m2), d_i Rademacher.  Sign stream (binding
// convention, reading R3): word (i mod 4) of philox((lo32(i/4), hi32(i/4), 3, 0), key),
// d_i = -1 if its lowest bit is set, else +1.
int rht_sign(uint64_t seed, int64_t i) {
  uint32_t key[2];
  seed_key(seed, key);
  const uint64_t c = (uint64_t)i >> 2;
  uint32_t ctr[4] = {(uint32_t)(c & 0xffffffffu), (uint32_t)(c >> 32), 3u, 0u};
  uint32_t w[4];
  philox(ctr, key, w);
  return (w[i & 3] & 1u) ? -1 : 1;
}

int64_t next_pow2(int64_t n) {
  int64_t p = 1;
  while (p < n) p <<= 1;
  return p;
}

// H_n v in place for the n = 2^k values v[0], v[stride], ...: Sylvester's recursion
// H_{2h} = [[H_h, H_h], [H_h, -H_h]] (Def E.1 convention; Alg 4 P:1230-1243 prints the second
// half with the opposite sign, SPEC S:189/S:204 -- we follow the definition), one butterfly
// (a, b) -> (a + b, a - b) per pair, half-sizes h = 1, 2, 4, ...
void fht(double* v, int64_t n, int64_t stride) {
  for (int64_t h = 1; h < n; h <<= 1)
    for (int64_t i0 = 0; i0 < n; i0 += 2 * h)
      for (int64_t i = i0; i < i0 + h; ++i) {
        const double a = v[i * stride], b = v[(i + h) * stride];
        v[i * stride] = a + b;
        v[(i + h) * stride] = a - b;
      }
}

}  // namespace

extern "C" {

void ora_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  philox(ctr, key, out);
}

void ora_fresh_block(uint64_t seed, int64_t pop, int32_t s, int64_t k, int32_t* S_out) {
  fresh_block(seed, pop, s, k, S_out);
}

int64_t ora_schedule(uint64_t seed, double C, int32_t memo, int64_t T, int32_t* bid, uint8_t* fresh) {
  int64_t nb = 0;
  for (int64_t t = 0; t < T; ++t) {
    uint32_t word1;
    if (is_fresh(seed, C, memo, t, &word1)) {
      bid[t] = (int32_t)nb;
      fresh[t] = 1;
      ++nb;
    } else {
      bid[t] = (int32_t)reuse_index(word1, nb);
      fresh[t] = 0;
    }
  }
  return nb;
}

double ora_kpp_C(int64_t m, int64_t n, int32_t s) {
  return ((double)std::min(m, n) / (double)s) * std::log((double)m);
}

double ora_cdpp_C(int64_t n, int32_t s) { return ((double)n / (double)s) * std::log((double)n); }

int ora_kpp_factor(const double* A, int64_t lda, int64_t n, const int32_t* S, int32_t s, double lam,
                   int32_t mode, int32_t reverse, double* R) {
  Par par{1, reverse != 0};
  if (mode == ORA_FACTOR_GRAM) return gram_factor(A, lda, n, S, s, lam, par, R);
  return householder_factor(A, lda, n, S, s, lam, par, R);
}

int ora_cdpp_factor(const double* A, int64_t lda, const int32_t* S, int32_t s, double lam,
                    int32_t reverse, double* R) {
  Par par{1, reverse != 0};
  return cdpp_factor(A, lda, S, s, lam, par, R);
}

int ora_kpp_run(const double* A, int64_t m, int64_t n, int64_t lda, const double* b, const double* x0,
                int32_t s, double lam, uint64_t seed, int64_t max_iters, double tol, const ora_opts* opt,
                double* x_out, double* hist_res, double* hist_rho, int64_t hist_cap, int64_t* n_hist,
                int64_t* iters_out, int64_t* nfresh_out) {
  return run(false, A, m, n, lda, b, x0, s, lam, seed, max_iters, tol, opt, x_out, hist_res, hist_rho,
             hist_cap, n_hist, iters_out, nfresh_out);
}

int ora_cdpp_run(const double* A, int64_t n, int64_t lda, const double* b, const double* x0, int32_t s,
                 double lam, uint64_t seed, int64_t max_iters, double tol, const ora_opts* opt,
                 double* x_out, double* hist_res, double* hist_rho, int64_t hist_cap, int64_t* n_hist,
                 int64_t* iters_out, int64_t* nfresh_out) {
  return run(true, A, n, n, lda, b, x0, s, lam, seed, max_iters, tol, opt, x_out, hist_res, hist_rho,
             hist_cap, n_hist, iters_out, nfresh_out);
}

void ora_rho_update(int64_t i, double rhat_prev, double E0, double E1, int64_t zeta, double* rhat_out,
                    double* rho_out) {
  rho_update(i, rhat_prev, E0, E1, zeta, rhat_out, rho_out);
}

int64_t ora_next_pow2(int64_t n) { return next_pow2(n); }

void ora_srht(uint64_t seed, int64_t n, int32_t tau, double* d_out, int32_t* T_out) {
  std::vector<double> d;
  std::vector<int32_t> T;
  srht_params(seed, next_pow2_(n), tau, d, T);
  for (size_t i = 0; i < d.size(); ++i) d_out[i] = d[i];
  for (size_t i = 0; i < T.size(); ++i) T_out[i] = T[i];
}

int ora_sketch_factor(const double* A, int64_t lda, int64_t n, const int32_t* S, int32_t s, double lam,
                      uint64_t seed, int32_t tau, double* R) {
  return sketch_factor(A, lda, n, S, s, lam, seed, tau, R);
}

void ora_lsqr_proj(const double* A, int64_t lda, int64_t n, const int32_t* S, int32_t s, double lam,
                   const double* R, const double* r, int32_t tmax, double* w) {
  lsqr_proj(A, lda, n, S, s, lam, R, r, tmax, w);
}

void ora_rht_signs(uint64_t seed, int64_t n, int8_t* d) {
  for (int64_t i = 0; i < n; ++i) d[i] = (int8_t)rht_sign(seed, i);
}

void ora_fht(double* v, int64_t n) { fht(v, n, 1); }

// K++ preprocessing (Alg 5 l.2-3): At = H D [A; 0] (m2 x n, row-major, ld n),
// bt = H D [b; 0] (m2); m2 = next power of 2 >= m, D = diag(d)/sqrt(m2).
void ora_rht_rows(const double* A, int64_t m, int64_t n, int64_t lda, const double* b, uint64_t seed,
                  double* At, double* bt) {
  const int64_t m2 = next_pow2(m);
  const double sc = 1.0 / std::sqrt((double)m2);
  for (int64_t i = 0; i < m2; ++i) {
    const double di = i < m ? rht_sign(seed, i) * sc : 0.0;
    for (int64_t j = 0; j < n; ++j) At[i * n + j] = i < m ? di * A[i * lda + j] : 0.0;
    if (bt) bt[i] = i < m ? di * b[i] : 0.0;
  }
  for (int64_t j = 0; j < n; ++j) fht(At + j, m2, n);
  if (bt) fht(bt, m2, 1);
}

// CD++ preprocessing (Alg 3 l.2-3): At = H D A_pad D H (n2 x n2), bt = H D [b; 0],
// with A_pad = [[A, 0], [0, I]] (reading R4: the padded diagonal is 1 so A_pad stays PD where A
// is, and the padded coordinates of the solution are 0).  H D A D H is formed as two one-sided
// transforms (the result SymFHT, Alg 2, computes with fewer operations).
void ora_rht_sym(const double* A, int64_t n, int64_t lda, const double* b, uint64_t seed, double* At,
                 double* bt) {
  const int64_t n2 = next_pow2(n);
  const double sc = 1.0 / std::sqrt((double)n2);
  std::vector<double> d((size_t)n2);
  for (int64_t i = 0; i < n2; ++i) d[(size_t)i] = rht_sign(seed, i) * sc;
  for (int64_t i = 0; i < n2; ++i)
    for (int64_t j = 0; j < n2; ++j) {
      const double a = (i < n && j < n) ? A[i * lda + j] : (i == j ? 1.0 : 0.0);
      At[i * n2 + j] = d[(size_t)i] * a * d[(size_t)j];
    }
  for (int64_t j = 0; j < n2; ++j) fht(At + j, n2, n2);   // H (D A D): mix rows
  for (int64_t i = 0; i < n2; ++i) fht(At + i * n2, n2, 1);  // (...) H: mix columns
  if (bt) {
    for (int64_t i = 0; i < n2; ++i) bt[i] = i < n ? d[(size_t)i] * b[i] : 0.0;
    fht(bt, n2, 1);
  }
}

// CD++ back-rotation (Alg 3 l.16): x = D H xt, first n of n2 entries.  Also the forward
// map of an initial iterate: xt = Q x = H D x (fwd = 1).
void ora_rht_vec(const double* v, int64_t n, int64_t n2, uint64_t seed, int32_t fwd, double* out) {
  const double sc = 1.0 / std::sqrt((double)n2);
  std::vector<double> w((size_t)n2);
  if (fwd) {
    for (int64_t i = 0; i < n2; ++i) w[(size_t)i] = i < n ? rht_sign(seed, i) * sc * v[i] : 0.0;
    fht(w.data(), n2, 1);
    for (int64_t i = 0; i < n2; ++i) out[i] = w[(size_t)i];
  } else {
    for (int64_t i = 0; i < n2; ++i) w[(size_t)i] = v[i];
    fht(w.data(), n2, 1);
    for (int64_t i = 0; i < n; ++i) out[i] = rht_sign(seed, i) * sc * w[(size_t)i];
  }
}

}  // extern "C"
