/*
 * kpp_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, sequential CPU reference of the Kaczmarz++ / CD++ hot path of
 * Derezinski et al., arXiv 2501.11673 ("the paper").  It exists so that tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg can check and time the
 * CUDA path.  The product (paper_2501_11673_b200/) never includes, links or calls
 * anything under oracle/, and this file shares no code with it.
 *
 * Citations: P:n = PAPER.md line n (LaTeX source).  Readings of silent/ambiguous
 * points are the Q-numbers of SURVEY.md section 8(c), restated in DESIGN.md.
 *
 * Arithmetic: IEEE fp64, compiled with -O2 -ffp-contract=off (no FMA contraction,
 * no reassociation).  Every dot product is a sequential left-to-right loop.
 * OpenMP (optional) only distributes independent outputs, so results do not
 * depend on the thread count.
 *
 * Parity status per function:
 *   ora_philox4x32_10   pinned: Random123 known-answer vectors + curand (GPU test)
 *   ora_fresh_block     pinned: subset uniformity (chi-square), validity
 *   ora_schedule        pinned: Bernoulli rate / expected count C(1+ln(T/C))
 *   ora_kpp_factor      pinned: R^T R = A_S A_S^T + lam I, LAPACK dpotrf, 2x2 SPEC example
 *   ora_cdpp_factor     pinned: LAPACK dpotrf, [[4,2],[2,5]] -> [[2,1],[0,2]]
 *   ora_kpp_run         pinned: exact projection (lam=0), dense-LU limit, min-norm
 *                       limit, classical RBK (accel/memo off), three-sequence
 *                       equivalence (Lemma equivalence), adaptive-rho
 *                       worked example (SPEC), A=I one-step solve.
 *   ora_cdpp_run        pinned: CD++ <-> K++ reduction z_t = Phi^T x_t,
 *                       scalar coordinate-descent step, A=I.
 *   ora_fht / ora_rht_*  pinned: H_2 and e_1 examples, H^2 = n I, dense
 *                       Sylvester H_8, isometry Q^T Q = I, spectrum of Q A Q^T, [[1,2],[2,3]]
 *                       -> [[8,-2],[-2,0]], solution invariance of the transformed system.
 *   adaptive-rho trajectory / stop iteration on the BASELINE configs:
 *                       "parity unpinned" (no closed form, no published values).
 */
#ifndef KPP_ORACLE_H
#define KPP_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORA_OK = 0, ORA_EINVAL = 1, ORA_ENOTPD = 5, ORA_EDIVERGED = 6, ORA_EMAXITER = 7 };
enum { ORA_FACTOR_HOUSEHOLDER = 0, ORA_FACTOR_GRAM = 1 };

typedef struct {
  int32_t accel;       /* 1: eta = s/(2n) (or eta_override); 0: eta = 0 (P:814-823 ablation) */
  int32_t memo;        /* 1: online block memoization; 0: fresh block every step */
  double eta_override; /* < 0: default s/(2n) */
  double rho_fixed;    /* < 0: adaptive rho; >= 0: rho fixed, never updated */
  int32_t factor;      /* ORA_FACTOR_*; K++ only (CD++ always chol(A_SS + lam I)) */
  int32_t reverse;     /* 1: every sum runs in reverse order (noise-floor experiments) */
  int32_t threads;     /* OpenMP threads over independent outputs (<=1: sequential) */
  int32_t proj;        /* K++ projection: 0 exact factor (K++(Cholesky)); 1 sketch-and-
                          precondition LSQR (Alg 6) */
  int32_t tmax;        /* LSQR iterations t_max (default 8) */
  int32_t tau;         /* sketch size tau (<= 0: 2 s) */
  double rho0;         /* initial rho (Alg 5 l.4 P:1340: 0) */
  double rho_max;      /* upper clamp of the adaptive rho (reading Q9: 0.99) */
  double* timing;      /* optional out (instrumentation, no arithmetic): [0] wall seconds of the
                          run, [1] seconds inside first-visit factorisations, [2] their count */
} ora_opts;

/* Philox-4x32-10 (Salmon et al., SC'11): out = philox(ctr, key). */
void ora_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);

/* k-th fresh block: s distinct indices of [0,pop), sorted ascending (Q6). */
void ora_fresh_block(uint64_t seed, int64_t pop, int32_t s, int64_t k, int32_t* S_out);

/* Block schedule for t in [0,T) (Q4-Q7): bid[t] = index of the block used at t
   (fresh blocks are numbered in order of creation), fresh[t] = 1 if new.
   Returns the number of fresh blocks. */
int64_t ora_schedule(uint64_t seed, double C, int32_t memo, int64_t T, int32_t* bid, uint8_t* fresh);

/* Bernoulli constant of the schedule, as printed (Q5):
   K++  C = (min(m,n)/s) ln m      CD++ C = (n/s) ln n */
double ora_kpp_C(int64_t m, int64_t n, int32_t s);
double ora_cdpp_C(int64_t n, int32_t s);

/* R (s x s, row-major, upper, positive diagonal) with R^T R = A_S A_S^T + lam I.
   mode = ORA_FACTOR_HOUSEHOLDER: Householder QR of [A_S^T; sqrt(lam) I] (Q18);
   mode = ORA_FACTOR_GRAM: literal Gram + Cholesky. */
int ora_kpp_factor(const double* A, int64_t lda, int64_t n, const int32_t* S, int32_t s,
                   double lam, int32_t mode, int32_t reverse, double* R);
/* R with R^T R = A_SS + lam I (Alg 3 l.8). */
int ora_cdpp_factor(const double* A, int64_t lda, const int32_t* S, int32_t s, double lam,
                    int32_t reverse, double* R);

/* Kaczmarz++ (Alg 5, with Proj := exact factor; no RHT, Q12).
   A: m x n row-major (lda >= n). b: m. x0: n or NULL (= 0). tol >= 0 (0: run max_iters
   unless the estimate is exactly 0). Outputs: x_out (n), hist_res/hist_rho (per
   checkpoint sqrt(E1/||b||^2) and the rho in force after it; may be NULL),
   n_hist, iters_out, nfresh_out. Returns ORA_OK (tolerance met), ORA_EMAXITER, or error. */
int ora_kpp_run(const double* A, int64_t m, int64_t n, int64_t lda, const double* b,
                const double* x0, int32_t s, double lam, uint64_t seed, int64_t max_iters,
                double tol, const ora_opts* opt, double* x_out, double* hist_res,
                double* hist_rho, int64_t hist_cap, int64_t* n_hist, int64_t* iters_out,
                int64_t* nfresh_out);

/* CD++ (Alg 3, without the SymFHT lines 2-3 and the back-rotation, Q12).
   A: n x n symmetric PSD row-major. */
int ora_cdpp_run(const double* A, int64_t n, int64_t lda, const double* b, const double* x0,
                 int32_t s, double lam, uint64_t seed, int64_t max_iters, double tol,
                 const ora_opts* opt, double* x_out, double* hist_res, double* hist_rho,
                 int64_t hist_cap, int64_t* n_hist, int64_t* iters_out, int64_t* nfresh_out);

/* One adaptive-rho checkpoint update (Eq (weighted), Q8/Q9):
   given checkpoint index i >= 1, previous r_hat, window sums E0, E1, zeta:
   writes the new r_hat and rho. */
void ora_rho_update(int64_t i, double rhat_prev, double E0, double E1, int64_t zeta,
                    double* rhat_out, double* rho_out);

/* ---- sketch-and-precondition projection (NEXT-2; Alg 6, Lemma l:inner P:491-493).
   SRHT Pi = sqrt(n2/tau) I_T H D over the column space (n padded to n2; reading R5): D from the
   sign stream 4, T = tau indices of [0, n2) by a partial Fisher-Yates on stream 5, sorted.
   A_hat = A_S Pi^T (s x tau); R = chol(A_hat A_hat^T + lam I). */
void ora_srht(uint64_t seed, int64_t n, int32_t tau, double* d_out /* n2 */, int32_t* T_out /* tau */);
int ora_sketch_factor(const double* A, int64_t lda, int64_t n, const int32_t* S, int32_t s, double lam,
                      uint64_t seed, int32_t tau, double* R);
/* w = first n entries of LSQR(R^{-T}[A_S, sqrt(lam) I], R^{-T} r, tmax) from zero (Paige-Saunders) */
void ora_lsqr_proj(const double* A, int64_t lda, int64_t n, const int32_t* S, int32_t s, double lam,
                   const double* R, const double* r, int32_t tmax, double* w);

/* ---- RHT preprocessing (Def 1.1, Alg 4 P:1230-1243,
   Alg 5 l.2-3 P:1337-1338, Alg 3 l.2-3 and l.16 P:745-746).  Sign stream: reading R3;
   padding: zero rows (K++), unit diagonal (CD++, reading R4). */
int64_t ora_next_pow2(int64_t n);
void ora_rht_signs(uint64_t seed, int64_t n, int8_t* d);
void ora_fht(double* v, int64_t n); /* in place, n a power of 2, Sylvester order */
void ora_rht_rows(const double* A, int64_t m, int64_t n, int64_t lda, const double* b, uint64_t seed,
                  double* At, double* bt);
void ora_rht_sym(const double* A, int64_t n, int64_t lda, const double* b, uint64_t seed, double* At,
                 double* bt);
void ora_rht_vec(const double* v, int64_t n, int64_t n2, uint64_t seed, int32_t fwd, double* out);

#ifdef __cplusplus
}
#endif
#endif
