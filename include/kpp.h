/*
 * kpp.h -- C ABI of the B200-native Kaczmarz++ / CD++ hot path
 * (Derezinski, Needell, Rebrova, Yang, arXiv 2501.11673; "the paper").
 *
 * Citations: P:n = line n of the paper's LaTeX source.
 *
 * Problem statement: solve a consistent system
 * A x = b.  Kaczmarz++ takes a general m x n matrix (min-norm solution when
 * under-determined); CD++ takes a symmetric positive semidefinite n x n matrix.
 *
 * Each kpp_solve runs, per block iteration t (Alg 5 P:1332-1360 with Proj replaced
 * by the exact factor; Alg 3 P:740-770 for CD++):
 *   1. block selection with online memoization
 *   2. on a block's first visit ("Phase 1"): its memoized factor
 *   3. r = A_S x - b_S
 *   4. w = A_S^T (A_S A_S^T + lam I)^{-1} r   [K++, Eq (bk) P:94-102]
 *      w = I_S^T (A_SS + lam I)^{-1} r        [CD++, Alg 3 l.11 P:756-757]
 *   5. m <- (1-rho)/(1+rho) (m - w);  x <- x - w + eta m   (Eq (momentum))
 *   6. residual-window estimate, stopping test E1 <= tol^2 ||b||^2, adaptive rho
 *      (Eq (residual), Eq (weighted)).
 * No RHT preprocessing (the inputs are assumed incoherent).
 *
 * Conventions
 *  - All floating point is IEEE fp64.  Matrices are row-major with leading dimension
 *    lda >= n (elements).  Index sets are int32, 0-based, sorted ascending.
 *  - Memory: A is a DEVICE pointer on the current CUDA device and is BORROWED: it is
 *    not copied, must outlive the context and must not change while it is in use.
 *    b, x0, x_out may be DEVICE or HOST pointers (detected with
 *    cudaPointerGetAttributes; host buffers are staged through the context's stream,
 *    so a call with host buffers includes the host<->device copies).
 *    res_hist and all introspection outputs are HOST pointers.
 *  - Ownership: the caller owns every buffer it passes.  The context owns its
 *    factor cache (memoized blocks), schedule, work vectors and NCCL communicator.
 *  - Errors: status codes only; nothing is thrown across the ABI and nothing exits.
 *    On KPP_EINVAL the outputs are untouched.  kpp_last_error() describes the last
 *    failure of a context.  A context is not thread-safe; distinct contexts are.
 *  - Determinism: identical (A, b, x0, s, lam, seed, options, device count) give
 *    bit-identical x and history (no floating-point atomics anywhere).
 *  - The memo cache persists across kpp_solve calls on one context: the k-th fresh
 *    block is a function of (seed, k) only, so a later solve reuses earlier factors.
 */
#ifndef KPP_H
#define KPP_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct kpp_ctx kpp_ctx; /* opaque; one per (A, s, lam, seed[, communicator]) */

typedef enum {
  KPP_OK = 0,
  KPP_EINVAL = 1,    /* invalid argument (outputs untouched) */
  KPP_ENOMEM = 2,    /* device or host allocation failed */
  KPP_ECUDA = 3,     /* CUDA runtime error (see kpp_last_error) */
  KPP_ENCCL = 4,     /* NCCL error */
  KPP_ENOTPD = 5,    /* non-positive pivot in chol(A_S A_S^T + lam I) / chol(A_SS + lam I) */
  KPP_EDIVERGED = 6, /* non-finite block residual */
  KPP_EMAXITER = 7   /* informational: max_iters reached before the tolerance; x_out written */
} kpp_status;

/* Options for kpp_set_option (value is a double; integers are passed as doubles). */
typedef enum {
  KPP_OPT_ACCEL = 1,      /* 1 (default): eta = s/(2n); 0: eta = 0, plain block Kaczmarz */
  KPP_OPT_MEMO = 2,       /* 1 (default): online memoization; 0: a fresh block every iteration */
  KPP_OPT_ETA = 3,        /* < 0 (default): s/(2n); otherwise the momentum step eta */
  KPP_OPT_RHO_FIXED = 4,  /* < 0 (default): adaptive rho; >= 0: fixed rho, never updated */
  KPP_OPT_FACTOR = 5,     /* K++ factor route (same R in exact arithmetic): 2 (default) Gram + Cholesky,
                             then a second (shifted CholeskyQR2) pass only for blocks whose power-
                             iteration estimate 4 u kappa(A_S)^2 exceeds 3e-11; 0 shifted CholeskyQR2
                             of [A_S, sqrt(lam) I] for every block; 1 literal Gram + Cholesky */
  KPP_OPT_WINDOW = 6,     /* iterations per device window (default 8192; rounded to >= 1) */
  KPP_OPT_PHASE1_MB = 7,  /* device workspace budget for a Phase-1 batch, MiB (default 4096) */
  KPP_OPT_RESIDENT = 8,   /* 1 (default): keep the block slab on chip across both passes when it
                             fits; 0: always stream A_S from HBM/L2 */
  KPP_OPT_ENGINE = 9,     /* -1 (default): automatic -- one GPU: 0; column-sharded: 2 when the peer
                             buffers are mapped, else 1.  0: persistent cluster kernel (one GPU);
                             1: replayed CUDA graph of step kernels (exchange per KPP_OPT_XCHG);
                             2: persistent kernel with the cross-GPU exchange fused in (dist.cu) */
  KPP_OPT_CLUSTER = 10,   /* 0 (default): choose the thread-block cluster size automatically;
                             1, 2, 4, 8 or 16: force it (the grid shrinks to co-resident clusters) */
  KPP_OPT_YGL = 11,       /* where the persistent kernel computes y = M r: -1 (default) automatic;
                             0: once per thread-block cluster from the CTAs' staged rows of M
                                (DSMEM all-gather of y);
                             1: once per GPU (rows of M spread over all CTAs), gathered through L2;
                             4: per cluster as the sum of the CTAs' partials M[slice,:]^T r_slice */
  KPP_OPT_PROJ = 13,      /* K++ projection (single-GPU contexts): 0 (default) the exact memoized factor,
                             "K++(Cholesky)" P:1319; 1 sketch-and-precondition LSQR, Alg 6
                             (SRHT sketch of size tau, Cholesky preconditioner memoized as R^{-1},
                             t_max LSQR steps per iteration from zero).  kpp_get_factor then returns
                             R^{-1} of the sketch factor. */
  KPP_OPT_TMAX = 14,      /* LSQR steps per iteration t_max (default 8) */
  KPP_OPT_TAU = 15,       /* sketch size tau (default 0 = 2 s); before the first solve only */
  KPP_OPT_XCHG = 16,      /* column-sharded contexts: the per-iteration exchange of the s-vector.
                             1 (default): fused into the reduce kernel -- each rank stores its tagged partial
                             into every rank's receive buffer over NVLink (CUDA IPC mappings made at setup)
                             and sums the ranks in rank order; 0: ncclAllReduce between kernels.  Falls back
                             to 0 when the buffers cannot be mapped (stats.xchg tells which runs). */
  KPP_OPT_RHO0 = 17,      /* initial momentum parameter rho_0 in [0, 1) (default 0, Alg 5 l.4 P:1340,
                             Alg 3 l.4 P:748); ignored when KPP_OPT_RHO_FIXED >= 0 */
  KPP_OPT_RHO_MAX = 18,   /* upper clamp of the adaptive rho = clamp(1 - r_hat^{1/zeta}, 0, rho_max),
                             in [0, 1) (default 0.99; the paper does not bound rho, DESIGN reading Q9) */
  KPP_OPT_VRANKS = 19,    /* one-GPU contexts, engine 2 only: emulate P column-sharded ranks (1..8, default 1)
                             inside the one launch -- rank v's CTAs own the columns [v n/P, (v+1) n/P),
                             reduce them over their own grid, publish the rank partial into every rank's
                             receive buffer and sum the P partials in rank order, exactly the protocol of
                             the multi-GPU path, with the buffers in this device's memory.
                             Test vehicle for the P > 1 exchange on a single GPU; not a performance mode */
  KPP_OPT_REASSOC = 12,   /* CD++ only.  1 (default): blocks that stream from HBM use the kernel that
                             re-associates r_{t+1} = A_{S'} (x_t + eta c m_t) - (1 + eta c) A[S', S] y_t
                             - b_{S'} (exact in real arithmetic, from Alg 3 l.11-13 P:756-759) so the
                             dense pass of t+1 overlaps the exchange of t; 0: off; 2: always */
} kpp_option;

/* ---- setup ------------------------------------------------------------------ */
/* Kaczmarz++ context (Alg 5, problem statement P:78 / P:179) for a general A (m x n):
   A DEVICE, row-major, lda >= n, borrowed; block_size = s, 1 <= s <= m; lambda >= 0 the
   Tikhonov shift of the projection (A_S A_S^T + lam I)^{-1} (Eq (bk), default 1e-8 P:850);
   seed keys the Philox-4x32-10 streams of the block schedule (reading R2).  *out receives the
   context (owned by the caller, freed by kpp_destroy).  Errors: KPP_EINVAL (null pointers, sizes,
   lambda < 0; *out untouched), KPP_ENOMEM, KPP_ECUDA.  No device work beyond allocation. */
kpp_status kpp_setup(kpp_ctx** out, const double* A, int64_t m, int64_t n, int64_t lda,
                     int32_t block_size, double lambda, uint64_t seed);
/* CD++ context (Alg 3) for a symmetric PSD A (n x n): A DEVICE, row-major, lda >= n,
   borrowed, exactly symmetric (A_SS is read from the stored rows); 1 <= block_size <= n; lambda >= 0
   shifts the principal block, (A_SS + lam I)^{-1} (Alg 3 l.8-11 P:753-757).  Same ownership and
   errors as kpp_setup. */
kpp_status cdpp_setup(kpp_ctx** out, const double* A, int64_t n, int64_t lda,
                      int32_t block_size, double lambda, uint64_t seed);

/* ---- solve ------------------------------------------------------------------ */
/* One solve: the block iterations of Alg 5 l.5-18 P:1341-1357 (Alg 3 l.5-20 P:749-766) from x0,
   with the memoized factors of the context (Phase 1 runs for every block seen for the first time).
   b: m values (n for CD++).  x0: n values or NULL (= 0).  max_iters >= 0.
   tol >= 0: stop at the first checkpoint with E1 <= tol^2 ||b||^2 (0 = run max_iters
   unless the estimate is exactly zero).  x_out: n values.  res_hist (HOST, may be
   NULL): per-checkpoint sqrt(E1/||b||^2), at most hist_cap entries; n_hist (may be
   NULL) receives the number of checkpoints; iters_out (may be NULL) receives the
   number of block iterations performed.  b / x0 / x_out: DEVICE or HOST (staged through the
   context's stream), caller-owned, sizes unchecked by the ABI (the Python binding checks them).
   Returns KPP_OK (tolerance met, Alg 5 l.15 P:1352), KPP_EMAXITER (x_out written), KPP_ENOTPD (a
   block's shifted Gram / principal block is not positive definite, reading Q13), KPP_EDIVERGED
   (non-finite block residual, reading Q13'), KPP_EINVAL (outputs untouched), KPP_ECUDA, KPP_ENCCL. */
kpp_status kpp_solve(kpp_ctx* ctx, const double* b, const double* x0, int64_t max_iters, double tol,
                     double* x_out, double* res_hist, int64_t hist_cap, int64_t* n_hist,
                     int64_t* iters_out);
/* Same entry point for CD++ contexts (kpp_solve accepts both kinds). */
kpp_status cdpp_solve(kpp_ctx* ctx, const double* b, const double* x0, int64_t max_iters, double tol,
                      double* x_out, double* res_hist, int64_t hist_cap, int64_t* n_hist,
                      int64_t* iters_out);

/* Free the context and everything it owns (factor cache, schedule, work vectors, NCCL
   communicator, peer mappings).  NULL is a no-op.  A (borrowed) is not touched. */
void kpp_destroy(kpp_ctx* ctx);
/* Static string naming a status code. */
const char* kpp_status_str(kpp_status s);
const char* kpp_last_error(const kpp_ctx* ctx); /* owned by ctx; "" if none */

/* Run the context's work on this cudaStream_t (default: the legacy default stream).  The stream is
   borrowed.  KPP_EINVAL on a null context. */
kpp_status kpp_set_stream(kpp_ctx* ctx, void* cuda_stream);
/* Set one kpp_option (each enumerator above cites its passage and range); KPP_EINVAL for an unknown
   key or an out-of-range value (the option keeps its previous value).  Takes effect at the next
   solve; changing the factor route or the projection invalidates the memoized factors (they are
   recomputed, for the same blocks, at the next solve). */
kpp_status kpp_set_option(kpp_ctx* ctx, int32_t key, double value);

/* ---- introspection (parity tests, benchmarks) ------------------------------- */
/* Schedule for t in [t0, t0+count) (Alg 5 l.6-8 P:1342-1345, Alg 3 l.6-8 P:750-754, online
   memoization P:653-665): block id (fresh blocks numbered in creation order) and fresh flag.
   Computed on the device; HOST outputs of count entries.  KPP_EINVAL for t0 < 0 or count < 0. */
kpp_status kpp_get_schedule(kpp_ctx* ctx, int64_t t0, int64_t count, int32_t* block_id,
                            uint8_t* is_fresh);
/* Index set S of memoized block `block_id` ("S ~ ([m] choose s)", P:752 / P:1344; sorted, 0-based;
   HOST, s ints).  The block must already exist (created by a solve or by kpp_get_schedule /
   kpp_prepare), else KPP_EINVAL. */
kpp_status kpp_get_block(kpp_ctx* ctx, int64_t block_id, int32_t* S_out);
/* Memoized projection operator of block `block_id` (Phase 1, P:104-109 / P:140 / P:753, DESIGN
   reading R1): M = (A_S A_S^T + lam I)^{-1} (K++) or (A_SS + lam I)^{-1} (CD++), s x s row-major,
   HOST output.  Requires the factor to exist (run kpp_prepare or a solve first), else KPP_EINVAL.
   CD++ contexts that run the streaming kernel memoize Z = X + X^T - diag(X) (X = R^{-1}, no M is
   formed on the GPU); M = X X^T is then formed on the host for this call (introspection only). */
kpp_status kpp_get_factor(kpp_ctx* ctx, int64_t block_id, double* M_out);
/* Drop every memoized block (the next solve regenerates and refactors them: a cold solve). */
kpp_status kpp_clear_cache(kpp_ctx* ctx);
/* Generate and factor (Phase 1) every fresh block needed by iterations [0, iters). */
kpp_status kpp_prepare(kpp_ctx* ctx, int64_t iters);
/* Rho history of the last solve (Eq (weighted), reading Q8/Q9): HOST, per checkpoint, the
   rho in force after it; at most cap entries written, *n receives the number available. */
kpp_status kpp_get_rho_history(kpp_ctx* ctx, double* rho_hist, int64_t cap, int64_t* n);

typedef struct {
  double phase1_ms;      /* device time in schedule + block generation + factorisation */
  double phase2_ms;      /* device time in the iteration kernel */
  double iter_kernel_ms; /* same as phase2_ms, summed over the iteration-kernel launches */
  int64_t n_blocks;      /* memoized blocks held by the context */
  int64_t n_fresh_last;  /* blocks factored during the last solve */
  int64_t iter_launches; /* iteration-kernel launches during the last solve */
  int64_t kernel_launches; /* all kernel launches during the last solve */
  int32_t grid_ctas;     /* CTAs of the persistent iteration kernel */
  int32_t resident;      /* 1 if the persistent kernel keeps the block slab on chip */
  int32_t cluster;       /* thread-block cluster size of the persistent kernel */
  int32_t m_in_smem;     /* 1 if each CTA stages its rows of M in shared memory */
  int32_t tma;           /* 1 if resident slabs are gathered by TMA (tile::gather4) */
  int32_t ygl;           /* where y = M r is computed (KPP_OPT_YGL values 0, 1, 4) */
  int32_t reassoc;       /* 1 if the CD++ re-associated streaming kernel runs (KPP_OPT_REASSOC) */
  int64_t n_refined;     /* blocks that received the second CholeskyQR pass (since reset) */
  double rht_ms;         /* device time of the randomized Hadamard preprocessing (kpp_enable_rht) */
  int32_t xchg;          /* column-sharded: 1 fused NVLink peer exchange, 0 NCCL allreduce */
  int32_t engine;        /* Phase-2 engine of the last solve: 0 persistent, 1 step graph, 2 fused exchange,
                            3 sketch + LSQR */
} kpp_stats;
/* Timing and launch-plan counters (measurement); HOST output. */
kpp_status kpp_get_stats(kpp_ctx* ctx, kpp_stats* out);
/* Reset the timing counters of kpp_get_stats. */
kpp_status kpp_reset_stats(kpp_ctx* ctx);

/* ---- column-sharded multi-GPU (one process per GPU) ------------------------- */
/* Column-sharded multi-GPU (per iteration one all-reduce of the s-vector A_S x, the
   paper's Alg 5 l.9 P:1346 split over column slabs; per fresh block one of the s x s Gram).
   128-byte NCCL unique id; rank 0 creates it, the harness broadcasts it through its own process
   group (torch.distributed), every rank passes it to *_setup_dist.  KPP_ENCCL on failure. */
kpp_status kpp_get_unique_id(uint8_t id[128]);
/* A_slab = A[:, col_begin:col_end] (m x (col_end-col_begin), row-major, lda >= width) on this rank's
   device, borrowed.  b is full and replicated; x0 / x_out are the local slab.  Collective: every rank
   calls it with the same (m, n_global, s, lambda, seed, id, nranks) and its own slab; the contiguous
   slabs must tile [0, n_global).  Errors as kpp_setup, plus KPP_ENCCL. */
kpp_status kpp_setup_dist(kpp_ctx** out, const double* A_slab, int64_t m, int64_t n_global,
                          int64_t col_begin, int64_t col_end, int64_t lda, int32_t block_size,
                          double lambda, uint64_t seed, const uint8_t id[128], int32_t rank,
                          int32_t nranks);
/* CD++ on a column slab A[:, col_begin:col_end] of the symmetric A (Alg 3); fresh principal blocks
   A_SS are assembled from the ranks' disjoint column supports by one exact sum. */
kpp_status cdpp_setup_dist(kpp_ctx** out, const double* A_slab, int64_t n, int64_t col_begin,
                           int64_t col_end, int64_t lda, int32_t block_size, double lambda,
                           uint64_t seed, const uint8_t id[128], int32_t rank, int32_t nranks);

/* ---- randomized Hadamard preprocessing ----------------- */
/* Def 1.1: Q = H D, H the Sylvester-order Hadamard matrix, D = diag(d)/sqrt(m2) with
   Rademacher d (Philox-4x32-10 stream 3 of the context's seed).  K++ (Alg 5 l.2-3):
   the context solves (Q A) x = Q b, A zero-padded to m2 = next power of 2 >= m rows (x unchanged).
   CD++ (Alg 3 l.2-3 and l.16): it solves (Q A_pad Q^T) x~ = Q b with
   A_pad = [[A, 0], [0, I]] of size n2 and returns x = (Q^T x~)[0:n]; x0 is mapped by Q.
   The transformed matrix is computed once, here, into a buffer the context owns (m2 x n or
   n2 x n2 doubles; A is no longer read); the memo cache is dropped.  Later kpp_solve calls take
   and return the caller's sizes (b: m values, x0 / x_out: n).  K++ column-sharded contexts
   transform their own column slab (Q mixes rows only; every rank uses the same D); CD++ needs the
   whole matrix (Q A Q^T mixes columns): KPP_EINVAL on a column-sharded CD++ context.  Idempotent. */
kpp_status kpp_enable_rht(kpp_ctx* ctx);
/* The transformed matrix (HOST, m2 x n or n2 x n2 row-major); requires kpp_enable_rht. */
kpp_status kpp_get_rht_matrix(kpp_ctx* ctx, double* out);

/* Library version string. */
const char* kpp_version(void);

#ifdef __cplusplus
}
#endif
#endif /* KPP_H */
