// kpp_internal.h -- declarations shared by the host runtime and the kernels of libkpp.
// Product code: shares nothing with oracle/.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

namespace kpp {

// Number of kernels this library has launched (process-wide; read by kpp_get_stats).
void count_launches(long long k);

// Launch of a persistent kernel whose CTAs wait on one another (LL polling, DSMEM): every CTA must
// be resident at once.  The launch carries the cooperative attribute next to the cluster size, so
// the driver rejects a grid that cannot be co-resident (MPS / green-context partitions, SMs held by
// another kernel) with an error instead of the waits spinning into the watchdog.  If the driver
// refuses the attribute combination itself, co-residency is re-checked with the occupancy API and
// the kernel is launched without it.
// (KPP_NO_COOP=1: plain cluster launch, for tools that cannot replay cooperative launches.)
template <typename P>
cudaError_t launch_coresident(cudaLaunchConfig_t cfg, cudaLaunchAttribute* attr, void (*fn)(P), const P& p) {
  static const bool no_coop = getenv("KPP_NO_COOP") != nullptr;
  if (no_coop) {
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    count_launches(1);
    return cudaLaunchKernelEx(&cfg, fn, p);
  }
  attr[1].id = cudaLaunchAttributeCooperative;
  attr[1].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  count_launches(1);
  cudaError_t e = cudaLaunchKernelEx(&cfg, fn, p);
  if (e == cudaSuccess || e == cudaErrorCooperativeLaunchTooLarge) return e;
  cudaGetLastError();
  cfg.numAttrs = 1;
  int nclu = 0;
  if (cudaOccupancyMaxActiveClusters(&nclu, (const void*)fn, &cfg) != cudaSuccess) return cudaGetLastError();
  if ((long long)nclu * attr[0].val.clusterDim.x < (long long)cfg.gridDim.x) return cudaErrorCooperativeLaunchTooLarge;
  return cudaLaunchKernelEx(&cfg, fn, p);
}
long long launches_total();

// Replicated solver state of one solve, persisted in device memory between
// iteration-kernel launches (windows).  Every CTA of the persistent kernel keeps an
// identical copy; CTA 0 writes it back at the end of a launch.
struct DevState {
  double rho;    // momentum parameter in force (Eq (momentum))
  double rhat;   // weighted ratio average (Eq (weighted))
  double E0, E1; // residual window sums (Eq (residual))
  long long ichk;    // checkpoints passed
  long long nh;      // history entries written
  long long t_done;  // iterations completed
  long long nb;      // fresh blocks created by the schedule in [0, t_sched)
  int stopped;       // 0 running, 1 tolerance met, 2 non-finite residual
  int pad;
  double rho_max;    // upper clamp of the adaptive rho (reading Q9; KPP_OPT_RHO_MAX, default 0.99)
};

// ------------------------------------------------------------------ schedule.cu
// Bernoulli / reuse decisions for t in [t0, t0+count) and the block ids; reads the
// fresh-block count before t0 from *nb_io and writes the count after the window.
void launch_schedule(cudaStream_t st, uint64_t seed, double C, int memo, long long t0, int count,
                     long long* nb_io, uint32_t* word1_ws, uint8_t* fresh_out, int32_t* bid_out);
// Index sets of fresh blocks k in [k0, k1): S_pool[k*s .. k*s+s) sorted ascending.
void launch_fresh_blocks(cudaStream_t st, uint64_t seed, long long pop, int s, long long k0,
                         long long k1, int32_t* S_pool);

// ------------------------------------------------------------------ gemm.cu
// Batched fp64 GEMM on FP64 tensor cores (mma.sync m8n8k4 -> DMMA):
//   C[b*Z + z] = sum_{k in chunk z} opA_b(i,k) * opB_b(k,j)
// Operand memory is row-major with leading dimension ld; `trans` selects the logical view
// (A: 0 -> (i,k) = mem(i,k), 1 -> (i,k) = mem(k,i); B: 0 -> (k,j) = mem(k,j),
// 1 -> (k,j) = mem(j,k)); `idx` (optional) gathers memory rows.
struct Operand {
  const double* ptr;
  long long ld;
  long long bstride;      // elements between batch entries
  const int32_t* idx;     // optional memory-row gather (nullptr: identity)
  long long idx_bstride;  // ints between batch entries of idx
  int trans;
};
// Returns the effective split count Z (K chunks are rounded to the K step).
// a_tri: 1 the logical A is lower triangular (A(i,k) = 0 for k > i), 2 upper (A(i,k) = 0 for
// k < i): the K range is clipped per row tile.  C = alpha * A B (+ C when beta1; Z must be 1).
int launch_dgemm(cudaStream_t st, int batch, int M, int N, int K, const Operand& a,
                 const Operand& b, double* C, long long ldc, long long c_bstride, int Z,
                 int upper_only, int a_tri = 0, double alpha = 1.0, int beta1 = 0);
// out[b] = sum_z part[b*Z+z] (+ diag_add on the diagonal) (+ add_scale * add[b]);
// with upper_only, element (i,j), i>j, is taken from (j,i).
// Balanced Gram kernel (upper triangle of rows x rows^T per K chunk, s <= 256); returns Z, or 0 if
// the shape is not served (then use launch_dgemm)
int launch_gram_syrk(cudaStream_t st, int batch, int s, int K, const double* base, long long ld, long long bstride,
                     long long nrows, const int32_t* idx, long long idx_bstride, double* part, long long ss, int Z);
bool gram_i8_enabled(int s);
long long ozaki_npad(long long n);
void launch_ozaki_planes(cudaStream_t st, const double* A, long long m, long long n, long long lda, int8_t* planes,
                         int* erow);
int launch_gram_i8(cudaStream_t st, int batch, int s, int K, const int8_t* planes, long long m, const int* erow,
                   const int32_t* idx, long long idx_bstride, double* part, long long ss, int Z);
int launch_gram_tma(cudaStream_t st, int batch, int s, int K, const double* base, long long ld, long long bstride,
                    long long nrows, const int32_t* idx, long long idx_bstride, double* part, long long ss, int Z);
// trmm_tma.cu: Q (s x n per block) = X1^T A[S, :], X1 upper triangular (false: shape not served)
bool launch_trmm_tma(cudaStream_t st, int batch, int s, long long n, const double* A, long long lda, long long m,
                     const int32_t* S, const double* X1, double* Q);
void launch_splitk_reduce(cudaStream_t st, int batch, int M, int N, int Z, const double* part,
                          long long p_bstride, double diag_add, const double* add,
                          double add_scale, long long add_bstride, double* out,
                          long long o_bstride, int upper_only);

// ------------------------------------------------------------------ factor.cu
// G[b] (s x s, row-major) <- A[S_b, S_b] + lam I   (CD++ principal block, Alg 3 l.8)
// Multi-GPU: only columns S_l in [col_begin, col_end) of the local slab contribute (others 0).
void launch_gather_principal(cudaStream_t st, int batch, const double* A, long long lda,
                             const int32_t* S, int s, double lam, long long col_begin,
                             long long col_end, double* G);
// G[b] += lam on the diagonal
void launch_mirror_upper(cudaStream_t st, int batch, double* M, int s);  // lower triangle := upper^T
void launch_add_diag(cudaStream_t st, int batch, double* G, int s, double lam);
// In place: G[b] -> R[b] upper with R^T R = G (lower part zeroed); X[b] = R^{-1}.
// info[b] = 0 on success, 1 + pivot index on a non-positive pivot.
// ws: workspace of chol_inv_workspace(s) bytes per matrix (nullptr: one CTA per matrix).
void launch_chol_trtri(cudaStream_t st, int batch, double* G, double* X, int s, int* info, double* ws);
size_t chol_inv_workspace(int s);
int chol_diag_wave();  // matrices the diagonal-tile kernel runs in one wave
// lam[b] = power-iteration estimate (lower bound) of lambda_max of A[b] (mode 0, symmetric) or of
// A[b] A[b]^T with A[b] upper triangular (mode 1)
// (other != nullptr: stop as soon as lam * other[b] > stop)
void launch_lmax(cudaStream_t st, int batch, const double* A, int s, int mode, int iters, double* lam,
                 const double* other = nullptr, double stop = 0.0);
// list[0..*cnt) = blocks b with lamG[b] * lamM[b] > thresh (or NaN), ascending
void launch_refine_select(cudaStream_t st, int batch, const double* lamG, const double* lamM, double thresh,
                          int* list, int* cnt);
// gather (scatter = 0: dst[i] = src[list[i]]) or scatter (dst[list[i]] = src[i]) of `bytes` per item
void launch_batch_move(cudaStream_t st, int count, const void* src, void* dst, const int* list, long long bytes,
                       int scatter);

// ------------------------------------------------------------------ iterate.cu
constexpr int KPP_MAX_PEERS = 8;
struct alignas(64) IterParams {
  CUtensorMap tmA;       // 2D tensor map of A (cols x rows, box {sw, 1}) for TMA gather4, if tma
  int tma;               // 1: resident slabs are gathered with cp.async.bulk.tensor ... gather4
  const double* A;
  long long lda, m, n;   // A is m x n_local (this rank's columns)
  int s;
  int cd;                // 1: CD++ (w = I_S^T y), 0: K++ (w = A_S^T y)
  long long col_base;    // global index of local column 0 (CD++ scatter, multi-GPU)
  const double* b;       // length m (replicated)
  double tol2bb;         // tol^2 * ||b||^2
  double bb;             // ||b||^2
  const int32_t* S_pool; // block k at S_pool + k*s
  const double* M_pool;  // block k at M_pool + k*s*s: (A_S A_S^T + lam I)^{-1} or (A_SS + lam I)^{-1}
  const int32_t* bid;    // block id of iteration t0 + i
  long long t0, t1;
  double* x;             // local iterate (n_local)
  double* mom;           // local momentum (n_local)
  double eta;
  long long zeta;
  int adaptive;          // 0: rho fixed
  int writer;            // this rank writes the history
  unsigned long long* ll; // [2][clusters][s][2] tagged cluster partials (zeroed before launch)
  unsigned long long* yll; // [2][s][2] tagged y (global-y mode; zeroed before launch)
  unsigned long long* ull; // [2][s][2] tagged u = X^T r (CD++ streaming kernel with yx = 1; zeroed before launch)
  int yx;                // CD++ streaming kernel: M_pool holds Z = X + X^T - diag(X), X = R^{-1} upper
                         // (M = X X^T never formed); y = X (X^T r) in two row passes over Z
  int ygl;               // 1: y computed once on the GPU (CTA-owned rows) and gathered from L2
  int* err;              // set if a spin-wait times out
  DevState* st;
  double* hist_res;      // [hist_cap]
  double* hist_rho;
  long long hist_cap;
  int slab;              // columns per CTA (multiple of 4)
  int resident;          // the block slab lives in shared memory (double-buffered)
  int sw;                // shared-memory row stride of the slab (doubles)
  int tpr;               // threads per row in the A_S x pass (power of two <= 32)
  int cw;                // threads per column group in the A_S^T y pass (multiple of 32)
  int m_in_smem;         // rows of M staged in shared memory: 0 no, 1 double-buffered, 2 single
  int a_single;          // one slab buffer (the register tile holds the current block)
  long long* prof;       // optional [16] phase cycle counters (CTA 0), nullptr = off
  long long* trace;      // debug: [16][grid][8] globaltimer event stamps (iterations 64..79)
  int dbg_skip;          // debug: 1 skips the arithmetic of rows 3-5 (exchange-latency floor)
  int g2max;             // pollers per r row in the cross-cluster gather (<= 16; 0 = 16)
  int poll_ns;           // back-off between unsuccessful polling rounds of the gather (ns; 0 = none)
  // column-sharded exchange of the CD++ streaming kernel: ranks rank .. rank+vranks-1
  // run in this launch (vranks > 1: emulated on one GPU, see XParams::vranks), rank v's CTAs own the
  // local columns [vcol[v], vcol[v+1]); per iteration each rank publishes its partial of the
  // s-vector into every rank's receive buffer ([2][nranks][s] LL words, tags t+1 with the global t)
  int rank, nranks, vranks;
  long long vcol[KPP_MAX_PEERS + 1];
  unsigned long long* peer_recv[KPP_MAX_PEERS];
  long long ll_vstride;  // words between the ranks' grid-exchange regions (ll and yll), 0 if one rank
};
// Persistent Phase-2 kernel: grid = C * clusters CTAs, cluster size C.
cudaError_t launch_iterate(cudaStream_t st, const IterParams& p, int grid, int C, size_t smem);
int iterate_block_threads();
size_t iterate_smem_bytes(const IterParams& p, int C);
int iterate_max_clusters(const IterParams& p, int C, size_t smem);  // co-resident clusters of size C
bool iterate_register_tile(const IterParams& p);  // the resident passes run from a register tile

// ------------------------------------------------------------------ cdpp_stream.cu
// CD++ streaming kernel with the re-associated residual
size_t cdpp_stream_smem_bytes(const IterParams& p, int C);
cudaError_t launch_cdpp_stream(cudaStream_t st, const IterParams& p, int grid, int C, size_t smem);
int cdpp_stream_max_clusters(const IterParams& p, int C, size_t smem);

// ------------------------------------------------------------------ rht.cu (NEXT-1 preprocessing)
// dvec[i] = d_i / sqrt(m2) for i < m (Rademacher signs of the Philox stream 3), 0 beyond
void launch_rht_signs(cudaStream_t st, uint64_t seed, long long m, long long m2, double* dvec);
// dst (m2 x n, ld ldd) = H_m2 (diag(rowscale) src [diag(colscale)]) along rows; src is m_src x n_src
// (ld lds), zero beyond (or rowscale_i colscale_i on the padded diagonal when pad_diag)
void launch_fht_rows(cudaStream_t st, const double* src, long long lds, long long m_src, long long n_src,
                     double* dst, long long ldd, long long m2, long long n, const double* rowscale,
                     const double* colscale, int pad_diag);
void launch_transpose(cudaStream_t st, const double* src, double* dst, long long n);
void launch_scale(cudaStream_t st, const double* v, const double* dvec, long long n, double* out);

// ------------------------------------------------------------------ steps.cu (engine "graph")
// Iteration cursor of the step kernels (device memory), so a captured graph is reusable.
struct DevStep {
  long long t_cur;   // next iteration
  long long t_end;   // end of the current window
  long long t_base;  // iteration of bid[0]
};
struct StepParams {
  const double* A;
  long long lda, m, n;
  int s, cd, grid, slab;
  long long col_base;
  const double* b;
  double tol2bb, bb;
  const int32_t* S_pool;
  const double* M_pool;
  const int32_t* bid;
  double* x;
  double* mom;
  double eta;
  long long zeta;
  int adaptive;
  int writer;          // this rank writes the history
  double* part;        // [grid][s]
  double* rsum;        // [s] local partial sums, allreduced in place between kernels
  double* y;           // [s]
  DevState* st;
  DevStep* sp;
  double* hist_res;
  double* hist_rho;
  long long hist_cap;
  // fused cross-GPU exchange (KPP_OPT_XCHG = 1): every rank's LL receive buffer
  // [2 (iteration parity)][nranks][s] x 2 words, mapped into this process (peer_recv[rank] = own)
  int peer, rank, nranks;
  unsigned long long* peer_recv[KPP_MAX_PEERS];
  int* err;
};
// ------------------------------------------------------------------ dist.cu (engine 2)
struct XParams {
  const double* A;
  long long lda, n;  // n: local columns (the rank's slab)
  int s, cd, grid, slab;
  long long col_base;
  const double* b;
  double tol2bb, bb;
  const int32_t* S_pool;
  const double* M_pool;
  const int32_t* bid;
  long long t0, t1, t_base;
  double* x;
  double* mom;
  double eta;
  long long zeta;
  int adaptive, writer;
  unsigned long long* ll;  // [grid][s] x 2 words (local grid exchange)
  int rank, nranks;
  unsigned long long* peer_recv[KPP_MAX_PEERS];  // every rank's [2][nranks][s] x 2 words, mapped here
  // Ranks emulated inside this launch (one GPU standing in for several, B200_PROFILING.md: "emulate
  // the ranks as one kernel over all ranks' data"): CTAs [v*grid, (v+1)*grid) act as rank rank + v
  // on the local columns [vcol[v], vcol[v+1]), with their own grid-exchange words (ll + v * words)
  // and receive buffer peer_recv[rank + v].  1 on a real rank (vcol = {0, n}).
  int vranks;
  long long vcol[KPP_MAX_PEERS + 1];
  int a_smem, sl, m_smem;
  int pf_at;  // where the next slab's prefetch is issued: 0 after (a), 1 after (b), 2 after (d)
  int* err;
  DevState* st;
  double* hist_res;
  double* hist_rho;
  long long hist_cap;
  long long* prof;
};
size_t xeng_smem_bytes(int s, int a_smem, int sl, int m_smem);
size_t xeng_ll_words(int s, int grid);
cudaError_t launch_xeng_window(cudaStream_t st, const XParams& p);

void launch_step_partial(cudaStream_t st, const StepParams& p);
void launch_step_reduce(cudaStream_t st, const StepParams& p);   // rsum = sum_g part[g] (peer: + sum over ranks)
void launch_step_solve(cudaStream_t st, const StepParams& p);    // y = M (rsum - b_S)
void launch_step_update(cudaStream_t st, const StepParams& p);   // w, momentum, x
void launch_step_window(cudaStream_t st, const StepParams& p);   // e, checkpoint, t_cur++

// ------------------------------------------------------------------ lsqr.cu (NEXT-2: Alg 6)
struct LsqrParams {
  const double* A;
  long long lda, n;
  int s, grid, slab, tmax;
  const double* b;
  const int32_t* S_pool;
  const double* X_pool;  // memoized R^{-1} of the sketch factor, s x s per block (upper)
  const int32_t* bid;    // block id of iteration t at bid[t - t_base]
  long long t0, t1, t_base;
  double lam_sqrt;
  double* x;
  double* mom;
  double eta;
  long long zeta;
  int adaptive, writer;
  double tol2bb, bb;
  double* vn;  // [n] n-parts of the LSQR vectors v, w and the iterate (slab-local)
  double* wn;
  double* xn;
  unsigned long long* ll;  // LL exchange words (lsqr_ll_words)
  int* err;
  long long* prof;         // optional: ns per phase, accumulated by CTA 0 (KPP_PHASE_PROFILE)
  int a_smem, sl;          // the A_S slab resident in shared memory (row stride sl), see lsqr_plan
  int x_smem;              // X resident in shared memory
  int v_smem;              // the slab parts of v, w and the LSQR iterate in shared memory
  DevState* st;
  double* hist_res;
  double* hist_rho;
  long long hist_cap;
};
// SRHT parameters: dsign[j] = +-1 (Philox stream 4), T = sorted tau draws of [0, n2) (stream 5)
void launch_srht_setup(cudaStream_t st, uint64_t seed, long long n2, int tau, double* dsign, int32_t* T,
                       int32_t* perm_ws);
// Y[j][b s + k] = A[S_b[k]][j] (j < n), ldy = batch * s
void launch_sketch_gather_t(cudaStream_t st, int batch, const double* A, long long lda, long long n,
                            const int32_t* S, int s, double* Y, long long ldy);
// Ah[b][q][k] = scale * Y[T_q][b s + k]
void launch_sketch_select(cudaStream_t st, int batch, const double* Y, long long ldy, const int32_t* T, int tau,
                          int s, double scale, double* Ah);
size_t lsqr_ll_words(int s, int grid);
size_t lsqr_smem_bytes(int s, int a_smem, int sl, int x_smem, int v_smem);
cudaError_t launch_lsqr_window(cudaStream_t st, const LsqrParams& p);

// sum of squares of b (single CTA, fixed order) -> *out
void launch_sumsq(cudaStream_t st, const double* b, long long m, double* out);

}  // namespace kpp
