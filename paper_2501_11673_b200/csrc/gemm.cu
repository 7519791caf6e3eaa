// gemm.cu -- batched fp64 GEMM on the FP64 tensor cores for Phase 1.
//
// The Phase-1 Gram A_S A_S^T and the CholeskyQR2 products are
// dense contractions, so they run on DMMA: `mma.sync.aligned.m8n8k4.row.col.f64`
// (sm_100a has no tcgen05 kind for f64; ptxas lowers this to DMMA.8x8x4).
// Tile: 64 x 64 output per CTA, K step 16, 8 warps (2 x 4), each warp 32 x 16 = 4 x 2
// mma tiles, double-buffered shared-memory stages.  Split-K across gridDim.z; partial
// products are reduced in a fixed order by splitk_reduce (deterministic, no atomics).
#include <cstdint>
#include <cstdlib>

#include "kpp_internal.h"

namespace kpp {
namespace {

constexpr int BM = 64, BN = 64, BK = 16;
constexpr int PADS = 4;            // row stride 68 doubles: conflict-free fragment loads
constexpr int LDS = BM + PADS;
constexpr int THREADS = 256;

__device__ __forceinline__ void mma_f64(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// Load a 64 (outer) x 16 (k) logical tile of an operand into smem laid out [k][outer].
// kcontig: memory rows are indexed by `outer` and k runs along the row (contiguous);
// otherwise memory rows are indexed by k and `outer` runs along the row.
template <bool KCONTIG>
__device__ __forceinline__ void load_tile(double (*sm)[LDS], const double* base, long long ld,
                                          const int32_t* idx, int outer0, int outer_lim, int k0,
                                          int k_lim) {
  const int t = threadIdx.x;
  if (KCONTIG) {
    // 64 memory rows x 16 contiguous k: thread -> (row t/4, 4 consecutive k)
    const int o = t >> 2, kq = (t & 3) * 4;
    const int go = outer0 + o;
    const double* rowp = nullptr;
    if (go < outer_lim) rowp = base + (long long)(idx ? idx[go] : go) * ld;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int gk = k0 + kq + q;
      sm[kq + q][o] = (rowp && gk < k_lim) ? __ldg(rowp + gk) : 0.0;
    }
  } else {
    // 16 memory rows (k) x 64 contiguous outer: thread -> (k t/16, 4 consecutive outer)
    const int kk = t >> 4, oq = (t & 15) * 4;
    const int gk = k0 + kk;
    const double* rowp = nullptr;
    if (gk < k_lim) rowp = base + (long long)(idx ? idx[gk] : gk) * ld;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int go = outer0 + oq + q;
      sm[kk][oq + q] = (rowp && go < outer_lim) ? __ldg(rowp + go) : 0.0;
    }
  }
}

template <bool AT, bool BT>
__global__ void __launch_bounds__(THREADS) dgemm_kernel(int M, int N, int K, int Z, int kchunk,
                                                        Operand a, Operand b, double* C,
                                                        long long ldc, long long c_bstride,
                                                        int upper_only, double alpha, int beta1) {
  const int tn = blockIdx.x, tm = blockIdx.y;
  if (upper_only && tm > tn) return;
  const int bz = blockIdx.z;
  const int batch = bz / Z, z = bz % Z;
  const int kbeg = z * kchunk;
  const int kend = min(K, kbeg + kchunk);
  __shared__ __align__(16) double As[2][BK][LDS];
  __shared__ __align__(16) double Bs[2][BK][LDS];

  const double* abase = a.ptr + (long long)batch * a.bstride;
  const double* bbase = b.ptr + (long long)batch * b.bstride;
  const int32_t* aidx = a.idx ? a.idx + (long long)batch * a.idx_bstride : nullptr;
  const int32_t* bidx = b.idx ? b.idx + (long long)batch * b.idx_bstride : nullptr;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wm = warp >> 2, wn = warp & 3;
  const int fr = lane >> 2, fc = lane & 3;
  double acc[4][2][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  // logical A(i,k): !AT -> memory row i (k contiguous); AT -> memory row k
  // logical B(k,j): !BT -> memory row k (j contiguous); BT -> memory row j (k contiguous)
  int buf = 0;
  if (kbeg < kend) {
    load_tile<!AT>(As[0], abase, a.ld, aidx, tm * BM, M, kbeg, kend);
    load_tile<BT>(Bs[0], bbase, b.ld, bidx, tn * BN, N, kbeg, kend);
  }
  __syncthreads();
  for (int k0 = kbeg; k0 < kend; k0 += BK) {
    if (k0 + BK < kend) {
      load_tile<!AT>(As[buf ^ 1], abase, a.ld, aidx, tm * BM, M, k0 + BK, kend);
      load_tile<BT>(Bs[buf ^ 1], bbase, b.ld, bidx, tn * BN, N, k0 + BK, kend);
    }
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[4], bf[2];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = As[buf][kk + fc][wm * 32 + i * 8 + fr];
#pragma unroll
      for (int j = 0; j < 2; ++j) bf[j] = Bs[buf][kk + fc][wn * 16 + j * 8 + fr];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) mma_f64(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
    __syncthreads();
    buf ^= 1;
  }
  double* Cb = C + (long long)bz * c_bstride;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int gi = tm * BM + wm * 32 + i * 8 + fr;
    if (gi >= M) continue;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int gj = tn * BN + wn * 16 + j * 8 + fc * 2;
      double* cp = Cb + (long long)gi * ldc + gj;
      if (gj < N) cp[0] = beta1 ? cp[0] + alpha * acc[i][j][0] : alpha * acc[i][j][0];
      if (gj + 1 < N) cp[1] = beta1 ? cp[1] + alpha * acc[i][j][1] : alpha * acc[i][j][1];
    }
  }
}

// ------------------------------------------------------------------ pipelined DMMA GEMM
// 128 x 64 output tile, K step 16, 3-stage cp.async (16-byte, zero-filling) pipeline, 8 warps of
// 32 x 32 (4 x 4 m8n8k4 DMMA tiles: 8 fragment loads per 16 MMAs).  Each operand keeps its memory
// orientation in shared memory ([outer][k] when k is contiguous in memory, [k][outer] otherwise),
// padded so that the fragment loads of a half-warp hit distinct banks.  Requires 16-byte aligned
// rows (even ld and batch strides, aligned base pointers); launch_dgemm falls back otherwise.
// The M tile is a template parameter BM (128: 8 warps as 4 x 2; 64: 4 warps as 2 x 2, used for the
// upper-only Gram products, whose diagonal-crossing 128 x 64 tiles leave up to 5 of 8 warps idle).
// K step and pipeline depth: measured alternatives (K 32 / 3 stages, K 16 / 4, K 32 / 2) all lose
// occupancy and were slower or equal; overridable for such experiments
#ifndef KPP_B2K
#define KPP_B2K 16
#endif
#ifndef KPP_B2S
#define KPP_B2S 3
#endif
constexpr int B2M = 128, B2N = 64, B2K = KPP_B2K, B2S = KPP_B2S, B2T = 256;
constexpr int KC_LD = B2K + 4;      // [outer][k] row stride (doubles)
constexpr int BN_LD = B2N + 4;      // [k][outer] row stride of B
__host__ __device__ constexpr int am_ld(int bm) { return bm + 4; }  // [k][outer] row stride of A
__host__ __device__ constexpr int a_stage(int bm) { return (bm * KC_LD > B2K * am_ld(bm)) ? bm * KC_LD : B2K * am_ld(bm); }
constexpr int B_STAGE = (B2N * KC_LD > B2K * BN_LD) ? B2N * KC_LD : B2K * BN_LD;
constexpr size_t b2_smem(int bm) { return (size_t)B2S * (a_stage(bm) + B_STAGE) * sizeof(double); }
constexpr int KIDX_MAX = 1024;      // K-gathered operand: staged gather list (s <= 1024)

__device__ __forceinline__ void cp_async16z(double* dst, const double* src, int bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"((unsigned)__cvta_generic_to_shared(dst)),
               "l"(src), "r"(bytes)
               : "memory");
}

// Stage one OUTER x 16 operand tile.  KC: memory rows are `outer` (k contiguous) -> sm[outer][k];
// otherwise memory rows are k (outer contiguous) -> sm[k][outer].
template <bool KC, int OUTER, int LDO, int NTT = B2T>
__device__ __forceinline__ void stage_tile(double* sm, const double* base, long long ld, const int32_t* idx,
                                           int outer0, int outer_lim, int k0, int k_lim) {
  constexpr int CH = KC ? OUTER * (B2K / 2) : B2K * (OUTER / 2);  // 16-byte chunks
#pragma unroll
  for (int c = threadIdx.x; c < CH; c += NTT) {
    if (KC) {
      const int o = c / (B2K / 2), kc = (c % (B2K / 2)) * 2;
      const int go = outer0 + o, gk = k0 + kc;
      int valid = (go < outer_lim) ? min(2, max(0, k_lim - gk)) : 0;
      const double* src = valid ? base + (long long)(idx ? idx[go] : go) * ld + gk : base;
      cp_async16z(sm + o * KC_LD + kc, src, valid * 8);
    } else {
      const int kk = c / (OUTER / 2), oc = (c % (OUTER / 2)) * 2;
      const int gk = k0 + kk, go = outer0 + oc;
      int valid = (gk < k_lim) ? min(2, max(0, outer_lim - go)) : 0;
      const double* src = valid ? base + (long long)(idx ? idx[gk] : gk) * ld + go : base;
      cp_async16z(sm + kk * LDO + oc, src, valid * 8);
    }
  }
}

// KC tiles (k contiguous in memory): the memory row of each of the thread's chunks is fixed across
// the K loop, so it is resolved once (row gather included) into NI registers; -1 = out of range.
template <int OUTER, int NTT = B2T>
struct KcRows {
  static constexpr int NI = OUTER * (B2K / 2) / NTT;
  int r[NI];
  __device__ __forceinline__ void init(const int32_t* idx, int outer0, int outer_lim) {
#pragma unroll
    for (int i = 0; i < NI; ++i) {
      const int go = outer0 + (threadIdx.x + NTT * i) / (B2K / 2);
      r[i] = go < outer_lim ? (idx ? idx[go] : go) : -1;
    }
  }
};
template <int OUTER, int NTT = B2T>
__device__ __forceinline__ void stage_tile_kc(double* sm, const double* base, long long ld,
                                              const KcRows<OUTER, NTT>& rows, int k0, int k_lim) {
#pragma unroll
  for (int i = 0; i < KcRows<OUTER, NTT>::NI; ++i) {
    const int c = threadIdx.x + NTT * i;
    const int o = c / (B2K / 2), kc = (c % (B2K / 2)) * 2;
    const int gk = k0 + kc;
    const int valid = rows.r[i] >= 0 ? min(2, max(0, k_lim - gk)) : 0;
    const double* src = valid ? base + (long long)rows.r[i] * ld + gk : base;
    cp_async16z(sm + o * KC_LD + kc, src, valid * 8);
  }
}

// ATRI: 0 general A; 1 logical A lower triangular (A(i,k) = 0 for k > i); 2 upper (A(i,k) = 0 for
// k < i) -- the K range of each row tile / warp is clipped (the stored zeros are skipped, not
// assumed).  Epilogue: C = alpha * A B (+ C when beta1).
template <bool AT, bool BT, int ATRI, int BM = B2M>
__global__ void __launch_bounds__(2 * BM, BM == 128 ? 2 : 3) dgemm2_kernel(int M, int N, int K, int Z, int kchunk,
                                                                           Operand a, Operand b, double* C,
                                                                           long long ldc, long long c_bstride,
                                                                           int upper_only, double alpha, int beta1) {
  constexpr int NTT = 2 * BM, A_ST = a_stage(BM), AMLD = am_ld(BM);
  constexpr bool ALOWER = ATRI == 1;
  extern __shared__ __align__(16) double g2sm[];
  const int tn = blockIdx.x, tm = blockIdx.y;
  if (upper_only && tm * BM >= (tn + 1) * B2N) return;  // tile entirely below the diagonal
  const int bz = blockIdx.z;
  const int batch = bz / Z, z = bz % Z;
  const int kbeg = z * kchunk;
  int kbeg_t = kbeg;
  int kend = min(K, kbeg + kchunk);
  if (ALOWER) kend = min(kend, (tm + 1) * BM);  // A(i,k) = 0 for k > i
  if (ATRI == 2) kbeg_t = max(kbeg, (tm * BM) / B2K * B2K);  // A(i,k) = 0 for k < i
  double* As = g2sm;
  double* Bs = g2sm + B2S * A_ST;
  const double* abase = a.ptr + (long long)batch * a.bstride;
  const double* bbase = b.ptr + (long long)batch * b.bstride;
  const int32_t* aidx = a.idx ? a.idx + (long long)batch * a.idx_bstride : nullptr;
  const int32_t* bidx = b.idx ? b.idx + (long long)batch * b.idx_bstride : nullptr;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wm = warp >> 1, wn = warp & 1;
  const int fr = lane >> 2, fc = lane & 3;
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  const int nk = kend > kbeg_t ? (kend - kbeg_t + B2K - 1) / B2K : 0;
  const int wrow0 = tm * BM + wm * 32, wcol0 = tn * B2N + wn * 32;
  const bool wskip = upper_only && wrow0 >= wcol0 + 32;
  // a warp tile on the diagonal (upper only): its 8 x 8 fragments strictly below the diagonal
  // (6 of 16) are not computed either
  const bool wdiag = upper_only == 2 && wrow0 == wcol0;  // 2: fragment skipping on
  const int wrow_end = wrow0 + 32;
  // A logical (i,k): !AT -> memory row i (k contiguous); B logical (k,j): BT -> memory row j
  KcRows<BM, NTT> arows;
  KcRows<B2N, NTT> brows;
  if (!AT) arows.init(aidx, tm * BM, M);
  if (BT) brows.init(bidx, tn * B2N, N);
  // operands whose memory rows run along K with a row gather: the CTA's K range of the gather list
  // is staged in shared memory once (the per-stage address then needs no global load)
  __shared__ int32_t kidx_sh[KIDX_MAX];
  const int32_t* kidx_a = nullptr;
  const int32_t* kidx_b = nullptr;
  {
    const int32_t* g = (AT && aidx) ? aidx : (!BT && bidx) ? bidx : nullptr;
    if (g && kend - kbeg_t <= KIDX_MAX && !(AT && aidx && !BT && bidx)) {
      for (int i = threadIdx.x; i < kend - kbeg_t; i += NTT) kidx_sh[i] = g[kbeg_t + i];
      __syncthreads();
      if (AT && aidx) kidx_a = kidx_sh - kbeg_t;
      else kidx_b = kidx_sh - kbeg_t;
    }
  }
  // (separate calls for the staged and the global gather list: each pointer keeps its address space,
  // so the staged list is read with shared-memory loads)
  auto stage = [&](int slot, int k0) {
    if (!AT) stage_tile_kc<BM, NTT>(As + slot * A_ST, abase, a.ld, arows, k0, kend);
    else if (kidx_a) stage_tile<false, BM, AMLD, NTT>(As + slot * A_ST, abase, a.ld, kidx_sh - kbeg_t, tm * BM, M, k0, kend);
    else stage_tile<false, BM, AMLD, NTT>(As + slot * A_ST, abase, a.ld, aidx, tm * BM, M, k0, kend);
    if (BT) stage_tile_kc<B2N, NTT>(Bs + slot * B_STAGE, bbase, b.ld, brows, k0, kend);
    else if (kidx_b) stage_tile<false, B2N, BN_LD, NTT>(Bs + slot * B_STAGE, bbase, b.ld, kidx_sh - kbeg_t, tn * B2N, N, k0, kend);
    else stage_tile<false, B2N, BN_LD, NTT>(Bs + slot * B_STAGE, bbase, b.ld, bidx, tn * B2N, N, k0, kend);
  };
#pragma unroll
  for (int st = 0; st < B2S - 1; ++st) {
    if (st < nk) stage(st, kbeg_t + st * B2K);
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  }
  for (int kt = 0; kt < nk; ++kt) {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(B2S - 2) : "memory");
    __syncthreads();
    {
      const int ln = kt + B2S - 1;
      if (ln < nk) stage(ln % B2S, kbeg_t + ln * B2K);
      asm volatile("cp.async.commit_group;\n" ::: "memory");
    }
    const double* Ast = As + (kt % B2S) * A_ST;
    const double* Bst = Bs + (kt % B2S) * B_STAGE;
    if (wskip) continue;  // this warp's 32 x 32 tile lies below the diagonal (Gram, upper only)
    // logical A lower triangular: k-steps past this warp's last row contribute nothing
    if (ALOWER && kbeg_t + kt * B2K >= wrow_end) continue;
    if (ATRI == 2 && kbeg_t + kt * B2K + B2K <= wrow0) continue;  // whole k-step left of this warp's rows
#pragma unroll
    for (int kk = 0; kk < B2K; kk += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int m = wm * 32 + i * 8 + fr;
        af[i] = !AT ? Ast[m * KC_LD + kk + fc] : Ast[(kk + fc) * AMLD + m];
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int nn = wn * 32 + j * 8 + fr;
        bf[j] = BT ? Bst[nn * KC_LD + kk + fc] : Bst[(kk + fc) * BN_LD + nn];
      }
      if (wdiag) {
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = i; j < 4; ++j) mma_f64(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
      } else {
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) mma_f64(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
      }
    }
  }
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  double* Cb = C + (long long)bz * c_bstride;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int gi = tm * BM + wm * 32 + i * 8 + fr;
    if (gi >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int gj = tn * B2N + wn * 32 + j * 8 + fc * 2;
      double* cp = Cb + (long long)gi * ldc + gj;
      if (gj < N) cp[0] = beta1 ? cp[0] + alpha * acc[i][j][0] : alpha * acc[i][j][0];
      if (gj + 1 < N) cp[1] = beta1 ? cp[1] + alpha * acc[i][j][1] : alpha * acc[i][j][1];
    }
  }
}

__global__ void splitk_reduce_kernel(int M, int N, int Z, const double* part, long long p_bstride,
                                     double diag_add, const double* add, double add_scale,
                                     long long add_bstride, double* out, long long o_bstride,
                                     int upper_only) {
  const int batch = blockIdx.y;
  const long long MN = (long long)M * N;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < MN;
       e += (long long)gridDim.x * blockDim.x) {
    int i = (int)(e / N), j = (int)(e % N);
    int si = i, sj = j;
    if (upper_only && i > j) { si = j; sj = i; }
    const double* p = part + (long long)batch * Z * p_bstride + (long long)si * N + sj;
    double v = 0.0;
    for (int z = 0; z < Z; ++z) v += p[(long long)z * p_bstride];
    if (i == j) v += diag_add;
    if (add) v += add_scale * add[(long long)batch * add_bstride + (long long)si * N + sj];
    out[(long long)batch * o_bstride + (long long)i * N + j] = v;
  }
}

// ---------------------------------------------------------------- balanced Gram (SYRK) kernel
// The upper triangle of G = A_S A_S^T for one block and one K chunk per CTA, on DMMA.
// The s x s output is cut into F x F fragments of 8 x 8 (F = ceil(s/8)); fragment rows are paired
// (p, F-1-p), which together hold F+1 upper fragments, so every warp gets the same work (one pair,
// or half a pair when F > 16: 17 fragments at most) -- the tile kernel's diagonal tiles left up to
// half of their warps idle at every K step.  A_S is staged once per K step (it is both operands).
constexpr int GS_SLOTS = 17;                 // fragments per warp
constexpr int GS_LD = 16 + 4;                // [row][k] stride of the staged rows (doubles)
constexpr int GS_ST = 3;                     // pipeline stages
__host__ __device__ constexpr int gs_threads(int split) { return split == 1 ? 256 : 512; }
__host__ __device__ constexpr size_t gs_smem(int split) {
  return (size_t)GS_ST * (split == 1 ? 128 : 256) * GS_LD * sizeof(double);
}

// SPLIT 1: F <= 16, one warp per fragment-row pair, one CTA per (block, chunk);
// SPLIT 2: 16 < F <= 32, two warps per pair, 8 pairs per CTA, two CTAs per (block, chunk).
template <int SPLIT>
__global__ void __launch_bounds__(gs_threads(SPLIT), SPLIT == 1 ? 2 : 1)
gram_syrk_kernel(int s, int F, int K, int Z, int kchunk, const double* base, long long ld, long long bstride,
                 const int32_t* idx, long long idx_bstride, double* part, long long ss) {
  constexpr int NT = gs_threads(SPLIT), ROWS = SPLIT == 1 ? 128 : 256;
  extern __shared__ __align__(16) double gs_sm[];
  const int npairs = (F + 1) / 2;
  const int ncta = SPLIT == 1 ? 1 : (npairs + 7) / 8;
  const int bz = blockIdx.x / ncta, h = blockIdx.x % ncta;
  const int batch = bz / Z, z = bz % Z;
  const int kbeg = z * kchunk, kend = min(K, kbeg + kchunk);
  const double* ab = base + (long long)batch * bstride;
  const int32_t* ix = idx ? idx + (long long)batch * idx_bstride : nullptr;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int fr = lane >> 2, fc = lane & 3;
  const int p = h * 8 + warp / SPLIT, half = warp % SPLIT;
  const bool active = p < npairs;
  const int r1 = p, r2 = F - 1 - p;
  const int n1 = F - r1;                          // fragments of row r1 (columns r1 .. F-1)
  const int total = active ? (r1 != r2 ? n1 + (F - r2) : n1) : 0;
  const int hsz = (total + SPLIT - 1) / SPLIT;
  const int lo = half * hsz, hi = min(total, lo + hsz);
  // the thread's staged chunks (16 bytes): row, source row of A (gathered), -1 out of range
  constexpr int CH = ROWS * 8 / NT;               // chunks per thread per stage (4)
  int srow[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    const int rr = (threadIdx.x + NT * c) >> 3;
    srow[c] = rr < s ? (ix ? ix[rr] : rr) : -1;
  }
  auto stage = [&](int slot, int k0) {
    double* dst = gs_sm + slot * ROWS * GS_LD;
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      const int e = threadIdx.x + NT * c;
      const int rr = e >> 3, kc = (e & 7) * 2;
      const int gk = k0 + kc;
      const int valid = srow[c] >= 0 ? min(2, max(0, kend - gk)) : 0;
      const double* src = valid ? ab + (long long)srow[c] * ld + gk : ab;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"((unsigned)__cvta_generic_to_shared(
                       dst + rr * GS_LD + kc)),
                   "l"(src), "r"(valid * 8)
                   : "memory");
    }
  };
  double acc[GS_SLOTS][2];
#pragma unroll
  for (int i = 0; i < GS_SLOTS; ++i) acc[i][0] = acc[i][1] = 0.0;
  const int nk = kend > kbeg ? (kend - kbeg + 15) / 16 : 0;
#pragma unroll
  for (int st = 0; st < GS_ST - 1; ++st) {
    if (st < nk) stage(st, kbeg + st * 16);
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  }
  for (int kt = 0; kt < nk; ++kt) {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(GS_ST - 2) : "memory");
    __syncthreads();
    {
      const int ln = kt + GS_ST - 1;
      if (ln < nk) stage(ln % GS_ST, kbeg + ln * 16);
      asm volatile("cp.async.commit_group;\n" ::: "memory");
    }
    if (!active) continue;
    const double* As = gs_sm + (kt % GS_ST) * ROWS * GS_LD + fr * GS_LD + fc;
#pragma unroll
    for (int kk = 0; kk < 16; kk += 4) {
      const double a1 = As[(r1 * 8) * GS_LD + kk];
      const double a2 = As[(r2 * 8) * GS_LD + kk];
#pragma unroll
      for (int i = 0; i < GS_SLOTS; ++i) {
        const int sl = lo + i;
        if (sl < hi) {
          const bool first = sl < n1;
          const int col = first ? r1 + sl : r2 + (sl - n1);
          const double bv = As[(col * 8) * GS_LD + kk];
          mma_f64(acc[i][0], acc[i][1], first ? a1 : a2, bv);
        }
      }
    }
  }
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  if (!active) return;
  double* Cb = part + (long long)bz * ss;
#pragma unroll
  for (int i = 0; i < GS_SLOTS; ++i) {
    const int sl = lo + i;
    if (sl < hi) {
      const bool first = sl < n1;
      const int row = first ? r1 : r2, col = first ? r1 + sl : r2 + (sl - n1);
      const int gi = row * 8 + fr, gj = col * 8 + fc * 2;
      if (gi < s) {
        double* cp = Cb + (long long)gi * s + gj;
        if (gj < s) cp[0] = acc[i][0];
        if (gj + 1 < s) cp[1] = acc[i][1];
      }
    }
  }
}

}  // namespace

static bool aligned16(const Operand& o) {
  return (reinterpret_cast<uintptr_t>(o.ptr) & 15) == 0 && (o.ld & 1) == 0 && (o.bstride & 1) == 0;
}

// M tile of the pipelined kernel: 64 for upper-only (Gram) products unless KPP_GEMM_BM=128
static int gram_bm() {
  static int bm = [] {
    const char* e = getenv("KPP_GEMM_BM");
    return (e && atoi(e) == 128) ? 128 : 64;
  }();
  return bm;
}

template <bool AT, bool BT, int TRI, int TBM>
static void launch2m(cudaStream_t st, int M, int N, int Zb, int Z, int K, int kchunk, const Operand& a,
                     const Operand& b, double* C, long long ldc, long long c_bstride, int upper_only, double alpha,
                     int beta1) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(dgemm2_kernel<AT, BT, TRI, TBM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)b2_smem(TBM));
    attr = true;
  }
  dim3 grid((N + B2N - 1) / B2N, (M + TBM - 1) / TBM, Zb);
  dgemm2_kernel<AT, BT, TRI, TBM><<<grid, 2 * TBM, b2_smem(TBM), st>>>(M, N, K, Z, kchunk, a, b, C, ldc, c_bstride,
                                                                       upper_only, alpha, beta1);
}

template <bool AT, bool BT, int TRI>
static void launch2(cudaStream_t st, dim3 grid, int M, int N, int K, int Z, int kchunk, const Operand& a,
                    const Operand& b, double* C, long long ldc, long long c_bstride, int upper_only, double alpha,
                    int beta1) {
  static const int fskip = [] {
    const char* e = getenv("KPP_GEMM_FSKIP");  // 0: compute diagonal warp tiles whole (A/B switch)
    return e ? atoi(e) : 1;
  }();
  if (upper_only && fskip) upper_only = 2;
  static const int tri64 = [] {
    const char* e = getenv("KPP_GEMM_TRI64");  // 64-row tiles for triangular left operands (A/B switch)
    return e ? atoi(e) : 1;
  }();
  if ((upper_only || (TRI != 0 && tri64)) && gram_bm() == 64)
    launch2m<AT, BT, TRI, 64>(st, M, N, grid.z, Z, K, kchunk, a, b, C, ldc, c_bstride, upper_only, alpha, beta1);
  else
    launch2m<AT, BT, TRI, B2M>(st, M, N, grid.z, Z, K, kchunk, a, b, C, ldc, c_bstride, upper_only, alpha, beta1);
}

template <bool AT, bool BT>
static void launch2t(int tri, cudaStream_t st, dim3 grid, int M, int N, int K, int Z, int kchunk, const Operand& a,
                     const Operand& b, double* C, long long ldc, long long c_bstride, int upper_only, double alpha,
                     int beta1) {
  if (tri == 1) launch2<AT, BT, 1>(st, grid, M, N, K, Z, kchunk, a, b, C, ldc, c_bstride, upper_only, alpha, beta1);
  else if (tri == 2) launch2<AT, BT, 2>(st, grid, M, N, K, Z, kchunk, a, b, C, ldc, c_bstride, upper_only, alpha, beta1);
  else launch2<AT, BT, 0>(st, grid, M, N, K, Z, kchunk, a, b, C, ldc, c_bstride, upper_only, alpha, beta1);
}

int launch_dgemm(cudaStream_t st, int batch, int M, int N, int K, const Operand& a, const Operand& b,
                 double* C, long long ldc, long long c_bstride, int Z, int upper_only, int a_tri, double alpha,
                 int beta1) {
  if (batch <= 0 || M <= 0 || N <= 0) return Z;
  if (Z < 1) Z = 1;
  int kchunk = (K + Z - 1) / Z;
  kchunk = ((kchunk + BK - 1) / BK) * BK;
  Z = (K + kchunk - 1) / kchunk;
  if (Z < 1) Z = 1;
  count_launches(1);
  if (aligned16(a) && aligned16(b) && !getenv("KPP_GEMM_V1")) {
    dim3 grid((N + B2N - 1) / B2N, (M + B2M - 1) / B2M, batch * Z);
    if (!a.trans && !b.trans) launch2t<false, false>(a_tri, st, grid, M, N, K, Z, kchunk, a, b, C, ldc, c_bstride, upper_only, alpha, beta1);
    else if (!a.trans && b.trans) launch2t<false, true>(a_tri, st, grid, M, N, K, Z, kchunk, a, b, C, ldc, c_bstride, upper_only, alpha, beta1);
    else if (a.trans && !b.trans) launch2t<true, false>(a_tri, st, grid, M, N, K, Z, kchunk, a, b, C, ldc, c_bstride, upper_only, alpha, beta1);
    else launch2t<true, true>(a_tri, st, grid, M, N, K, Z, kchunk, a, b, C, ldc, c_bstride, upper_only, alpha, beta1);
    return Z;
  }
  dim3 grid((N + BN - 1) / BN, (M + BM - 1) / BM, batch * Z);
  if (!a.trans && !b.trans)
    dgemm_kernel<false, false><<<grid, THREADS, 0, st>>>(M, N, K, Z, kchunk, a, b, C, ldc, c_bstride, upper_only, alpha, beta1);
  else if (!a.trans && b.trans)
    dgemm_kernel<false, true><<<grid, THREADS, 0, st>>>(M, N, K, Z, kchunk, a, b, C, ldc, c_bstride, upper_only, alpha, beta1);
  else if (a.trans && !b.trans)
    dgemm_kernel<true, false><<<grid, THREADS, 0, st>>>(M, N, K, Z, kchunk, a, b, C, ldc, c_bstride, upper_only, alpha, beta1);
  else
    dgemm_kernel<true, true><<<grid, THREADS, 0, st>>>(M, N, K, Z, kchunk, a, b, C, ldc, c_bstride, upper_only, alpha, beta1);
  return Z;
}

// Upper Gram of s rows (gathered through idx, or dense rows of a batched operand) per K chunk:
// part[(b Z + z) s^2 ...] as launch_dgemm writes it (upper triangle), Z K-chunks of 16-multiples.
// Returns Z, or 0 when the shape is not served (s > 256 or unaligned rows).
int launch_gram_syrk(cudaStream_t st, int batch, int s, int K, const double* base, long long ld, long long bstride,
                     long long nrows, const int32_t* idx, long long idx_bstride, double* part, long long ss, int Z) {
  if (int zt = launch_gram_tma(st, batch, s, K, base, ld, bstride, nrows, idx, idx_bstride, part, ss, Z)) return zt;
  static const bool off = getenv("KPP_GRAM_SYRK") && atoi(getenv("KPP_GRAM_SYRK")) == 0;
  // measured (B200, Phase 1 ms per bench step, balanced kernel vs the tile kernel): c2 (s = 128) 14.01 vs
  // 14.30; with two warps per pair for s = 256 it loses (c3 37.2 vs 32.1, c4 521 vs 441): s <= 128 only
  if (off || batch <= 0 || s > 128 || (reinterpret_cast<uintptr_t>(base) & 15) || (ld & 1) || (bstride & 1)) return 0;
  if (Z < 1) Z = 1;
  int kchunk = (K + Z - 1) / Z;
  kchunk = ((kchunk + 15) / 16) * 16;
  Z = (K + kchunk - 1) / kchunk;
  const int F = (s + 7) / 8;
  count_launches(1);
  if (F <= 16) {
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(gram_syrk_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gs_smem(1));
      attr = true;
    }
    gram_syrk_kernel<1><<<batch * Z, gs_threads(1), gs_smem(1), st>>>(s, F, K, Z, kchunk, base, ld, bstride, idx,
                                                                       idx_bstride, part, ss);
  } else {
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(gram_syrk_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gs_smem(2));
      attr = true;
    }
    const int ncta = ((F + 1) / 2 + 7) / 8;
    gram_syrk_kernel<2><<<batch * Z * ncta, gs_threads(2), gs_smem(2), st>>>(s, F, K, Z, kchunk, base, ld, bstride,
                                                                               idx, idx_bstride, part, ss);
  }
  return Z;
}

void launch_splitk_reduce(cudaStream_t st, int batch, int M, int N, int Z, const double* part,
                          long long p_bstride, double diag_add, const double* add, double add_scale,
                          long long add_bstride, double* out, long long o_bstride, int upper_only) {
  if (batch <= 0) return;
  long long MN = (long long)M * N;
  int gx = (int)((MN + 255) / 256);
  if (gx > 1024) gx = 1024;
  dim3 grid(gx, batch);
  splitk_reduce_kernel<<<grid, 256, 0, st>>>(M, N, Z, part, p_bstride, diag_add, add, add_scale,
                                             add_bstride, out, o_bstride, upper_only);
  count_launches(1);
}

}  // namespace kpp
