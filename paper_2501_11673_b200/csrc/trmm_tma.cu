// trmm_tma.cu -- the triangular product Q1 = X1^T A_S of the shifted CholeskyQR2 second pass
// (DESIGN reading R1: Q1 = R1^{-T} A_aug, the sqrt(lam) I part entering as
// lam X1^T X1) on DMMA, fed by TMA through a full/empty mbarrier ring with a producer warp.
//
// Q1[i][j] = sum_{k <= i} X1[k][i] A[S_k][j]   (X1 = R1^{-1} upper triangular, s x s per block).
// One CTA owns a stripe of 64 columns of one block and ALL s rows of Q1, so every gathered element
// of A_S crosses HBM once (the tile GEMM re-read the stripe once per 64-row tile: 2.5x at s = 256).
// Per stage of 16 k-rows the producer gathers A_S[k0:k0+16, stripe] (16 x `tile::gather4`) and the
// 16-column boxes of X1[k0:k0+16, :] that are not entirely below the diagonal (box ib is needed iff
// 16 ib + 15 >= k0: the triangle halves X1's bytes and DMMAs).  Consumer warp w owns the row blocks
// p and TB-1-p (32 rows each: every pair carries the same triangular work, 4 TB + 2 box-stages) and
// 16 columns (w % 4: each SM sub-partition one column quarter of every pair).  Staged rows are
// 128-byte swizzled; fragment row r takes staged position o(r) = (r&1) + 8((r>>1)&1) + 2(r>>2) (+4
// for the second fragment of a 16-box), which puts each half-warp's 64-bit loads on 32 distinct
// banks for any k; the epilogue maps o back (o(2c), o(2c)+1 stay adjacent: 16-byte stores).
// Summation order per element: k ascending in DMMA k4 groups -- the order of the tile kernel.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>

#include "kernel_common.cuh"

namespace kpp {
PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder();  // gram_tma.cu

namespace {
using namespace itk;

constexpr int TR_BN = 64;            // columns per CTA
constexpr int TR_MAXST = 8;
constexpr int TR_RING = 200 * 1024;  // ring bytes (+1 KB alignment slack)

struct TrmmArgs {
  int s, n, nstripe, batch;
  const int32_t* idx;  // S of each block, s ints per block
  double* Q;           // Q1, s x n per block (ld = n)
};

__device__ __forceinline__ void tr_mma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}
__device__ __forceinline__ void tr_tile2d(unsigned dst, const CUtensorMap* tm, int c0, int r0, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          dst),
      "l"(reinterpret_cast<unsigned long long>(tm)), "r"(c0), "r"(r0), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tr_gather4(unsigned dst, const CUtensorMap* tm, int c0, int r0, int r1, int r2, int r3,
                                           unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];\n" ::"r"(dst),
      "l"(reinterpret_cast<unsigned long long>(tm)), "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3),
      "r"(smem_u32(bar))
      : "memory");
}
// staged position of fragment row r (0..7) in its 16-box, h = which of the box's two fragments
__device__ __forceinline__ int tr_o(int r, int h) { return (r & 1) + 8 * ((r >> 1) & 1) + 2 * (r >> 2) + 4 * h; }
// byte offset of (staged row k, position o) in a 2 KB box of 16 rows x 128 B, 128-byte swizzle
__device__ __forceinline__ unsigned tr_off(int k, int o) {
  return (unsigned)k * 128u + ((((unsigned)(o >> 1)) ^ (unsigned)(k & 7)) << 4) + ((unsigned)(o & 1) << 3);
}

// One stage (16 k-rows) of a consumer warp with boxes U0..3 active and CW column boxes of the stripe.
template <int U0, int CW, int nst, int stage_bytes>
__device__ __forceinline__ void tr_stage(unsigned gk, const unsigned char* ring, unsigned long long* full,
                                         unsigned long long* empty, const int (&bx)[4], int r, int kl, unsigned boff,
                                         int lane, double (&acc)[4][2][CW][2][2]) {
  const int st = (int)(gk % (unsigned)nst);
  mbar_wait(&full[st], (gk / (unsigned)nst) & 1u, 82);
  const unsigned char* sb = ring + st * (unsigned)stage_bytes;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const unsigned kb = (unsigned)(q >> 1) * 1024u;  // rows 8..15 of a box: +1 KB, same swizzle phase
    const unsigned o0 = tr_off(4 * (q & 1) + kl, tr_o(r, 0)), o1 = tr_off(4 * (q & 1) + kl, tr_o(r, 1));
    double bf[CW][2];
#pragma unroll
    for (int c = 0; c < CW; ++c)
#pragma unroll
      for (int hj = 0; hj < 2; ++hj)
        bf[c][hj] = *reinterpret_cast<const double*>(sb + boff + (unsigned)c * 2048u + kb + (hj ? o1 : o0));
#pragma unroll
    for (int u = U0; u < 4; ++u) {
      double af[2];
#pragma unroll
      for (int h = 0; h < 2; ++h)
        af[h] = *reinterpret_cast<const double*>(sb + (unsigned)bx[u] * 2048u + kb + (h ? o1 : o0));
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int c = 0; c < CW; ++c)
#pragma unroll
          for (int hj = 0; hj < 2; ++hj) tr_mma(acc[u][h][c][hj][0], acc[u][h][c][hj][1], af[h], bf[c][hj]);
    }
  }
  __syncwarp();
  if (lane == 0) mbar_arrive(&empty[st]);  // (the MMAs consumed every fragment: registers)
}

// Load global stage gf of this CTA (tile blockIdx.x + (gf / TB16) gridDim.x, k-rows 16 (gf % TB16) ..)
// into ring slot gf % NST once every consumer has released the slot's previous stage.  One warp.
template <int TB16, int NST, int SB>
__device__ __forceinline__ void tr_fill(unsigned gf, int ntile, const TrmmArgs& g, const CUtensorMap* tmA,
                                        const CUtensorMap* tmX, unsigned sbase, unsigned long long* full,
                                        unsigned long long* empty, int lane) {
  const int tile = (int)blockIdx.x + (int)(gf / (unsigned)TB16) * (int)gridDim.x;
  if (tile >= ntile) return;
  const int kt = (int)(gf % (unsigned)TB16);
  const int b = tile / g.nstripe, c0 = (tile % g.nstripe) * TR_BN;
  const int st = (int)(gf % (unsigned)NST);
  if (gf >= (unsigned)NST) mbar_wait(&empty[st], ((gf / (unsigned)NST) - 1u) & 1u, 81);
  if (lane == 0) mbar_expect_tx(&full[st], 16u * 512u + (unsigned)(TB16 - kt) * 2048u);
  __syncwarp();
  const unsigned dst = sbase + st * SB;
  if (lane < 16) {  // A_S rows k0 + 4 gq .. +3, column box cb of the stripe
    const int32_t* S = g.idx + (long long)b * g.s;
    const int cb = lane >> 2, gq = lane & 3;
    const int k = 16 * kt + 4 * gq;
    tr_gather4(dst + (unsigned)(TB16 + cb) * 2048u + (unsigned)gq * 512u, tmA, c0 + 16 * cb, S[k], S[k + 1], S[k + 2],
               S[k + 3], &full[st]);
  } else {  // X1 boxes kt .. TB16-1 (rows 16 kt .. +15 of block b, columns 16 ib .. +15)
    for (int ib = kt + lane - 16; ib < TB16; ib += 16)
      tr_tile2d(dst + (unsigned)ib * 2048u, tmX, 16 * ib, b * g.s + 16 * kt, &full[st]);
  }
}

// Persistent over tiles (block, stripe); the producer warp (the last one) runs ahead across tiles, so
// the next stripe's stages land while the consumers write the epilogue.  CW column boxes (16 columns
// each) per consumer warp: CW = 1 -> TB16 consumer warps of 16 accumulator fragments, CW = 2 -> TB16 / 2
// warps of 32 (4 + 8 fragment loads per 32 DMMAs instead of 2 + 8 per 16).  A sub-partition's 16 K
// registers hold ceil(warps / 4) warps: CW = 1 at s = 256 (17 warps) is capped at 96 registers per
// thread and spills ~100 bytes; CW = 2 (9 warps) gets 168 and spills too (it wants ~200).  Measured:
// CW = 1 is faster (the launch default).
template <int TB16, int CW>
__global__ void __launch_bounds__((TB16 * (4 / CW) / 4 + 1) * 32, 1)
trmm_tma_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmX,
                const __grid_constant__ TrmmArgs g) {
  extern __shared__ unsigned char tr_sm[];
  __shared__ unsigned long long full[TR_MAXST], empty[TR_MAXST];
  const int ntile = g.batch * g.nstripe;  // tile = (block, stripe), stripes fastest
  // stages of 16 k-rows (s = 16 TB16); the ring holds nst stages of SB bytes
  constexpr int nk = TB16, NQ = 4 / CW, NWC = (TB16 / 4) * NQ, SB = (TB16 + 4) * 2048;
  constexpr int nst = TR_RING / SB < TR_MAXST ? TR_RING / SB : TR_MAXST;
  const unsigned sm0 = smem_u32(tr_sm), sbase = (sm0 + 1023u) & ~1023u;
  const unsigned char* ring = tr_sm + (sbase - sm0);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < nst; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], (unsigned)NWC);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (warp == NWC) {  // ------------------------------------------------------- producer warp
    const unsigned total = (unsigned)((ntile - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x) * nk;
    for (unsigned gf = 0; gf < total; ++gf) tr_fill<TB16, nst, SB>(gf, ntile, g, &tmA, &tmX, sbase, full, empty, lane);
    return;
  }
  // ---------------------------------------------------------------------------- consumer warps
  // warp -> (row-block pair p, column group cq of CW boxes); warp w runs on sub-partition w % 4, so
  // each sub-partition holds whole pairs' worth of equal work
  const int p = warp / NQ, cq = warp % NQ;
  const int TB = TB16 >> 1;  // row blocks of 32
  int bx[4];
  bx[0] = 2 * p;
  bx[1] = 2 * p + 1;
  bx[2] = 2 * (TB - 1 - p);
  bx[3] = 2 * (TB - 1 - p) + 1;
  const int r = lane >> 2, kl = lane & 3;
  const unsigned boff = (unsigned)(TB16 + CW * cq) * 2048u;  // this warp's columns of the A_S stage
  // The active boxes only shrink from the front (bx[0] < bx[1] <= bx[2] < bx[3]): stages run in four
  // segments with boxes U0..3 active, so the stage body has no per-box branches.
  const int e0 = bx[0] + 1, e1 = bx[1] + 1, e2 = bx[2] + 1, e3 = bx[3] + 1;
  const bool v2 = (g.n & 1) == 0;
  unsigned gk = 0;
  for (int tile = blockIdx.x; tile < ntile; tile += gridDim.x) {
    const int b = tile / g.nstripe, c0 = (tile % g.nstripe) * TR_BN;
    double acc[4][2][CW][2][2];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int c = 0; c < CW; ++c)
#pragma unroll
          for (int hj = 0; hj < 2; ++hj) acc[u][h][c][hj][0] = acc[u][h][c][hj][1] = 0.0;
    int kt = 0;
    for (; kt < e0; ++kt, ++gk) tr_stage<0, CW, nst, SB>(gk, ring, full, empty, bx, r, kl, boff, lane, acc);
    for (; kt < e1; ++kt, ++gk) tr_stage<1, CW, nst, SB>(gk, ring, full, empty, bx, r, kl, boff, lane, acc);
    for (; kt < e2; ++kt, ++gk) tr_stage<2, CW, nst, SB>(gk, ring, full, empty, bx, r, kl, boff, lane, acc);
    for (; kt < e3; ++kt, ++gk) tr_stage<3, CW, nst, SB>(gk, ring, full, empty, bx, r, kl, boff, lane, acc);
    for (; kt < nk; ++kt, ++gk) {  // (no box of this warp left: release the stage)
      const int st = (int)(gk % (unsigned)nst);
      mbar_wait(&full[st], (gk / (unsigned)nst) & 1u, 82);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
    }
    // epilogue: lane holds rows 16 bx + o(r, h), columns c0 + 16 (CW cq + c) + o(2 kl, hj) and the next
    double* Qb = g.Q + (long long)b * g.s * g.n;
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int i = 16 * bx[u] + tr_o(r, h);
        double* qrow = Qb + (long long)i * g.n;
#pragma unroll
        for (int c = 0; c < CW; ++c)
#pragma unroll
          for (int hj = 0; hj < 2; ++hj) {
            const int j = c0 + 16 * (CW * cq + c) + tr_o(2 * kl, hj);
            if (v2 && j + 1 < g.n) {
              __stcs(reinterpret_cast<double2*>(qrow + j), make_double2(acc[u][h][c][hj][0], acc[u][h][c][hj][1]));
            } else {
              if (j < g.n) qrow[j] = acc[u][h][c][hj][0];
              if (j + 1 < g.n) qrow[j + 1] = acc[u][h][c][hj][1];
            }
          }
      }
  }
}

}  // namespace

// Q (s x n per block, ld n, batch stride s n) = X1^T A[S, :] with X1 (s x s per block, contiguous
// batch) upper triangular.  Served when s is a multiple of 64 (<= 256), A's rows are 16-byte
// aligned and the tensor maps encode; returns false otherwise (the caller runs the tile GEMM).
bool launch_trmm_tma(cudaStream_t st, int batch, int s, long long n, const double* A, long long lda, long long m,
                     const int32_t* S, const double* X1, double* Q) {
  static const bool off = getenv("KPP_TRMM_TMA") && atoi(getenv("KPP_TRMM_TMA")) == 0;
  if (off || batch <= 0 || s <= 0 || s % 64 || s > 256 || n <= 0 || n > 0x7fffffffLL || m > 0x7fffffffLL) return false;
  if ((reinterpret_cast<uintptr_t>(A) & 15) || (lda & 1) || (reinterpret_cast<uintptr_t>(X1) & 15)) return false;
  if ((long long)batch * s > 0x7fffffffLL) return false;
  PFN_cuTensorMapEncodeTiled_v12000 encode = tmap_encoder();
  if (!encode) return false;
  CUtensorMap tmA, tmX;
  {
    cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)m};
    cuuint64_t strides[1] = {(cuuint64_t)lda * sizeof(double)};
    cuuint32_t box[2] = {16u, 1u};
    cuuint32_t estr[2] = {1u, 1u};
    if (encode(&tmA, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)A, dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return false;
  }
  {
    cuuint64_t dims[2] = {(cuuint64_t)s, (cuuint64_t)batch * s};
    cuuint64_t strides[1] = {(cuuint64_t)s * sizeof(double)};
    cuuint32_t box[2] = {16u, 16u};
    cuuint32_t estr[2] = {1u, 1u};
    if (encode(&tmX, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)X1, dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return false;
  }
  TrmmArgs g;
  g.s = s;
  g.n = (int)n;
  g.nstripe = (int)((n + TR_BN - 1) / TR_BN);
  g.idx = S;
  g.Q = Q;
  const int TB16 = s / 16;
  const size_t sb = (size_t)(TB16 + 4) * 2048;
  const size_t smem = std::min<size_t>(TR_MAXST, TR_RING / sb) * sb + 1024;
  static bool attr = false;
  if (!attr) {
#define TR_ATTR(T, C) cudaFuncSetAttribute(trmm_tma_kernel<T, C>, cudaFuncAttributeMaxDynamicSharedMemorySize, TR_RING + 1024);
    TR_ATTR(4, 1) TR_ATTR(8, 1) TR_ATTR(12, 1) TR_ATTR(16, 1) TR_ATTR(4, 2) TR_ATTR(8, 2) TR_ATTR(12, 2) TR_ATTR(16, 2)
#undef TR_ATTR
    attr = true;
  }
  const long long ntile = (long long)batch * g.nstripe;
  if (ntile > 0x7fffffffLL) return false;
  g.batch = batch;
  // persistent: one CTA per SM (206 KB of ring), tiles strided over the grid
  static int nsm = 0;
  if (!nsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || nsm <= 0) nsm = 148;
  }
  static const bool persist = !(getenv("KPP_TRMM_PERSIST") && atoi(getenv("KPP_TRMM_PERSIST")) == 0);
  const int grid = (int)(persist ? std::min<long long>(ntile, nsm) : ntile);  // (0: one tile per CTA, A/B)
  count_launches(1);
  // column boxes per consumer warp (KPP_TRMM_CW=2: two, A/B).  Measured at s = 256 (Phase 1 ms per
  // bench step, CW 1 / 2): c4 389.4 / 395.6, c3 29.37 / 29.76 -- the 17-warp layout wins despite its
  // spills (profiles/r02/trmm/)
  static const int CW = getenv("KPP_TRMM_CW") && atoi(getenv("KPP_TRMM_CW")) == 2 ? 2 : 1;
  const int nt = (TB16 * (4 / CW) / 4 + 1) * 32;
#define TR_LAUNCH(T, C) \
  if (TB16 == T && CW == C) trmm_tma_kernel<T, C><<<grid, nt, smem, st>>>(tmA, tmX, g);
  TR_LAUNCH(4, 1) TR_LAUNCH(8, 1) TR_LAUNCH(12, 1) TR_LAUNCH(16, 1) TR_LAUNCH(4, 2) TR_LAUNCH(8, 2) TR_LAUNCH(12, 2)
  TR_LAUNCH(16, 2)
#undef TR_LAUNCH
  return true;
}

}  // namespace kpp
