// gram_tma.cu -- the Phase-1 Gram G = A_S A_S^T on DMMA,
// fed by TMA through a full/empty mbarrier ring with a dedicated producer warp.
//
// One CTA computes the upper triangle of one block's s x s Gram over one K chunk (two CTAs when
// s > 128).  The output is cut into 32 x 32 warp tiles (4 x 4 fragments of 8 x 8); a warp owns one
// tile on or above the diagonal: an off-diagonal tile is 16 DMMA per k-step of 4 for 8 fragment
// loads, a diagonal tile 10 DMMA (upper fragments) for 4 loads, since both operands are rows of
// A_S.  Tiles are assigned so that the four SM sub-partitions (warp % 4) carry about the same
// number of DMMAs.  The producer warp gathers the block's rows 16 columns at a time with
// `cp.async.bulk.tensor ... tile::gather4` (4 rows per instruction, 128-byte rows, 128-byte
// swizzle so the fragment loads are conflict-free) into a ring of stages; consumers wait on the
// stage's full barrier and release it through its empty barrier -- no CTA-wide barrier in the loop.
// Same split-K chunks and the same partial layout as launch_dgemm, so the reduction and the bits
// of M do not depend on which Gram kernel ran.
#include <cudaTypedefs.h>

#include <algorithm>
#include <vector>

#include "kernel_common.cuh"

namespace kpp {
namespace {
using namespace itk;

constexpr int GT_MAXW = 19;          // consumer warps per CTA
constexpr int GT_MAXST = 16;         // ring stages
constexpr int GT_RING = 196608;      // ring bytes

struct GramTmaArgs {
  int s, TB, K, Z, kchunk, ncta, nst;
  long long rows_per_batch;          // row offset of batch b is b * rows_per_batch (idx == nullptr)
  const int32_t* idx;
  long long idx_bstride;
  double* part;
  long long ss;
  int nw[4];                         // warps with a piece, per CTA of a (block, chunk)
  unsigned short tile[4][GT_MAXW];   // type << 8 | h << 7 | bi << 4 | bj of each warp's piece
};

__device__ __forceinline__ void gt_mma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void gt_gather4(unsigned dst, const CUtensorMap* tm, int c0, int r0, int r1, int r2,
                                           int r3, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];\n" ::"r"(dst),
      "l"(reinterpret_cast<unsigned long long>(tm)), "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3),
      "r"(smem_u32(bar))
      : "memory");
}

// Lane-row permutation inside a fragment: lane row r reads staged row sigma(r) = 2 (r & 3) + (r >> 2)
// of the fragment's 8.  A 64-bit shared load is served per half-warp (lane rows 0-3, 4-7); with the
// 128-byte swizzle (16-byte chunk ^ (row & 7)) rows {0, 2, 4, 6} and {1, 3, 5, 7} put each half-warp's
// 16 loads on 32 distinct banks, where rows 0-3 would pair up (2-way conflicts, measured 4.07
// wavefronts per LDS.64 on c4).  The same permutation applies to the Gram's rows and columns; the
// epilogue maps it back.
__device__ __forceinline__ int gt_sigma(int r) { return ((r & 3) << 1) | (r >> 2); }

enum { GT_OFF = 0, GT_DIAG = 1, GT_HALF = 2 };

// One warp's piece of the upper Gram: GT_OFF a 4 x 4-fragment tile (bi, bj), GT_DIAG the 10 upper
// fragments of diagonal tile (bi, bi), GT_HALF fragment rows 2h, 2h+1 of tile (bi, bj) (h = bit 7).
template <int TYPE, int KH>
__device__ __forceinline__ void gt_consume(const GramTmaArgs& g, int tt, int bz, int lane, int nk16, int nst,
                                           unsigned stage_bytes, const unsigned char* ring,
                                           unsigned long long* full, unsigned long long* empty) {
  constexpr int NI = TYPE == GT_HALF ? 2 : 4;
  const int bi = (tt >> 4) & 7, bj = tt & 15, h = (tt >> 7) & 1;
  const int sg = gt_sigma(lane >> 2);
  // byte offset of the lane's element (staged row sg of a fragment, k = 4q + lane%4) in a 128-byte row:
  // chunk (2q + (lane%4)/2) ^ sg = ((q ^ sg/2) << 1) | ((lane%4)/2 ^ sg%2)
  const unsigned obase = sg * 128u + ((((lane & 3) >> 1) ^ (sg & 1)) << 4) + ((lane & 1) << 3);
  const unsigned sh = (unsigned)sg >> 1;
#define GT_OFFQ(q) (obase + ((((unsigned)(q)) ^ sh) << 5))
  const unsigned ra = bi * 4096u + (TYPE == GT_HALF ? h * 2048u : 0u), rb = bj * 4096u;
  const unsigned half_bytes = stage_bytes / KH;
  double acc[NI * 4][2];
#pragma unroll
  for (int i = 0; i < NI * 4; ++i) acc[i][0] = acc[i][1] = 0.0;
  const int nk = (nk16 + KH - 1) / KH;
  for (int kt = 0; kt < nk; ++kt) {
    const int st = kt % nst;
    mbar_wait(&full[st], (kt / nst) & 1, 72);
    const int nh = KH == 1 ? 1 : min(KH, nk16 - KH * kt);
    for (int hh = 0; hh < nh; ++hh) {
      const unsigned char* sb = ring + st * stage_bytes + hh * half_bytes;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        double a[NI], b[4];
#pragma unroll
        for (int i = 0; i < NI; ++i) a[i] = *reinterpret_cast<const double*>(sb + ra + i * 1024u + GT_OFFQ(q));
        if (TYPE != GT_DIAG) {
#pragma unroll
          for (int j = 0; j < 4; ++j) b[j] = *reinterpret_cast<const double*>(sb + rb + j * 1024u + GT_OFFQ(q));
        }
#pragma unroll
        for (int i = 0; i < NI; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            if (TYPE == GT_DIAG && j < i) continue;
            gt_mma(acc[i * 4 + j][0], acc[i * 4 + j][1], a[i], TYPE == GT_DIAG ? a[j] : b[j]);
          }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
  }
#undef GT_OFFQ
  double* Cb = g.part + (long long)bz * g.ss;
  const int s = g.s;
  const int fi0 = 4 * bi + (TYPE == GT_HALF ? 2 * h : 0);
#pragma unroll
  for (int i = 0; i < NI; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (TYPE == GT_DIAG && j < i) continue;
      const int gi = (fi0 + i) * 8 + sg;
      const int gj0 = (4 * bj + j) * 8 + gt_sigma((lane & 3) * 2), gj1 = (4 * bj + j) * 8 + gt_sigma((lane & 3) * 2 + 1);
      if (gi < s) {
        double* cp = Cb + (long long)gi * s;
        if (gj0 < s) cp[gj0] = acc[i * 4 + j][0];
        if (gj1 < s) cp[gj1] = acc[i * 4 + j][1];
      }
    }
}

// NW warps: NW - 1 consumers at most, the producer is warp NW - 1.  A sub-partition's register file
// (16 K registers) holds ceil(NW / 4) warps, so NW sets the register budget: 12 -> 168, 16 -> 128,
// 20 -> 96 (enough for whole tiles only: HALF = false).
template <int NW, bool HALF, int KH>
__global__ void __launch_bounds__(NW * 32, 1)
gram_tma_kernel(const __grid_constant__ CUtensorMap tm, const __grid_constant__ GramTmaArgs g) {
  extern __shared__ unsigned char gt_sm[];
  __shared__ unsigned long long full[GT_MAXST], empty[GT_MAXST];
  const int cta = blockIdx.x % g.ncta, bz = blockIdx.x / g.ncta;
  const int batch = bz / g.Z, z = bz % g.Z;
  const int kbeg = z * g.kchunk, kend = min(g.K, kbeg + g.kchunk);
  const int nk16 = kend > kbeg ? (kend - kbeg + 15) >> 4 : 0;  // 16-column boxes of the chunk
  const int nk = (nk16 + KH - 1) / KH;                            // stages of KH boxes
  const int rows = g.TB * 32;
  const unsigned half_bytes = (unsigned)rows * 128u, stage_bytes = KH * half_bytes;
  // the ring starts on a 1024-byte boundary: the 128-byte swizzle repeats every 8 rows of 128 B
  const unsigned sm0 = smem_u32(gt_sm), sbase = (sm0 + 1023u) & ~1023u;
  const unsigned char* ring = gt_sm + (sbase - sm0);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = g.nw[cta];
  const int nst = g.nst;
  if (threadIdx.x == 0) {
    for (int i = 0; i < nst; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], (unsigned)nw);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (warp == NW - 1) {  // ------------------------------------------------ producer warp
    // gathers q = lane and lane + 32 (4 rows each); rows past s repeat row s-1 (their products land in
    // fragments past s, which are not stored)
    const int ng = rows >> 2;
    int rr[2][4];
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int r = min(4 * (lane + 32 * j) + e, g.s - 1);
        rr[j][e] = g.idx ? g.idx[(long long)batch * g.idx_bstride + r] : (int)(batch * g.rows_per_batch + r);
      }
    for (int kt = 0; kt < nk; ++kt) {
      const int st = kt % nst;
      if (kt >= nst) mbar_wait(&empty[st], ((kt / nst) - 1) & 1, 71);
      // the chunk's last stage may hold one half: the next 16 columns belong to the next chunk
      const int nh = min(KH, nk16 - KH * kt);
      if (lane == 0) mbar_expect_tx(&full[st], nh * half_bytes);
      __syncwarp();
      for (int hh = 0; hh < nh; ++hh) {
        const int c0 = kbeg + (kt * KH + hh) * 16;
        const unsigned dst = sbase + st * stage_bytes + hh * half_bytes;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int q = lane + 32 * j;
          if (q < ng) gt_gather4(dst + q * 512u, &tm, c0, rr[j][0], rr[j][1], rr[j][2], rr[j][3], &full[st]);
        }
      }
    }
    return;
  }
  if (warp >= nw) return;
  const int tt = g.tile[cta][warp];
  const int type = tt >> 8;
  if (type == GT_OFF) gt_consume<GT_OFF, KH>(g, tt, bz, lane, nk16, nst, stage_bytes, ring, full, empty);
  else if (type == GT_DIAG) gt_consume<GT_DIAG, KH>(g, tt, bz, lane, nk16, nst, stage_bytes, ring, full, empty);
  else if (HALF) gt_consume<GT_HALF, KH>(g, tt, bz, lane, nk16, nst, stage_bytes, ring, full, empty);
}

// Warp pieces of the TB x TB tile triangle for ncta CTAs.  Off-diagonal tiles weigh 16 DMMAs per
// k-step, diagonal ones 10; `nsplit` off-diagonal tiles are cut into two halves of 8, which lets the
// four sub-partitions of a CTA (warp w runs on sub-partition w % 4, so sub-partition j holds
// W/4 + (j < W%4) warps) carry equal loads: s = 128 -> each sub-partition one tile, one diagonal
// tile and one half, 34 DMMAs (whole tiles only: 36 / 36 / 32 / 32).  Returns the busiest
// sub-partition's load, or -1 when a CTA would need more than GT_MAXW warps.
int assign_pieces(int TB, int ncta, int nsplit, GramTmaArgs& g) {
  if (ncta > 4) return -1;
  struct T { int code, w; };
  std::vector<T> pcs;
  int noff = 0;
  for (int bi = 0; bi < TB; ++bi)
    for (int bj = bi; bj < TB; ++bj) {
      if (bi == bj) {
        pcs.push_back({GT_DIAG << 8 | bi << 4 | bj, 10});
      } else if (noff++ < nsplit) {
        pcs.push_back({GT_HALF << 8 | bi << 4 | bj, 8});
        pcs.push_back({GT_HALF << 8 | 1 << 7 | bi << 4 | bj, 8});
      } else {
        pcs.push_back({GT_OFF << 8 | bi << 4 | bj, 16});
      }
    }
  std::stable_sort(pcs.begin(), pcs.end(), [](const T& x, const T& y) { return x.w > y.w; });
  std::vector<std::vector<T>> per(ncta);
  std::vector<int> load(ncta, 0);
  for (const T& t : pcs) {
    int c = 0;
    for (int k = 1; k < ncta; ++k)
      if (load[k] < load[c] || (load[k] == load[c] && per[k].size() < per[c].size())) c = k;
    per[c].push_back(t);
    load[c] += t.w;
  }
  int worst = 0;
  for (int c = 0; c < ncta; ++c) {
    const int W = (int)per[c].size();
    if (W > GT_MAXW) return -1;
    g.nw[c] = W;
    int cap[4];
    for (int j = 0; j < 4; ++j) cap[j] = W / 4 + (j < W % 4);
    // pieces by weight class (16, 10, 8); choose how many of each every sub-partition takes by
    // exhaustive search (a greedy fill left 74 / 74 / 58 / 58 where 68 / 68 / 64 / 64 exists)
    std::vector<int> cls[3];
    for (const T& t : per[c]) cls[t.w == 16 ? 0 : t.w == 10 ? 1 : 2].push_back(t.code);
    const int NO = (int)cls[0].size(), ND = (int)cls[1].size(), NH = (int)cls[2].size();
    int bo[4] = {0, 0, 0, 0}, bh[4] = {0, 0, 0, 0}, bestmax = 1 << 30;
    int co[4], ch[4];
    for (co[0] = 0; co[0] <= std::min(cap[0], NO); ++co[0])
      for (ch[0] = 0; ch[0] <= std::min(cap[0] - co[0], NH); ++ch[0])
        for (co[1] = 0; co[1] <= std::min(cap[1], NO - co[0]); ++co[1])
          for (ch[1] = 0; ch[1] <= std::min(cap[1] - co[1], NH - ch[0]); ++ch[1])
            for (co[2] = 0; co[2] <= std::min(cap[2], NO - co[0] - co[1]); ++co[2])
              for (ch[2] = 0; ch[2] <= std::min(cap[2] - co[2], NH - ch[0] - ch[1]); ++ch[2]) {
                co[3] = NO - co[0] - co[1] - co[2];
                ch[3] = NH - ch[0] - ch[1] - ch[2];
                int mx = 0, nd = 0;
                bool ok = co[3] >= 0 && ch[3] >= 0 && co[3] + ch[3] <= cap[3];
                for (int j = 0; ok && j < 4; ++j) {
                  const int d = cap[j] - co[j] - ch[j];
                  nd += d;
                  mx = std::max(mx, 16 * co[j] + 10 * d + 8 * ch[j]);
                }
                if (ok && nd == ND && mx < bestmax) {
                  bestmax = mx;
                  for (int j = 0; j < 4; ++j) bo[j] = co[j], bh[j] = ch[j];
                }
              }
    if (bestmax == (1 << 30)) return -1;
    int io = 0, id = 0, ih = 0;
    for (int j = 0; j < 4; ++j)
      for (int q = 0; q < cap[j]; ++q) {
        const int code = q < bo[j] ? cls[0][io++] : q < bo[j] + bh[j] ? cls[2][ih++] : cls[1][id++];
        g.tile[c][j + 4 * q] = (unsigned short)code;
      }
    worst = std::max(worst, bestmax);
  }
  return worst;
}

// CTAs per (block, chunk) and split count with the least SM time, ncta x the busiest
// sub-partition's load, with 10 % per extra CTA: every CTA stages all rows of the block, and four CTAs
// per block at s = 256 starved the DMMA pipe (48 % busy on c4 against 83 % with two).  More than 15
// warps (96 registers) only with whole tiles.
bool plan_pieces(int TB, GramTmaArgs& g) {
  const int noff = TB * (TB - 1) / 2;
  double best = -1;
  int bestn = 0, bestk = 0, bestw = 0;
  for (int n = 1; n <= 4; ++n)
    for (int k = 0; k <= noff; ++k) {
      GramTmaArgs t = g;
      const int w = assign_pieces(TB, n, k, t);
      if (w < 0) continue;
      int nw = 0;
      for (int c = 0; c < n; ++c) nw = std::max(nw, t.nw[c]);
      if (nw > 15 && k > 0) continue;
      const double cost = (double)n * w * (1.0 + 0.1 * (n - 1));
      if (best < 0 || cost < best || (cost == best && nw < bestw)) best = cost, bestn = n, bestk = k, bestw = nw;
    }
  if (best < 0) return false;
  g.ncta = bestn;
  assign_pieces(TB, bestn, bestk, g);
  return true;
}

}  // namespace

// cuTensorMapEncodeTiled through the runtime's driver entry point (nullptr when unavailable)
PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
    cudaDriverEntryPointQueryResult qr;
    void* fn = nullptr;
    PFN_cuTensorMapEncodeTiled_v12000 e = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr) == cudaSuccess &&
        qr == cudaDriverEntryPointSuccess)
      e = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    cudaGetLastError();
    return e;
  }();
  return encode;
}

// Upper Gram per K chunk through the TMA ring (see the header comment).  `nrows` is the height of
// the row space the rows are gathered from (A's m for idx gathers; batch * bstride / ld for dense
// batched rows).  Returns Z, or 0 when the shape is not served (s <= 64 or s > 256, unaligned rows,
// no tensor-map encoder, KPP_GRAM_TMA=0).
int launch_gram_tma(cudaStream_t st, int batch, int s, int K, const double* base, long long ld, long long bstride,
                    long long nrows, const int32_t* idx, long long idx_bstride, double* part, long long ss, int Z) {
  static const bool off = getenv("KPP_GRAM_TMA") && atoi(getenv("KPP_GRAM_TMA")) == 0;
  const int TB = (s + 31) / 32;
  if (off || batch <= 0 || TB < 3 || TB > 8 || (reinterpret_cast<uintptr_t>(base) & 15) || (ld & 1)) return 0;
  if (!idx && (ld <= 0 || bstride % ld)) return 0;
  const long long height = idx ? nrows : (long long)batch * (bstride / ld);
  if (height <= 0 || height > 0x7fffffffLL) return 0;
  PFN_cuTensorMapEncodeTiled_v12000 encode = tmap_encoder();
  if (!encode) return 0;
  // the piece plan depends on TB only: computed once per TB
  static GramTmaArgs plans[9];
  static int planned[9] = {0};
  if (!planned[TB]) planned[TB] = plan_pieces(TB, plans[TB]) ? 1 : -1;
  if (planned[TB] < 0) return 0;
  GramTmaArgs g = plans[TB];
  CUtensorMap tm;
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)height};
  cuuint64_t strides[1] = {(cuuint64_t)ld * sizeof(double)};
  cuuint32_t box[2] = {16u, 1u};
  cuuint32_t estr[2] = {1u, 1u};
  if (encode(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)base, dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return 0;
  if (Z < 1) Z = 1;
  int kchunk = (K + Z - 1) / Z;
  kchunk = ((kchunk + 15) / 16) * 16;
  Z = (K + kchunk - 1) / kchunk;
  int nwmax = 0;
  for (int c = 0; c < g.ncta; ++c) nwmax = std::max(nwmax, g.nw[c]);
  // stages of 32 columns (16 with 19 warps: the 96-register variant spills with the two-box loop)
  const int KH = nwmax <= 15 ? 2 : 1;
  const unsigned stage_bytes = (unsigned)KH * TB * 32u * 128u;
  g.s = s;
  g.TB = TB;
  g.K = K;
  g.Z = Z;
  g.kchunk = kchunk;
  g.nst = std::min(GT_MAXST, (int)(GT_RING / stage_bytes));
  g.rows_per_batch = idx ? 0 : bstride / ld;
  g.idx = idx;
  g.idx_bstride = idx_bstride;
  g.part = part;
  g.ss = ss;
  const size_t smem = (size_t)g.nst * stage_bytes + 1024;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(gram_tma_kernel<12, true, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, GT_RING + 1024);
    cudaFuncSetAttribute(gram_tma_kernel<16, true, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, GT_RING + 1024);
    cudaFuncSetAttribute(gram_tma_kernel<20, false, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, GT_RING + 1024);
    attr = true;
  }
  count_launches(1);
  if (nwmax <= 11)
    gram_tma_kernel<12, true, 2><<<batch * Z * g.ncta, 12 * 32, smem, st>>>(tm, g);
  else if (nwmax <= 15)
    gram_tma_kernel<16, true, 2><<<batch * Z * g.ncta, 16 * 32, smem, st>>>(tm, g);
  else
    gram_tma_kernel<20, false, 1><<<batch * Z * g.ncta, 20 * 32, smem, st>>>(tm, g);
  return Z;
}

}  // namespace kpp
