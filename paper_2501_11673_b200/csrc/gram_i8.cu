// gram_i8.cu -- the Phase-1 Gram G = A_S A_S^T on the int8 tensor cores,
// `tcgen05.mma.kind::i8`, with an exact integer splitting of fp64 (Ozaki scheme).  sm_100a has no f64
// tcgen05 kind; its int8 rate (4.5 POPS nominal) is ~130x the DMMA rate.
//
// Splitting (once per context, A is constant): row r of A gets an exponent e_r with |a_rk| < 2^e_r;
// v = rint(a_rk 2^(54 - e_r)) (|v| <= 2^54, rounding error <= 2^-55 |a_r|_inf) is written as 7
// balanced base-256 digits, v = sum_t d_t 256^t, d_t in [-128, 127] (|d_6| <= 65), stored as 7 int8
// digit planes of A (7/8 of A's bytes), interleaved per row and 128-column block.  Then for two rows r, c of a block
//   G[r][c] = 2^(e_r + e_c - 108) sum_L 256^L D_L[r][c],   D_L = sum_{t+u=L} sum_k d_t[r][k] d_u[c][k],
// every D_L exact in int32 (at most 7 pairs x 4096 columns x 2^14 < 2^29 per K chunk).  Levels
// L = 6..12 are kept (28 ordered digit pairs); the dropped ones weigh < 2^-53 of |a_r|_inf |a_c|_inf
// summed over K.  Measured (tools/ozaki_i8.cu, B200): max |G - exact| / (|a_r| |a_c|) = 3.7e-16
// against 4.6e-15 for a sequential fp64 FMA dot product.
//
// Kernel: one CTA per (block, K chunk, column half h).  A producer warp gathers the block's rows of
// all 7 planes, 128 bytes of K per stage (`cp.async.bulk.tensor ... tile::gather4`, 128-byte
// swizzle = the canonical K-major UMMA layout); one lane issues tcgen05.mma M = 128 (all rows),
// N = 64 (rows 64h .. 64h+63 of the same staged tiles), K = 32 per instruction, into 7 int32
// accumulators of 64 TMEM columns; tcgen05.commit frees the stage.  The epilogue reads the levels
// with tcgen05.ld, assembles them in fp64 (exact power-of-2 scalings, smallest level first) and
// writes the upper triangle into the split-K partial layout of launch_dgemm.
#include <cudaTypedefs.h>

#include <algorithm>

#include "kernel_common.cuh"

namespace kpp {
namespace {
using namespace itk;

constexpr int OZ_DIG = 7;             // digit planes
constexpr int OZ_KT = 128;            // K bytes per stage
constexpr int OZ_ST = 2;              // stages
constexpr int OZ_TILE = 128 * OZ_KT;  // 16 KB: one plane, 128 rows
constexpr int OZ_SMEM = OZ_ST * OZ_DIG * OZ_TILE + 1024;

__global__ void oz_row_exp_kernel(const double* A, long long n, long long lda, int* erow) {
  const long long r = blockIdx.x;
  double mx = 0.0;
  for (long long k = threadIdx.x; k < n; k += blockDim.x) mx = fmax(mx, fabs(A[r * lda + k]));
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  __shared__ double wm[32];
  if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) mx = fmax(mx, wm[w]);
    int e = 0;
    if (mx > 0) frexp(mx, &e);  // mx = f 2^e, f in [0.5, 1): every |a_rk| < 2^e
    erow[r] = e;
  }
}

// 4 consecutive columns per thread -> one 32-bit word per plane; columns n .. npad-1 are zero
__global__ void oz_slice_kernel(const double* A, long long m, long long n, long long lda, long long npad,
                                const int* erow, int8_t* planes) {
  const long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long qpr = npad / 4;
  if (q >= m * qpr) return;
  const long long r = q / qpr, k0 = (q % qpr) * 4;
  const int sc = 54 - erow[r];
  long long v[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) v[e] = k0 + e < n ? __double2ll_rn(ldexp(A[r * lda + k0 + e], sc)) : 0;
  // interleaved: row r, 128-column block kb holds the 7 digit segments of 128 bytes contiguously
  int8_t* seg = planes + (r * (npad / OZ_KT) + k0 / OZ_KT) * (OZ_DIG * OZ_KT) + (k0 % OZ_KT);
#pragma unroll
  for (int t = 0; t < OZ_DIG; ++t) {
    unsigned w = 0;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int d = (int)(signed char)(unsigned char)(v[e] & 0xff);
      v[e] = (v[e] - d) >> 8;
      w |= (unsigned)(unsigned char)(signed char)d << (8 * e);
    }
    *reinterpret_cast<unsigned*>(seg + t * OZ_KT) = w;
  }
}

// K-major, 128-byte swizzle, 8-row atoms of 1024 B: SBO = 1024, version 1, layout type 2
__device__ __forceinline__ unsigned long long oz_desc(unsigned addr) {
  return (unsigned long long)((addr >> 4) & 0x3fff) | (1ull << 16) | ((unsigned long long)(1024 >> 4) << 32) |
         (1ull << 46) | (2ull << 61);
}
// kind::i8: D s32, A and B s8, both K-major, N = 64, M = 128
constexpr unsigned OZ_IDESC = (2u << 4) | (1u << 7) | (1u << 10) | ((64u >> 3) << 17) | ((128u >> 4) << 24);

__device__ __forceinline__ void oz_mma(unsigned dt, unsigned long long a, unsigned long long b, unsigned acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(dt),
      "l"(a), "l"(b), "r"(OZ_IDESC), "r"(acc)
      : "memory");
}

// multicast to both CTAs of the cluster pair (same shared offset, complete_tx on both barriers)
__device__ __forceinline__ void oz_gather4_mc(unsigned dst, const CUtensorMap* tm, int c0, int r0, int r1, int r2,
                                              int r3, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7], %8;\n" ::"r"(dst),
      "l"(reinterpret_cast<unsigned long long>(tm)), "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3),
      "r"(smem_u32(bar)), "h"((unsigned short)3)
      : "memory");
}

__device__ __forceinline__ void oz_gather4(unsigned dst, const CUtensorMap* tm, int c0, int r0, int r1, int r2, int r3,
                                           unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];\n" ::"r"(dst),
      "l"(reinterpret_cast<unsigned long long>(tm)), "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3),
      "r"(smem_u32(bar))
      : "memory");
}

struct OzArgs {
  int s, Z, kchunk, K;
  long long m;                // rows of A (plane height)
  const int8_t* planes;       // [7][m][K] (PROD 2 reads them directly)
  const int* erow;
  const int32_t* idx;
  long long idx_bstride;
  double* part;
  long long ss;
};

// Producers.  PROD 0: one warp, TMA gather4 (one 128-byte row per request: request-bound at ~17
// cycles per row, tensor pipe 23 % busy on c2).  PROD 1: the two column halves run as a cluster pair,
// each CTA gathers half of the planes and multicasts them into both CTAs' stages; the stage is
// released when both CTAs' MMAs are done.  PROD 2: four warps of cp.async (16 bytes per lane, a warp
// covers 4 rows x 128 bytes), written into the 128-byte-swizzled layout by address arithmetic,
// completion through cp.async.mbarrier.arrive; the MMA lane fences the generic->async proxy.
template <int PROD>
__global__ void __launch_bounds__(PROD == 2 ? 192 : 128, 1)
gram_i8_kernel(const __grid_constant__ CUtensorMap tm, const __grid_constant__ OzArgs g) {
  constexpr bool MC = PROD == 1;
  constexpr int MMA_W = PROD == 2 ? 4 : 1, ALLOC_W = PROD == 2 ? 5 : 2;
  extern __shared__ unsigned char oz_sm[];
  __shared__ unsigned long long full[OZ_ST], empty[OZ_ST], done;
  __shared__ unsigned tbase;
  const int h = blockIdx.x & 1, bz = blockIdx.x >> 1;
  const int batch = bz / g.Z, z = bz % g.Z;
  const int kbeg = z * g.kchunk, kend = min(g.K, kbeg + g.kchunk);
  const int nk = kend > kbeg ? (kend - kbeg + OZ_KT - 1) / OZ_KT : 0;
  const unsigned sbase = (smem_u32(oz_sm) + 1023u) & ~1023u;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int32_t* ix = g.idx + (long long)batch * g.idx_bstride;
  if (threadIdx.x == 0) {
    for (int i = 0; i < OZ_ST; ++i) {
      mbar_init(&full[i], PROD == 2 ? 128 : 1);
      mbar_init(&empty[i], MC ? 2 : 1);
    }
    mbar_init(&done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == ALLOC_W) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  if (MC) {  // the peer's barriers must be initialised before any multicast lands
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  } else {
    __syncthreads();
  }
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const unsigned tm0 = tbase;
  if (PROD == 2 && warp < 4) {  // ------------------------------------------- cp.async producers
    // row r's stage = 56 chunks of 16 bytes (7 digit segments of 128 bytes, contiguous); a warp
    // instruction copies 512 contiguous bytes; warp w handles rows w, w + 4, ...
    const long long nkb = g.K / OZ_KT;
    for (int kt = 0; kt < nk; ++kt) {
      const int st = kt % OZ_ST;
      if (kt >= OZ_ST) mbar_wait(&empty[st], ((kt / OZ_ST) - 1) & 1, 81);
      const long long kb = (kbeg / OZ_KT) + kt;
      const unsigned sb = sbase + st * OZ_DIG * OZ_TILE;
#pragma unroll 1
      for (int r = warp; r < 128; r += 4) {
        const int8_t* src = g.planes + ((long long)ix[min(r, g.s - 1)] * nkb + kb) * (OZ_DIG * OZ_KT);
#pragma unroll
        for (int j0 = 0; j0 < 64; j0 += 32) {
          const int j = j0 + lane;  // 16-byte chunk of the row-stage: plane j / 8, chunk j % 8
          if (j < 56) {
            const int t = j >> 3, c = j & 7;
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sb + t * OZ_TILE + r * 128u +
                                                                                ((c ^ (r & 7)) << 4)),
                         "l"(src + j * 16)
                         : "memory");
          }
        }
      }
      asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_u32(&full[st])) : "memory");
    }
  } else if (PROD != 2 && warp == 0) {  // ---------------------------------------- TMA producer
    // gather q = lane: rows 4q .. 4q+3 of the block (rows past s repeat row s-1: their products land
    // in rows / columns past s, which are not stored)
    // interleaved planes as a 2D (rows = (r, kb, t), 128 bytes) tensor
    const int nkb = g.K / OZ_KT;
    int rr[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) rr[e] = ix[min(4 * lane + e, g.s - 1)] * nkb * OZ_DIG;
    for (int kt = 0; kt < nk; ++kt) {
      const int st = kt % OZ_ST;
      if (kt >= OZ_ST) mbar_wait(&empty[st], ((kt / OZ_ST) - 1) & 1, 81);
      if (lane == 0) mbar_expect_tx(&full[st], OZ_DIG * OZ_TILE);
      __syncwarp();
      const int c0 = 0;  // the row index carries the 128-column block
#pragma unroll 1
      for (int t = MC ? h : 0; t < OZ_DIG; t += MC ? 2 : 1) {
        const int pr = (kbeg / OZ_KT + kt) * OZ_DIG + t;
        const unsigned dst = sbase + (st * OZ_DIG + t) * OZ_TILE + lane * 512u;
        if (MC)
          oz_gather4_mc(dst, &tm, c0, pr + rr[0], pr + rr[1], pr + rr[2], pr + rr[3], &full[st]);
        else
          oz_gather4(dst, &tm, c0, pr + rr[0], pr + rr[1], pr + rr[2], pr + rr[3], &full[st]);
      }
    }
  } else if (warp == MMA_W) {  // ---------------------------------------------- MMA issuer
    if (lane == 0) {
      for (int kt = 0; kt < nk; ++kt) {
        const int st = kt % OZ_ST;
        mbar_wait(&full[st], (kt / OZ_ST) & 1, 82);
        if (PROD == 2) asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        const unsigned pl = sbase + st * OZ_DIG * OZ_TILE;
#pragma unroll 1
        for (int L = 6; L <= 12; ++L) {
          const unsigned dt = tm0 + (unsigned)((L - 6) * 64);
          bool first = kt == 0;
          for (int t = L - 6; t <= 6; ++t) {
            const int u = L - t;
            const unsigned at = pl + t * OZ_TILE, bt = pl + u * OZ_TILE + h * 8192u;
#pragma unroll
            for (int k4 = 0; k4 < OZ_KT / 32; ++k4) {
              oz_mma(dt, oz_desc(at + k4 * 32), oz_desc(bt + k4 * 32), first ? 0u : 1u);
              first = false;
            }
          }
        }
        if (MC)
          asm volatile(
              "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::"r"(
                  smem_u32(&empty[st])),
              "h"((unsigned short)3)
              : "memory");
        else
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                           smem_u32(&empty[st]))
                       : "memory");
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                       smem_u32(&done))
                   : "memory");
    }
    __syncwarp();
  }
  if (warp >= 4) {  // the MMA / allocator warps of PROD 2 take no part in the epilogue
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    if (warp == ALLOC_W) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tm0));
    return;
  }
  // ------------------------------------------------------------------------ epilogue (4 warps)
  // warp w reads TMEM lanes 32w .. 32w+31 = rows of the block; 16 columns per load
  const int r = warp * 32 + lane;
  const int s = g.s;
  const int er = g.erow[ix[min(r, s - 1)]];
  double* Cb = g.part + (long long)bz * g.ss;
  if (nk > 0) mbar_wait(&done, 0, 83);
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  for (int c0 = 0; c0 < 64; c0 += 16) {
    double acc[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = 0.0;
#pragma unroll 1
    for (int L = 6; L <= 12; ++L) {  // smallest level first
      unsigned v[16];
      const unsigned ta = tm0 + ((unsigned)(warp * 32) << 16) + (unsigned)((L - 6) * 64 + c0);
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
            "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
          : "r"(ta));
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
      if (nk > 0) {
#pragma unroll
        for (int i = 0; i < 16; ++i) acc[i] += ldexp((double)(int)v[i], 8 * (L - 6));
      }
    }
    if (r < s) {
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int c = h * 64 + c0 + i;
        if (c >= r && c < s) Cb[(long long)r * s + c] = ldexp(acc[i], er + g.erow[ix[c]] - 60);
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  if (MC) {  // no CTA leaves while its peer may still multicast into it or arrive on its barriers
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  } else {
    __syncthreads();
  }
  if (warp == ALLOC_W) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tm0));
}

PFN_cuTensorMapEncodeTiled_v12000 oz_encoder() {
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

}  // namespace

// Opt-in (KPP_GRAM_I8=1): measured slower than the fp64 TMA-ring Gram on c2.
bool gram_i8_enabled(int s) {
  static const int on = getenv("KPP_GRAM_I8") ? atoi(getenv("KPP_GRAM_I8")) : 0;
  return on && s > 64 && s <= 128;
}

long long ozaki_npad(long long n) { return (n + OZ_KT - 1) / OZ_KT * OZ_KT; }

// Digit planes of A (m x n, lda): planes [m][npad/128][7][128] int8 (the 7 digit segments of a row's
// 128-column block contiguous), erow [m].
void launch_ozaki_planes(cudaStream_t st, const double* A, long long m, long long n, long long lda, int8_t* planes,
                         int* erow) {
  const long long npad = ozaki_npad(n);
  oz_row_exp_kernel<<<(unsigned)m, 256, 0, st>>>(A, n, lda, erow);
  const long long nq = m * (npad / 4);
  oz_slice_kernel<<<(unsigned)((nq + 255) / 256), 256, 0, st>>>(A, m, n, lda, npad, erow, planes);
  count_launches(2);
}

// Upper Gram partials of `batch` blocks of s rows (row lists idx) per K chunk, from the digit planes.
// Returns Z, or 0 when not served.
int launch_gram_i8(cudaStream_t st, int batch, int s, int K, const int8_t* planes, long long m, const int* erow,
                   const int32_t* idx, long long idx_bstride, double* part, long long ss, int Z) {
  if (batch <= 0 || !gram_i8_enabled(s) || !planes || !idx || 7 * m * (ozaki_npad(K) / OZ_KT) > 0x7fffffffLL)
    return 0;
  PFN_cuTensorMapEncodeTiled_v12000 encode = oz_encoder();
  if (!encode) return 0;
  const long long npad = ozaki_npad(K);
  CUtensorMap tm;
  cuuint64_t dims[2] = {(cuuint64_t)OZ_KT, (cuuint64_t)(OZ_DIG * m * (npad / OZ_KT))};
  cuuint64_t strides[1] = {(cuuint64_t)OZ_KT};
  cuuint32_t box[2] = {(cuuint32_t)OZ_KT, 1u};
  cuuint32_t estr[2] = {1u, 1u};
  if (encode(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, (void*)planes, dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return 0;
  // K chunks: multiples of 128 columns (padded planes: the last chunk reads zeros past K)
  if (Z < 1) Z = 1;
  int kchunk = (int)((npad + Z - 1) / Z);
  kchunk = (kchunk + OZ_KT - 1) / OZ_KT * OZ_KT;
  if (kchunk > 16384) return 0;  // 7 digit pairs x kchunk x 2^14 must stay below 2^31
  Z = (int)((npad + kchunk - 1) / kchunk);
  OzArgs g{};
  g.s = s;
  g.Z = Z;
  g.kchunk = kchunk;
  g.K = (int)npad;
  g.m = m;
  g.erow = erow;
  g.idx = idx;
  g.idx_bstride = idx_bstride;
  g.part = part;
  g.ss = ss;
  g.planes = planes;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(gram_i8_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, OZ_SMEM);
    cudaFuncSetAttribute(gram_i8_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, OZ_SMEM);
    cudaFuncSetAttribute(gram_i8_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, OZ_SMEM);
    attr = true;
  }
  static const int prod = getenv("KPP_GRAM_I8_PROD") ? atoi(getenv("KPP_GRAM_I8_PROD")) : 1;
  count_launches(1);
  const unsigned nblk = (unsigned)(batch * Z * 2);
  if (prod == 1) {
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(nblk);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = OZ_SMEM;
    cfg.stream = st;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    if (cudaLaunchKernelEx(&cfg, gram_i8_kernel<1>, tm, g) == cudaSuccess) return Z;
    cudaGetLastError();
  }
  if (prod == 2)
    gram_i8_kernel<2><<<nblk, 192, OZ_SMEM, st>>>(tm, g);
  else
    gram_i8_kernel<0><<<nblk, 128, OZ_SMEM, st>>>(tm, g);
  return Z;
}

}  // namespace kpp
