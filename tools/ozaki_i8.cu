// ozaki_i8.cu -- microbenchmark prototype (last bullet): the Phase-1 Gram
// G = A_S A_S^T emulated on the int8 tensor cores, `tcgen05.mma.kind::i8`, Ozaki-style.
// Not part of the product library; it answers "how fast would the int8 route be on sm_100a" with
// numbers before any integration.
//
// Splitting: every row r of A_S gets an exponent e_r with |a_rk| < 2^e_r; v = rint(a 2^(54 - e_r))
// is a 55-bit integer, written as 7 balanced base-256 digits d_0..d_6 (d_t in [-128, 127],
// v = sum_t d_t 256^t, |d_6| <= 64).  Then
//   G[r][c] = 2^(e_r + e_c - 108) sum_{t,u} 256^(t+u) D_tu[r][c],  D_tu = sum_k d_t[r][k] d_u[c][k],
// exact in int32 (|D_tu| <= K 2^14; a level L = t + u sums at most 7 of them: < 2^31 for K <= 8192).
// Levels L = 6..12 are kept (28 ordered digit pairs); the dropped ones weigh <= 2^-56 of the top.
//
// Kernels: (1) slice: fp64 rows -> 7 int8 digit planes (global); (2) gram: one CTA per (block,
// level group); a producer lane loads 128-row x 128-byte digit tiles with TMA (SWIZZLE_128B, the
// canonical K-major UMMA layout), one lane issues tcgen05.mma (M = N = 128, K = 32 per
// instruction, int32 accumulators in TMEM, one 128-column accumulator per level), tcgen05.commit
// frees the stage; four warps read the levels back with tcgen05.ld and store them as int32.
// The host checks every level exactly against int64 sums of the same digits, and the assembled fp64
// Gram against a long-double Gram of A_S.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o tools/ozaki_i8 tools/ozaki_i8.cu -lcuda
// Run:   tools/ozaki_i8 [blocks=64] [K=4096] [reps=20]
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#define CK(x)                                                                                  \
  do {                                                                                         \
    cudaError_t e_ = (x);                                                                      \
    if (e_ != cudaSuccess) {                                                                   \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_));       \
      exit(1);                                                                                 \
    }                                                                                          \
  } while (0)

constexpr int ROWS = 128;       // rows of a block (s = 128, c2)
constexpr int NDIG = 7;         // digit planes
constexpr int KT = 128;         // K bytes per stage (one 128-byte swizzle row)
constexpr int NST = 2;          // stages (7 digit tiles of 16 KB each)
constexpr int TILE = ROWS * KT; // 16 KB per digit tile

// --------------------------------------------------------------------------------------- slicing
__global__ void row_exp_kernel(const double* A, int K, int* erow) {
  const int r = blockIdx.x;
  double m = 0.0;
  for (int k = threadIdx.x; k < K; k += blockDim.x) m = fmax(m, fabs(A[(long long)r * K + k]));
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  __shared__ double wm[32];
  if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = fmax(m, wm[w]);
    m = fmax(m, wm[0]);
    int e;
    frexp(m, &e);  // m = f 2^e, f in [0.5, 1): |a| < 2^e
    erow[r] = m > 0 ? e : 0;
  }
}

// 4 consecutive elements per thread -> one 32-bit word per digit plane
__global__ void slice_kernel(const double* A, long long nrows, int K, const int* erow, int8_t* D) {
  const long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x;  // quad index
  const long long nq = nrows * K / 4;
  if (q >= nq) return;
  const long long r = q * 4 / K;
  const int sc = 54 - erow[r];
  const double4 a = reinterpret_cast<const double4*>(A)[q];
  long long v[4] = {__double2ll_rn(ldexp(a.x, sc)), __double2ll_rn(ldexp(a.y, sc)), __double2ll_rn(ldexp(a.z, sc)),
                    __double2ll_rn(ldexp(a.w, sc))};
  const long long plane = nrows * (long long)K;
#pragma unroll
  for (int t = 0; t < NDIG; ++t) {
    unsigned w = 0;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int d = (int)(signed char)(unsigned char)(v[e] & 0xff);
      v[e] = (v[e] - d) >> 8;
      w |= ((unsigned)(unsigned char)(signed char)d) << (8 * e);
    }
    reinterpret_cast<unsigned*>(D + t * plane)[q] = w;
  }
}

// ------------------------------------------------------------------------------------ tcgen05 gram
__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(unsigned long long* b, unsigned c) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(su32(b)), "r"(c));
}
__device__ __forceinline__ void mb_expect(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mb_wait(unsigned long long* b, unsigned par) {
  unsigned ok = 0;
  while (!ok)
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(su32(b)), "r"(par)
        : "memory");
}
__device__ __forceinline__ void tma2d(unsigned dst, const CUtensorMap* tm, int c0, int c1, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          dst),
      "l"(reinterpret_cast<unsigned long long>(tm)), "r"(c0), "r"(c1), "r"(su32(bar))
      : "memory");
}
// K-major, SWIZZLE_128B, 8-row atoms of 1024 B: SBO = 1024, version 1, layout type 2
__device__ __forceinline__ unsigned long long sdesc(unsigned addr) {
  return (unsigned long long)((addr >> 4) & 0x3fff) | (1ull << 16) | ((unsigned long long)(1024 >> 4) << 32) |
         (1ull << 46) | (2ull << 61);
}
// kind::i8: D s32 (bits 4-5 = 2), A s8 (bits 7-9 = 1), B s8 (bits 10-12 = 1), K-major both,
// N >> 3 at bit 17, M >> 4 at bit 24
constexpr unsigned IDESC = (2u << 4) | (1u << 7) | (1u << 10) | ((128u >> 3) << 17) | ((128u >> 4) << 24);

__device__ __forceinline__ void mma_i8(unsigned dt, unsigned long long a, unsigned long long b, unsigned acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(dt),
      "l"(a), "l"(b), "r"(IDESC), "r"(acc));
}

// grid: blocks x groups; group g covers levels [lo, hi] (L = t + u, 6..12)
struct Groups {
  int lo[4], hi[4];
};

__global__ void __launch_bounds__(128, 1)
gram_i8_kernel(const __grid_constant__ CUtensorMap tm, int K, long long nrows, Groups gr, int* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ unsigned long long full[NST], empty[NST], done;
  __shared__ unsigned tbase;
  const int blk = blockIdx.x, g = blockIdx.y;
  const int lo = gr.lo[g], hi = gr.hi[g];
  const int nlev = hi - lo + 1;
  const int tmin = lo - 6 < 0 ? 0 : lo - 6;  // digits used: t = L - u with u <= 6 -> t >= L - 6
  const int nt = NDIG - tmin;                // digit planes tmin..6 are loaded
  const unsigned sbase = (su32(sm) + 1023u) & ~1023u;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NST; ++i) mb_init(&full[i], 1), mb_init(&empty[i], 1);
    mb_init(&done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const unsigned tm0 = tbase;
  const int nk = K / KT;
  if (warp == 0 && lane == 0) {  // TMA producer
    for (int kt = 0; kt < nk; ++kt) {
      const int st = kt % NST;
      if (kt >= NST) mb_wait(&empty[st], ((kt / NST) - 1) & 1);
      mb_expect(&full[st], nt * TILE);
      for (int t = tmin; t < NDIG; ++t)
        tma2d(sbase + (st * NDIG + t) * TILE, &tm, kt * KT, (int)(t * nrows + (long long)blk * ROWS), &full[st]);
    }
  } else if (warp == 1 && lane == 0) {  // MMA issuer
    for (int kt = 0; kt < nk; ++kt) {
      const int st = kt % NST;
      mb_wait(&full[st], (kt / NST) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      for (int L = lo; L <= hi; ++L) {
        const unsigned dt = tm0 + (unsigned)((L - lo) * 128);
        bool first = kt == 0;
        for (int t = L - 6 < 0 ? 0 : L - 6; t <= 6 && t <= L; ++t) {
          const int u = L - t;
          const unsigned at = sbase + (st * NDIG + t) * TILE, bt = sbase + (st * NDIG + u) * TILE;
#pragma unroll
          for (int k4 = 0; k4 < KT / 32; ++k4) {
            mma_i8(dt, sdesc(at + k4 * 32), sdesc(bt + k4 * 32), first ? 0u : 1u);
            first = false;
          }
        }
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&empty[st]))
                   : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&done))
                 : "memory");
  }
  __syncwarp();
  // epilogue: warp w reads TMEM lanes 32w..32w+31 (rows), 16 columns per load
  mb_wait(&done, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int row = warp * 32 + lane;
  for (int l = 0; l < nlev; ++l)
    for (int c0 = 0; c0 < 128; c0 += 16) {
      unsigned v[16];
      const unsigned ta = tm0 + ((unsigned)(warp * 32) << 16) + (unsigned)(l * 128 + c0);
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
            "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
          : "r"(ta));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      int* o = out + (((long long)blk * 7 + (lo - 6 + l)) * ROWS + row) * ROWS + c0;
#pragma unroll
      for (int i = 0; i < 16; ++i) o[i] = (int)v[i];
    }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm0));
}

// ------------------------------------------------------------------------------------------ host
int main(int argc, char** argv) {
  const int B = argc > 1 ? atoi(argv[1]) : 64;
  const int K = argc > 2 ? atoi(argv[2]) : 4096;
  const int reps = argc > 3 ? atoi(argv[3]) : 20;
  const long long nrows = (long long)B * ROWS;
  printf("blocks %d  K %d  (block = %d rows)\n", B, K, ROWS);
  std::mt19937_64 rng(1);
  std::normal_distribution<double> nd;
  std::uniform_real_distribution<double> ud(-6.0, 0.0);
  std::vector<double> hA(nrows * K);
  for (auto& x : hA) x = nd(rng) * std::exp2(ud(rng)) / std::sqrt((double)K);
  double *dA;
  int *derow, *dout;
  int8_t* dD;
  CK(cudaMalloc(&dA, hA.size() * 8));
  CK(cudaMalloc(&derow, nrows * 4));
  CK(cudaMalloc(&dD, (size_t)NDIG * nrows * K));
  CK(cudaMalloc(&dout, (size_t)B * 7 * ROWS * ROWS * 4));
  CK(cudaMemcpy(dA, hA.data(), hA.size() * 8, cudaMemcpyHostToDevice));
  row_exp_kernel<<<(int)nrows, 256>>>(dA, K, derow);
  const long long nq = nrows * K / 4;
  const int sgrid = (int)((nq + 255) / 256);
  slice_kernel<<<sgrid, 256>>>(dA, nrows, K, derow, dD);
  CK(cudaDeviceSynchronize());

  // tensor map over the digit planes: (NDIG * nrows) x K int8, box 128 x 128, 128-byte swizzle
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult qr;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &qr));
  CUtensorMap tm;
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)(NDIG * nrows)};
  cuuint64_t strides[1] = {(cuuint64_t)K};
  cuuint32_t box[2] = {KT, ROWS}, es[2] = {1, 1};
  CUresult cr = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, dD, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) {
    printf("tensor map encode failed %d\n", (int)cr);
    return 1;
  }
  // level groups balanced by digit pairs: L = 6..12 has 7,6,5,4,3,2,1 pairs -> {6} 7, {7} 6, {8,9} 9, {10,11,12} 6
  Groups gr{{6, 7, 8, 10}, {6, 7, 9, 12}};
  const size_t smem = (size_t)NST * NDIG * TILE + 1024;
  CK(cudaFuncSetAttribute(gram_i8_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  dim3 grid(B, 4);
  gram_i8_kernel<<<grid, 128, smem>>>(tm, K, nrows, gr, dout);
  CK(cudaDeviceSynchronize());

  // ---- exact check of the level accumulators (first 2 blocks)
  std::vector<int8_t> hD((size_t)NDIG * nrows * K);
  std::vector<int> hout((size_t)B * 7 * ROWS * ROWS), herow(nrows);
  CK(cudaMemcpy(hD.data(), dD, hD.size(), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(hout.data(), dout, hout.size() * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(herow.data(), derow, nrows * 4, cudaMemcpyDeviceToHost));
  long long bad = 0, checked = 0;
  const int nchk = B < 2 ? B : 2;
  for (int b = 0; b < nchk; ++b)
    for (int L = 6; L <= 12; ++L)
      for (int r = 0; r < ROWS; r += 3)
        for (int c = 0; c < ROWS; c += 5) {
          long long s = 0;
          for (int t = 0; t <= 6; ++t) {
            const int u = L - t;
            if (u < 0 || u > 6) continue;
            const int8_t* x = &hD[(size_t)t * nrows * K + ((size_t)b * ROWS + r) * K];
            const int8_t* y = &hD[(size_t)u * nrows * K + ((size_t)b * ROWS + c) * K];
            for (int k = 0; k < K; ++k) s += (long long)x[k] * y[k];
          }
          const long long g = hout[(((size_t)b * 7 + (L - 6)) * ROWS + r) * ROWS + c];
          ++checked;
          if (g != s && bad++ < 5) printf("  mismatch b%d L%d r%d c%d: gpu %lld exact %lld\n", b, L, r, c, g, s);
        }
  printf("level accumulators: %lld of %lld checked entries differ\n", bad, checked);
  // ---- fp64 assembly against a long-double Gram (block 0)
  double maxrel = 0, maxrel_d = 0;
  for (int r = 0; r < ROWS; ++r)
    for (int c = r; c < ROWS; ++c) {
      long double ex = 0, nrm_r = 0, nrm_c = 0;
      double dg = 0;
      for (int k = 0; k < K; ++k) {
        const double x = hA[(size_t)r * K + k], y = hA[(size_t)c * K + k];
        ex += (long double)x * y;
        dg = fma(x, y, dg);
        nrm_r += (long double)x * x;
        nrm_c += (long double)y * y;
      }
      double g = 0;
      for (int L = 6; L <= 12; ++L)
        g += std::ldexp((double)hout[((size_t)(L - 6) * ROWS + r) * ROWS + c], 8 * L + herow[r] + herow[c] - 108);
      const long double scale = std::sqrt(nrm_r * nrm_c);
      maxrel = std::fmax(maxrel, (double)(std::fabs((long double)g - ex) / scale));
      maxrel_d = std::fmax(maxrel_d, (double)(std::fabs((long double)dg - ex) / scale));
    }
  printf("block 0 Gram, max |G - exact| / (|a_r| |a_c|): int8 Ozaki %.3e, sequential fp64 FMA %.3e (u = 1.1e-16)\n",
         maxrel, maxrel_d);

  // ---- timing
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int i = 0; i < reps; ++i) slice_kernel<<<sgrid, 256>>>(dA, nrows, K, derow, dD);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms_s = 0;
  cudaEventElapsedTime(&ms_s, e0, e1);
  ms_s /= reps;
  cudaEventRecord(e0);
  for (int i = 0; i < reps; ++i) gram_i8_kernel<<<grid, 128, smem>>>(tm, K, nrows, gr, dout);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms_g = 0;
  cudaEventElapsedTime(&ms_g, e0, e1);
  ms_g /= reps;
  CK(cudaGetLastError());
  const double elems = (double)nrows * K;
  const double ops = 28.0 * 2.0 * ROWS * ROWS * (double)K * B;
  printf("slice: %.3f ms  %.1f G elements/s  (fp64 in %.0f GB/s, int8 out %.0f GB/s)\n", ms_s, elems / ms_s / 1e6,
         elems * 8 / ms_s / 1e6, elems * NDIG / ms_s / 1e6);
  printf("gram i8: %.3f ms  %.0f TOPS int8 (28 digit pairs, M = N = 128, K = %d, %d blocks x 4 level groups)\n", ms_g,
         ops / ms_g / 1e9, K, B);
  printf("fp64-equivalent Gram rate (2 s^2 K per block, full square): %.1f TF/s\n",
         2.0 * ROWS * ROWS * (double)K * B / ms_g / 1e9);
  return 0;
}
