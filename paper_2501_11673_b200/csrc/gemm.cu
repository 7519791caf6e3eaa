// gemm.cu -- batched fp64 GEMM on the FP64 tensor cores for Phase 1.
//
// The Phase-1 Gram A_S A_S^T and the CholeskyQR2 products are
// dense contractions, so they run on DMMA: `mma.sync.aligned.m8n8k4.row.col.f64`
// (sm_100a has no tcgen05 kind for f64; ptxas lowers this to DMMA.8x8x4).
// Tile: 64 x 64 output per CTA, K step 16, 8 warps (2 x 4), each warp 32 x 16 = 4 x 2
// mma tiles, double-buffered shared-memory stages.  Split-K across gridDim.z; partial
// products are reduced in a fixed order by splitk_reduce (deterministic, no atomics).
#include <cstdint>

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
                                                        int upper_only) {
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
      if (gj < N) Cb[(long long)gi * ldc + gj] = acc[i][j][0];
      if (gj + 1 < N) Cb[(long long)gi * ldc + gj + 1] = acc[i][j][1];
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

}  // namespace

int launch_dgemm(cudaStream_t st, int batch, int M, int N, int K, const Operand& a, const Operand& b,
                 double* C, long long ldc, long long c_bstride, int Z, int upper_only) {
  if (batch <= 0 || M <= 0 || N <= 0) return Z;
  if (Z < 1) Z = 1;
  int kchunk = (K + Z - 1) / Z;
  kchunk = ((kchunk + BK - 1) / BK) * BK;
  Z = (K + kchunk - 1) / kchunk;
  if (Z < 1) Z = 1;
  dim3 grid((N + BN - 1) / BN, (M + BM - 1) / BM, batch * Z);
  if (!a.trans && !b.trans)
    dgemm_kernel<false, false><<<grid, THREADS, 0, st>>>(M, N, K, Z, kchunk, a, b, C, ldc, c_bstride, upper_only);
  else if (!a.trans && b.trans)
    dgemm_kernel<false, true><<<grid, THREADS, 0, st>>>(M, N, K, Z, kchunk, a, b, C, ldc, c_bstride, upper_only);
  else if (a.trans && !b.trans)
    dgemm_kernel<true, false><<<grid, THREADS, 0, st>>>(M, N, K, Z, kchunk, a, b, C, ldc, c_bstride, upper_only);
  else
    dgemm_kernel<true, true><<<grid, THREADS, 0, st>>>(M, N, K, Z, kchunk, a, b, C, ldc, c_bstride, upper_only);
  count_launches(1);
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
