// iterate.cu -- Phase 2: the per-iteration memoized block update.
//
// For each iteration t of a window (Alg 5 l.9-18 P:1346-1357 / Alg 3 l.10-20 P:755-766):
//   r   = A_S x - b_S                                   (row 3)
//   y   = M r,  M = (A_S A_S^T + lam I)^{-1} memoized    (row 4; K++)  / (A_SS + lam I)^{-1} (CD++)
//   w   = A_S^T y (K++, Eq (bk))  |  I_S^T y (CD++, Alg 3 l.11)        (row 5)
//   m   = (1-rho)/(1+rho) (m - w);  x = x - w + eta m   (row 6, Eq (momentum))
//   E0/E1 window sums, checkpoint every 2 zeta: stop test, adaptive rho   (row 8)
//
// Engine "persistent": one cooperative launch per window, one CTA per SM.  CTA g owns a
// column slab [g*slab, (g+1)*slab) of x, m and A; the s-vector partials of A_S x are
// combined through a deterministic grid reduction (fixed order, no atomics on data),
// every CTA replicates the scalar window logic on identical bits, so all CTAs take the
// same stop / rho decisions without further exchange.
//
// Engine "graph" (multi-GPU, and a single-GPU cross-check): the same arithmetic split
// into step kernels so that an NCCL allreduce of the s-vector can sit between them.
#include <cmath>
#include <cstdint>

#include "kpp_internal.h"
#include "window.cuh"

namespace kpp {
namespace {

constexpr int IT_THREADS = 512;
constexpr int NWARPS = IT_THREADS / 32;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Grid-wide barrier over a monotonically increasing arrival counter.
__device__ __forceinline__ void grid_sync(unsigned* bar, unsigned& target) {
  target += gridDim.x;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(bar, 1u);
    while (ld_acquire(bar) < target) {
    }
    __threadfence();
  }
  __syncthreads();
}

// CD++ scatter: position of global column gj in the sorted block S (or -1).
__device__ __forceinline__ int find_sorted(const int32_t* S, int s, long long gj) {
  int lo = 0, hi = s - 1;
  while (lo <= hi) {
    const int mid = (lo + hi) >> 1;
    const long long v = S[mid];
    if (v == gj) return mid;
    if (v < gj) lo = mid + 1; else hi = mid - 1;
  }
  return -1;
}

__global__ void __launch_bounds__(IT_THREADS, 1) iterate_kernel(IterParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int s = p.s;
  double* y_sh = reinterpret_cast<double*>(smem_raw);
  double* r_sh = y_sh + s;
  int32_t* S_sh = reinterpret_cast<int32_t*>(r_sh + s);
  __shared__ DevState st;
  __shared__ int stop_sh;
  const int G = gridDim.x, g = blockIdx.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const long long c0 = (long long)g * p.slab;
  const long long c1 = (c0 + p.slab < p.n) ? c0 + p.slab : p.n;
  if (tid == 0) {
    st = *p.st;
    stop_sh = 0;
  }
  __syncthreads();
  unsigned target = 0;
  long long t = p.t0;
  for (; t < p.t1; ++t) {
    const long long k = p.bid[t - p.t0];
    const int32_t* S = p.S_pool + k * s;
    const double* M = p.M_pool + k * (long long)s * s;
    for (int i = tid; i < s; i += IT_THREADS) S_sh[i] = S[i];
    __syncthreads();
    const double rho = st.rho;  // set at the last checkpoint strictly before t (reading Q11)
    // row 3: partial block residual over this CTA's slab
    for (int kk = warp; kk < s; kk += NWARPS) {
      const double* row = p.A + (long long)S_sh[kk] * p.lda;
      double acc = 0.0;
      for (long long j = c0 + lane; j < c1; j += 32) acc = fma(row[j], p.x[j], acc);
      acc = warp_sum(acc);
      if (lane == 0) p.part[(long long)g * s + kk] = acc;
    }
    grid_sync(p.bar, target);
    // combine partials in a fixed order: r_k = sum_g part[g][k] - b_{S_k}
    for (int kk = g * NWARPS + warp; kk < s; kk += G * NWARPS) {
      double acc = 0.0;
      for (int q = lane; q < G; q += 32) acc += __ldcg(p.part + (long long)q * s + kk);
      acc = warp_sum(acc);
      if (lane == 0) p.r[kk] = acc - p.b[S_sh[kk]];
    }
    grid_sync(p.bar, target);
    // row 4: y = M r
    for (int kk = g * NWARPS + warp; kk < s; kk += G * NWARPS) {
      const double* Mrow = M + (long long)kk * s;
      double acc = 0.0;
      for (int l = lane; l < s; l += 32) acc = fma(Mrow[l], __ldcg(p.r + l), acc);
      acc = warp_sum(acc);
      if (lane == 0) p.y[kk] = acc;
    }
    grid_sync(p.bar, target);
    for (int i = tid; i < s; i += IT_THREADS) {
      y_sh[i] = __ldcg(p.y + i);
      r_sh[i] = __ldcg(p.r + i);
    }
    __syncthreads();
    // rows 5-6: back-projection and momentum update on the slab
    const double c = (1.0 - rho) / (1.0 + rho);
    for (long long j = c0 + tid; j < c1; j += IT_THREADS) {
      double w = 0.0;
      if (!p.cd) {
        for (int q = 0; q < s; ++q) w = fma(p.A[(long long)S_sh[q] * p.lda + j], y_sh[q], w);
      } else {
        const int pos = find_sorted(S_sh, s, p.col_base + j);
        if (pos >= 0) w = y_sh[pos];
      }
      const double mm = c * (p.mom[j] - w);
      p.mom[j] = mm;
      p.x[j] = p.x[j] - w + p.eta * mm;
    }
    // row 8: ||r||^2 and the replicated window logic
    if (warp == 0) {
      double e = 0.0;
      for (int i = lane; i < s; i += 32) e = fma(r_sh[i], r_sh[i], e);
      e = warp_sum(e);
      if (lane == 0) {
        const int res = window_step_dev(st, t, e, p.zeta, p.tol2bb, p.bb, p.adaptive, g == 0,
                                    p.hist_res, p.hist_rho, p.hist_cap);
        if (res) {
          st.stopped = res;
          stop_sh = 1;
        }
      }
    }
    __syncthreads();
    if (stop_sh) {
      ++t;
      break;
    }
  }
  if (g == 0 && tid == 0) {
    st.t_done = t;
    *p.st = st;
  }
}

}  // namespace

int iterate_block_threads() { return IT_THREADS; }

size_t iterate_smem_bytes(int s, int /*slab*/, int /*resident*/) {
  return (size_t)s * (2 * sizeof(double) + sizeof(int32_t)) + 16;
}

cudaError_t launch_iterate(cudaStream_t stream, const IterParams& p, int grid, int block, size_t smem) {
  IterParams pp = p;
  void* args[] = {&pp};
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(iterate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  count_launches(1);
  return cudaLaunchCooperativeKernel((const void*)iterate_kernel, dim3(grid), dim3(block), args, smem, stream);
}

int iterate_max_grid(int device, size_t smem) {
  int sms = 0, per = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  if (smem > 48 * 1024) cudaFuncSetAttribute(iterate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, iterate_kernel, IT_THREADS, smem);
  return sms * (per > 0 ? 1 : 0);
}

}  // namespace kpp
