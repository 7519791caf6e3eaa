// Exchange-skeleton microbenchmark of the c2 persistent-kernel iteration (B200, sm_100a).
// Grid of NQ clusters x C CTAs x 512 threads; per iteration, with no arithmetic of the method:
//   stage 1  every warp sends its 8 row partials to the slice-owner CTA of the cluster (st.async)
//   stage 2  owner warp waits (mbarrier), sums, publishes the cluster partial as LL words in L2
//   stage 3  pollers gather the slice over all clusters (G2 pollers per row, optional back-off)
//   stage 4  r slice -> every CTA of the cluster (st.async), wait
//   stage 5  y slice -> every CTA of the cluster (st.async), wait      (mode & 1: skipped)
//   stage 6  __syncthreads (the w / x update barrier)
// Prints cycles per iteration for each variant.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

constexpr int T = 512, NW = 16, S = 128;

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ unsigned mapa(unsigned a, int r) {
  unsigned o;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r));
  return o;
}
__device__ __forceinline__ void st_async(unsigned ra, double v, unsigned rb) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(ra), "d"(v), "r"(rb)
               : "memory");
}
__device__ __forceinline__ void expect(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void wait(unsigned long long* b, unsigned par) {
  asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}" ::"r"(
                   smem_u32(b)),
               "r"(par)
               : "memory");
}
__device__ __forceinline__ void ll_st(unsigned long long* d, double v, unsigned tag) {
  unsigned long long u = __double_as_longlong(v), t = (unsigned long long)tag << 32;
  asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(d), "l"(t | (u & 0xffffffffull)), "l"(t | (u >> 32))
               : "memory");
}
__device__ __forceinline__ void ll_ld(const unsigned long long* s, unsigned long long& a, unsigned long long& b) {
  asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(s) : "memory");
}

__global__ void __launch_bounds__(T, 1) skel(unsigned long long* ll, int iters, int mode, int g2max, int backoff,
                                               long long* out) {
  __shared__ __align__(8) unsigned long long bars[4];
  __shared__ double rp[4 * 32], r_sm[S], y_sm[S], red[16 * 32];
  cg::cluster_group cl = cg::this_cluster();
  const int C = cl.num_blocks(), c = cl.block_rank(), q = blockIdx.x / C, NQ = gridDim.x / C;
  const int sl = S / C, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int i = 0; i < 4; ++i) asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(smem_u32(bars + i)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  cl.sync();
  const unsigned la_rp = smem_u32(rp), la_r = smem_u32(r_sm), la_y = smem_u32(y_sm);
  long long t0 = clock64();
  double acc = 0.0;
  for (int it = 0; it < iters; ++it) {
    const unsigned tag = it + 1, par = it & 1;
    unsigned long long* g = ll + (long long)(it & 1) * NQ * S * 2;
    if (tid == 0) {
      expect(bars + 0, C * sl * 8);
      expect(bars + 1, S * 8);
      if (!(mode & 1)) expect(bars + 2, S * 8);
    }
    __syncthreads();
    // stage 1: warp w owns rows w + 16 i (i < 8); lane (i) sends row w + 16 i
    if (lane < 8) {
      const int k = warp + 16 * lane, owner = k / sl;
      st_async(mapa(la_rp + (c * sl + k - owner * sl) * 8, owner), 1.0 + acc, mapa(smem_u32(bars + 0), owner));
    }
    // stage 2
    if (warp == 0) {
      wait(bars + 0, par);
      double v = 0.0;
      for (int cc = 0; cc < C; ++cc) v += rp[cc * sl + lane];
      ll_st(g + ((long long)q * S + c * sl + lane) * 2, v, tag);
    }
    // stage 3
    const int G2 = min(g2max, T / sl);
    if (tid < sl * G2) {
      const int row = tid % sl, grp = tid / sl;
      double v = 0.0;
      for (int qq = grp; qq < NQ; qq += G2) {
        unsigned long long a, b;
        const unsigned long long* src = g + ((long long)qq * S + c * sl + row) * 2;
        ll_ld(src, a, b);
        while ((unsigned)(a >> 32) != tag || (unsigned)(b >> 32) != tag) {
          if (backoff) __nanosleep(backoff);
          ll_ld(src, a, b);
        }
        v += __longlong_as_double((a & 0xffffffffull) | (b << 32));
      }
      red[grp * sl + row] = v;
    }
    __syncthreads();
    // stage 4
    if (tid < sl) {
      double v = 0.0;
      for (int i = 0; i < G2; ++i) v += red[i * sl + tid];
      for (int cc = 0; cc < C; ++cc) st_async(mapa(la_r + (c * sl + tid) * 8, cc), v, mapa(smem_u32(bars + 1), cc));
    }
    wait(bars + 1, par);
    // stage 5
    if (!(mode & 1)) {
      if (tid < sl) {
        const double v = r_sm[c * sl + tid] * 0.5;
        for (int cc = 0; cc < C; ++cc) st_async(mapa(la_y + (c * sl + tid) * 8, cc), v, mapa(smem_u32(bars + 2), cc));
      }
      wait(bars + 2, par);
      acc += y_sm[lane] * 1e-300;
    } else {
      acc += r_sm[lane] * 1e-300;
    }
    // stage 6
    __syncthreads();
  }
  if (blockIdx.x == 0 && tid == 0) out[0] = (clock64() - t0) / iters;
  if (acc == 12345.0) out[1] = 1;
  cl.sync();
}

int main(int argc, char** argv) {
  unsigned long long* ll;
  long long* out;
  cudaMalloc(&ll, 2LL * 160 * S * 2 * 8);
  cudaMalloc(&out, 64);
  struct V { int C, grid, mode, g2, bo; } vs[] = {
      {4, 132, 0, 16, 0}, {4, 132, 1, 16, 0}, {4, 132, 0, 4, 0}, {4, 132, 0, 1, 0}, {4, 132, 0, 16, 64},
      {4, 132, 0, 4, 64}, {8, 128, 0, 16, 0}, {8, 128, 0, 4, 0}, {2, 132, 0, 16, 0}, {4, 64, 0, 16, 0},
      {4, 32, 0, 16, 0}, {4, 8, 0, 16, 0}};
  for (auto v : vs) {
    cudaMemset(ll, 0, 2LL * 160 * S * 2 * 8);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(v.grid);
    cfg.blockDim = dim3(T);
    cudaLaunchAttribute a[1];
    a[0].id = cudaLaunchAttributeClusterDimension;
    a[0].val.clusterDim.x = v.C;
    a[0].val.clusterDim.y = 1;
    a[0].val.clusterDim.z = 1;
    cfg.attrs = a;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, skel, ll, 4000, v.mode, v.g2, v.bo, out);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[2];
    cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
    printf("C=%d grid=%d %s G2max=%d backoff=%d: %lld cycles/iter (%.2f us at 1965 MHz) %s\n", v.C, v.grid,
           v.mode & 1 ? "r only " : "r and y", v.g2, v.bo, h[0], h[0] / 1965.0, cudaGetErrorString(e));
  }
  return 0;
}
