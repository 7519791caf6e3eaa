// Latency microbenchmarks for the exchange primitives of the persistent kernel (B200).
#include <cstdio>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned long long ldr(const unsigned long long* p) {
  unsigned long long v; asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory"); return v; }
__device__ __forceinline__ void str(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" :: "l"(p), "l"(v) : "memory"); }
__device__ __forceinline__ unsigned long long ldv(const unsigned long long* p) {
  unsigned long long v; asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory"); return v; }

// global ping-pong between block 0 and block `other` (different SMs): N round trips
__global__ void pingpong(unsigned long long* flags, int N, long long* out, int other) {
  if (threadIdx.x != 0) return;
  if (blockIdx.x == 0) {
    long long t0 = clock64();
    for (int i = 1; i <= N; ++i) {
      str(flags, i);
      while (ldr(flags + 16) != (unsigned long long)i) {}
    }
    out[0] = (clock64() - t0) / N;
  } else if (blockIdx.x == other) {
    for (int i = 1; i <= N; ++i) {
      while (ldr(flags) != (unsigned long long)i) {}
      str(flags + 16, i);
    }
  }
}

// DSMEM ping-pong in a cluster of 2 via st.async + mbarrier
__global__ void __cluster_dims__(2, 1, 1) dsmem_pp(int N, long long* out) {
  __shared__ __align__(8) unsigned long long bar;
  __shared__ double buf;
  cg::cluster_group cl = cg::this_cluster();
  const int r = cl.block_rank();
  unsigned lb = (unsigned)__cvta_generic_to_shared(&bar), la = (unsigned)__cvta_generic_to_shared(&buf);
  if (threadIdx.x == 0) asm volatile("mbarrier.init.shared.b64 [%0], 1;" :: "r"(lb));
  cl.sync();
  if (threadIdx.x == 0) {
    unsigned ra, rb;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(la), "r"(r ^ 1));
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(lb), "r"(r ^ 1));
    long long t0 = clock64();
    for (int i = 0; i < N; ++i) {
      asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], 8;" :: "r"(lb) : "memory");
      if (r == 0) asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" :: "r"(ra), "d"(1.0 * i), "r"(rb) : "memory");
      asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}" :: "r"(lb), "r"(i & 1) : "memory");
      if (r == 1) asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" :: "r"(ra), "d"(1.0 * i), "r"(rb) : "memory");
    }
    if (r == 0) out[1] = (clock64() - t0) / N;
  }
  cl.sync();
}

__global__ void syncbench(int N, long long* out) {
  long long t0 = clock64();
  for (int i = 0; i < N; ++i) __syncthreads();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[2] = (clock64() - t0) / N;
}

__global__ void __cluster_dims__(4, 1, 1) clsync(int N, long long* out) {
  cg::cluster_group cl = cg::this_cluster();
  long long t0 = clock64();
  for (int i = 0; i < N; ++i) cl.sync();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[3] = (clock64() - t0) / N;
}

int main() {
  unsigned long long* flags; long long* out;
  cudaMalloc(&flags, 4096); cudaMalloc(&out, 64);
  long long h[8];
  int others[] = {1, 2, 37, 74, 100, 147};
  for (int o : others) {
    cudaMemset(flags, 0, 4096);
    pingpong<<<148, 32>>>(flags, 2000, out, o);
    cudaDeviceSynchronize();
    cudaMemcpy(h, out, 8, cudaMemcpyDeviceToHost);
    printf("global relaxed ping-pong block0<->block%d: %lld cycles/round trip\n", o, h[0]);
  }
  dsmem_pp<<<2, 32>>>(2000, out);
  syncbench<<<1, 512>>>(10000, out);
  clsync<<<4, 512>>>(10000, out);
  cudaDeviceSynchronize();
  cudaMemcpy(h, out, 64, cudaMemcpyDeviceToHost);
  printf("dsmem st.async+mbarrier ping-pong: %lld cycles/round trip\n", h[1]);
  printf("__syncthreads (512 thr): %lld cycles\n", h[2]);
  printf("cluster.sync (4 x 512 thr): %lld cycles\n", h[3]);
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
