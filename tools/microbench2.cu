// st.async issue throughput vs plain DSMEM stores (cluster of 2)
#include <cstdio>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;
__global__ void __cluster_dims__(2, 1, 1) k(int N, int lanes, int mode, long long* out) {
  __shared__ __align__(8) unsigned long long bar;
  __shared__ double buf[1024];
  cg::cluster_group cl = cg::this_cluster();
  const int r = cl.block_rank();
  unsigned lb = (unsigned)__cvta_generic_to_shared(&bar), la = (unsigned)__cvta_generic_to_shared(buf);
  if (threadIdx.x == 0) asm volatile("mbarrier.init.shared.b64 [%0], 1;" :: "r"(lb));
  cl.sync();
  unsigned ra, rb;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(la + 8 * threadIdx.x), "r"(r ^ 1));
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(lb), "r"(r ^ 1));
  double* peer = cl.map_shared_rank(buf, r ^ 1);
  long long t0 = clock64();
  if (r == 0 && threadIdx.x < lanes) {
    for (int i = 0; i < N; ++i) {
      if (mode == 0)
        asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" :: "r"(ra), "d"(1.0 * i), "r"(rb) : "memory");
      else
        ((volatile double*)peer)[threadIdx.x] = 1.0 * i;
    }
  }
  __syncwarp();
  long long t1 = clock64();
  if (threadIdx.x == 0 && r == 0) out[0] = (t1 - t0);
  cl.sync();
}
int main() {
  long long* out; cudaMalloc(&out, 64); long long h;
  for (int mode = 0; mode < 2; ++mode)
    for (int lanes : {1, 8, 32}) {
      k<<<2, 32>>>(100, lanes, mode, out);
      cudaDeviceSynchronize();
      cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
      printf("%s lanes=%d: %.1f cycles per warp-instruction\n", mode ? "plain DSMEM st" : "st.async", lanes, h / 100.0);
    }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
