// grid_common.cuh -- device helpers of the persistent grid-wide kernels (lsqr.cu, dist.cu): warp and
// block reductions with a fixed order, tagged LL words through L2 / peer memory, cp.async.
// Product code: shares nothing with oracle/.
#pragma once
#include <cstdint>

namespace kpp {
namespace gx {

__device__ __forceinline__ double wsum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Sums of V values over the 32 lanes with V - 1 + log2(32 / V) shuffles (reduce-scatter butterflies,
// then a plain butterfly): afterwards every lane l holds the total of value (l >> (5 - log2 V)),
// returned.  Fixed order: the same in every warp and CTA.
template <int V>
__device__ __forceinline__ double warp_multi_sum(double (&a)[V]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int h = V / 2, o = 16; h >= 1; h >>= 1, o >>= 1) {
    const bool up = (lane & o) != 0;
#pragma unroll
    for (int i = 0; i < h; ++i) {
      const double send = up ? a[i] : a[i + h];
      const double keep = up ? a[i + h] : a[i];
      a[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
  }
  double v = a[0];
#pragma unroll
  for (int o = 16 / V; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
template <int V>
__device__ __forceinline__ int warp_multi_index() {
  constexpr int SH = V == 1 ? 5 : V == 2 ? 4 : V == 4 ? 3 : V == 8 ? 2 : V == 16 ? 1 : 0;
  return (threadIdx.x & 31) >> SH;
}

// block-wide fixed-order sums (every thread gets the results, one barrier): red holds 2 slots of
// 2 x 32 doubles used alternately (slot toggled by the caller), so a slot is rewritten only after
// every thread has passed the barrier of the call in between.
__device__ __forceinline__ void block_sum2(double& a, double& b, double* red, int& slot) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  a = wsum(a);
  b = wsum(b);
  double* r = red + 64 * slot;
  slot ^= 1;
  if (lane == 0) {
    r[warp] = a;
    r[32 + warp] = b;
  }
  __syncthreads();
  a = wsum(lane < nw ? r[lane] : 0.0);
  b = wsum(lane < nw ? r[32 + lane] : 0.0);
}
__device__ __forceinline__ double block_sum(double v, double* red, int& slot) {
  double z = 0.0;
  block_sum2(v, z, red, slot);
  return v;
}

__device__ __forceinline__ void ll_put(unsigned long long* dst, double v, unsigned tag) {
  const unsigned long long u = (unsigned long long)__double_as_longlong(v);
  const unsigned long long tg = (unsigned long long)tag << 32;
  asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};\n" ::"l"(dst), "l"(tg | (u & 0xffffffffull)),
               "l"(tg | (u >> 32))
               : "memory");
}
__device__ __forceinline__ void cp_async16(void* smem, const void* g) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(g) : "memory");
}
static __device__ __noinline__ void ll_fail(int* err) {
  atomicExch(err, 3);
  __trap();
}
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long v;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
  return v;
}
// fixed-order sum of the values src[q * stride] (q = q0, q0 + 32, ... < nq): all loads in flight,
// re-polled until every tag matches (watchdog: 20 s, then trap)
// BACKOFF (ns): sleep between unsuccessful polling rounds (many SMs polling the same lines)
template <int KQ, int BACKOFF = 0>
__device__ __forceinline__ double ll_sum(const unsigned long long* src, long long stride, int q0, int nq, unsigned tag,
                                         int* err) {
  unsigned long long a[KQ], b[KQ];
#pragma unroll
  for (int i = 0; i < KQ; ++i) {
    const int q = q0 + 32 * i;
    if (q < nq)
      asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];\n" : "=l"(a[i]), "=l"(b[i]) : "l"(src + q * stride) : "memory");
    else
      a[i] = b[i] = (unsigned long long)tag << 32;
  }
  unsigned long long t0 = 0;
  unsigned n = 0;
  for (;;) {
    bool all = true;
#pragma unroll
    for (int i = 0; i < KQ; ++i)
      if ((unsigned)(a[i] >> 32) != tag || (unsigned)(b[i] >> 32) != tag) {
        all = false;
        asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];\n" : "=l"(a[i]), "=l"(b[i]) : "l"(src + (q0 + 32 * i) * stride) : "memory");
      }
    if (all) break;
    if (BACKOFF) __nanosleep(BACKOFF);
    if (n == 0) t0 = gtimer();
    if ((++n & 1023u) == 0 && gtimer() - t0 > 20000000000ull) ll_fail(err);
  }
  double v = 0.0;
#pragma unroll
  for (int i = 0; i < KQ; ++i)
    if (q0 + 32 * i < nq) v += __longlong_as_double((long long)((a[i] & 0xffffffffull) | (b[i] << 32)));
  return v;
}

// LL store with system scope: the destination may be a peer GPU's memory mapped over NVLink.
__device__ __forceinline__ void ll_put_sys(unsigned long long* dst, double v, unsigned tag) {
  const unsigned long long u = (unsigned long long)__double_as_longlong(v);
  const unsigned long long tg = (unsigned long long)tag << 32;
  asm volatile("st.relaxed.sys.global.v2.u64 [%0], {%1, %2};\n" ::"l"(dst), "l"(tg | (u & 0xffffffffull)),
               "l"(tg | (u >> 32))
               : "memory");
}
// Poll one LL value written with system scope (by this or a peer GPU).
__device__ __forceinline__ double ll_get_sys(const unsigned long long* src, unsigned tag, int* err) {
  unsigned long long a, b, t0 = 0;
  unsigned n = 0;
  for (;;) {
    asm volatile("ld.relaxed.sys.global.v2.u64 {%0, %1}, [%2];\n" : "=l"(a), "=l"(b) : "l"(src) : "memory");
    if ((unsigned)(a >> 32) == tag && (unsigned)(b >> 32) == tag) break;
    if (n == 0) t0 = gtimer();
    if ((++n & 1023u) == 0 && gtimer() - t0 > 20000000000ull) ll_fail(err);
  }
  return __longlong_as_double((long long)((a & 0xffffffffull) | (b << 32)));
}

}  // namespace gx
}  // namespace kpp
