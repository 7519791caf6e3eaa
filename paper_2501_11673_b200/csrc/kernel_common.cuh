// kernel_common.cuh -- device helpers shared by the persistent Phase-2 kernels
// (iterate_kernel.cuh, cdpp_stream.cu): LL words over L2, mbarriers with a watchdog, TMA bulk
// copies, DSMEM stores, cp.async, warp reductions.  Product code: shares nothing with oracle/.
#pragma once
#include <cooperative_groups.h>

#include <cmath>
#include <cstdio>
#include <cstdint>

#include "kpp_internal.h"
#include "window.cuh"

namespace cg = cooperative_groups;

namespace kpp {
namespace itk {

constexpr int T2 = 512;
constexpr int NW2 = T2 / 32;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// ------------------------------------------------------------------ LL words
// value v with tag g -> two words (g << 32 | lo32(v)), (g << 32 | hi32(v))
__device__ __forceinline__ void ll_store_global(unsigned long long* dst, double v, unsigned tag) {
  const unsigned long long u = (unsigned long long)__double_as_longlong(v);
  const unsigned long long t = (unsigned long long)tag << 32;
  asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};\n" ::"l"(dst), "l"(t | (u & 0xffffffffull)),
               "l"(t | (u >> 32))
               : "memory");
}
static __device__ __noinline__ void spin_fail(int* err) {
  atomicExch(err, 1);
  __trap();
}
__device__ __forceinline__ double ll_wait_global(const unsigned long long* src, unsigned tag, int* err) {
  unsigned long long a, b;
  asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];\n" : "=l"(a), "=l"(b) : "l"(src) : "memory");
  if ((unsigned)(a >> 32) != tag || (unsigned)(b >> 32) != tag) {
    const unsigned long long t0 = globaltimer();
    unsigned n = 0;
    while ((unsigned)(a >> 32) != tag || (unsigned)(b >> 32) != tag) {
      asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];\n" : "=l"(a), "=l"(b) : "l"(src) : "memory");
      if ((++n & 1023u) == 0 && globaltimer() - t0 > 20000000000ull) spin_fail(err);
    }
  }
  return __longlong_as_double((long long)((a & 0xffffffffull) | (b << 32)));
}

// Sum of LL values at src[q * stride] for q = q0, q0 + dq, ... < nq (fixed order), with every
// load of the thread in flight at once: one L2 round trip once the data is there.
// BACKOFF (ns): sleep between unsuccessful polling rounds (pollers that overlap an HBM stream
// should not flood L2 with requests)
template <int KQ, int BACKOFF = 0>
__device__ __forceinline__ double ll_gather_sum(const unsigned long long* src, long long stride, int q0, int dq, int nq,
                                                unsigned tag, int* err, int backoff_ns = 0) {
  unsigned long long a[KQ], b[KQ];
  int cnt = 0;
#pragma unroll
  for (int i = 0; i < KQ; ++i) {
    const int qq = q0 + i * dq;
    if (qq < nq) {
      asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];\n" : "=l"(a[i]), "=l"(b[i]) : "l"(src + qq * stride) : "memory");
      cnt = i + 1;
    } else {
      a[i] = b[i] = (unsigned long long)tag << 32;
    }
  }
  const unsigned long long t0 = globaltimer();
  unsigned n = 0;
  for (;;) {
    bool all = true;
#pragma unroll
    for (int i = 0; i < KQ; ++i) {
      if ((unsigned)(a[i] >> 32) != tag || (unsigned)(b[i] >> 32) != tag) {
        all = false;
        asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];\n" : "=l"(a[i]), "=l"(b[i]) : "l"(src + (q0 + i * dq) * stride) : "memory");
      }
    }
    if (all) break;
    if (BACKOFF) __nanosleep(BACKOFF);
    if (backoff_ns) __nanosleep(backoff_ns);
    if ((++n & 1023u) == 0 && globaltimer() - t0 > 20000000000ull) spin_fail(err);
  }
  double v = 0.0;
#pragma unroll
  for (int i = 0; i < KQ; ++i)
    if (i < cnt) v += __longlong_as_double((long long)((a[i] & 0xffffffffull) | (b[i] << 32)));
  return v;
}

// LL words with system scope: the destination / source may be a peer GPU's memory mapped over NVLink
__device__ __forceinline__ void ll_store_sys(unsigned long long* dst, double v, unsigned tag) {
  const unsigned long long u = (unsigned long long)__double_as_longlong(v);
  const unsigned long long tg = (unsigned long long)tag << 32;
  asm volatile("st.relaxed.sys.global.v2.u64 [%0], {%1, %2};\n" ::"l"(dst), "l"(tg | (u & 0xffffffffull)),
               "l"(tg | (u >> 32))
               : "memory");
}
__device__ __forceinline__ double ll_wait_sys(const unsigned long long* src, unsigned tag, int* err) {
  unsigned long long a, b;
  asm volatile("ld.relaxed.sys.global.v2.u64 {%0, %1}, [%2];\n" : "=l"(a), "=l"(b) : "l"(src) : "memory");
  if ((unsigned)(a >> 32) != tag || (unsigned)(b >> 32) != tag) {
    const unsigned long long t0 = globaltimer();
    unsigned n = 0;
    while ((unsigned)(a >> 32) != tag || (unsigned)(b >> 32) != tag) {
      asm volatile("ld.relaxed.sys.global.v2.u64 {%0, %1}, [%2];\n" : "=l"(a), "=l"(b) : "l"(src) : "memory");
      if ((++n & 1023u) == 0 && globaltimer() - t0 > 20000000000ull) spin_fail(err);
    }
  }
  return __longlong_as_double((long long)((a & 0xffffffffull) | (b << 32)));
}

// Rank stage of the column-sharded exchange: cluster 0 of each rank (publish)
// stores the rank's partial v of s-vector row `row`, tagged with the global iteration t + 1, into
// slot [t mod 2][rank] of EVERY rank's receive buffer ([2][P][s] LL words, peer memory over NVLink or
// device memory when emulated); then the P partials of the row are summed in rank order (the same
// bits on every rank).  Out of line: single-GPU runs never call it and keep their loop bodies small.
static __device__ __noinline__ double rank_stage_sum(double v, bool publish, unsigned long long* const* recv, int rank,
                                                     int P, int s, int row, long long t, int* err) {
  const long long pslot = (t & 1) * (long long)P * s;
  const unsigned ptag = (unsigned)(t + 1);
  if (publish)
    for (int rr = 0; rr < P; ++rr) ll_store_sys(recv[rr] + 2 * (pslot + (long long)rank * s + row), v, ptag);
  double tot = 0.0;
  for (int rr = 0; rr < P; ++rr) tot += ll_wait_sys(recv[rank] + 2 * (pslot + (long long)rr * s + row), ptag, err);
  return tot;
}

// ------------------------------------------------------------------ TMA bulk copies + mbarriers
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_try(unsigned long long* bar, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n .reg .pred p;\n"
      " mbarrier.try_wait.parity.shared.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// Watchdog: a wait that has not completed after 10 s reports the barrier and traps (a lost
// transaction would otherwise hang the GPU).
static __device__ __noinline__ void mbar_hang(int code, unsigned parity) {
  printf("kpp: mbarrier wait timed out (site %d, parity %u, CTA %d, thread %d)\n", code, parity, (int)blockIdx.x,
         (int)threadIdx.x);
  __trap();
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity, int code = 0) {
  if (mbar_try(bar, parity)) return;
  const unsigned long long t0 = globaltimer();
  unsigned n = 0;
  while (!mbar_try(bar, parity))
    if ((++n & 255u) == 0 && globaltimer() - t0 > 10000000000ull) mbar_hang(code, parity);
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// TMA gather4: 4 rows (r0..r3) x box columns starting at column c0 -> dst (dense rows)
__device__ __forceinline__ void tma_gather4(void* dst, const CUtensorMap* tm, int c0, int r0, int r1, int r2, int r3,
                                            unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<unsigned long long>(tm)), "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(bar))
      : "memory");
}
// TMA gather4 prefetch into L2 only (no shared-memory destination, no mbarrier)
__device__ __forceinline__ void tma_prefetch_gather4(const CUtensorMap* tm, int c0, int r0, int r1, int r2, int r3) {
  asm volatile(
      "cp.async.bulk.prefetch.tensor.2d.L2.global.tile::gather4 [%0, {%1, %2, %3, %4, %5}];\n" ::"l"(
          reinterpret_cast<unsigned long long>(tm)),
      "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3)
      : "memory");
}
// DSMEM: remote shared::cluster address of a local shared variable in CTA `rank`
__device__ __forceinline__ unsigned mapa_u32(unsigned la, int rank) {
  unsigned ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(ra) : "r"(la), "r"(rank));
  return ra;
}
// asynchronous remote store that completes `8` transaction bytes on the remote mbarrier
__device__ __forceinline__ void st_async_f64(unsigned raddr, double v, unsigned rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];\n" ::"r"(raddr), "d"(v),
               "r"(rbar)
               : "memory");
}
// Wait for bytes delivered by peers' st.async.  CTA-scope acquire is enough: the data are in this
// CTA's shared memory and complete_tx makes them visible with the phase; a cluster-scope acquire
// would also invalidate L1 (CCTL.IVALL) on every wait.
__device__ __forceinline__ bool mbar_try_cta(unsigned long long* bar, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n .reg .pred p;\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait_cluster(unsigned long long* bar, unsigned parity, int code = 0) {
  if (mbar_try_cta(bar, parity)) return;
  const unsigned long long t0 = globaltimer();
  unsigned n = 0;
  while (!mbar_try_cta(bar, parity))
    if ((++n & 255u) == 0 && globaltimer() - t0 > 10000000000ull) mbar_hang(code, parity);
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

// cp.async fallback (rows that are not 16-byte aligned)
__device__ __forceinline__ void cp_async8(void* smem, const void* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(smem)), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async4(void* smem, const void* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(smem_u32(smem)), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

// Warp 0: load s row segments of the slab (and optionally `mcount` doubles of M rows).
// bulk: TMA bulk copies completing on `bar` (lane 0 registers the byte count first);
// otherwise 8-byte cp.async (waited with cp.async.wait_group by warp 0).
__device__ __forceinline__ void issue_loads(bool bulk, const CUtensorMap* tm, const double* A, long long lda,
                                            const int32_t* S, int s, long long c0, int w, double* adst, int sw,
                                            bool slab, const double* msrc, int mcount, double* mdst,
                                            unsigned long long* bar) {
  const int lane = threadIdx.x & 31;
  if (bulk) {
    const int nops = (s + 3) >> 2;  // gather4 ops (TMA path)
    unsigned bytes = 0;
    if (slab && w > 0) bytes += tm ? (unsigned)nops * 4u * (unsigned)sw * 8u : (unsigned)s * (unsigned)w * 8u;
    if (msrc && mcount > 0) bytes += (unsigned)mcount * 8u;
    if (lane == 0) mbar_expect_tx(bar, bytes);
    __syncwarp();
    if (slab && w > 0) {
      if (tm) {
        for (int j = lane; j < nops; j += 32) {
          const int k = 4 * j;
          tma_gather4(adst + (long long)k * sw, tm, (int)c0, S[k], S[min(k + 1, s - 1)], S[min(k + 2, s - 1)],
                      S[min(k + 3, s - 1)], bar);
        }
      } else {
        for (int k = lane; k < s; k += 32)
          bulk_g2s(adst + (long long)k * sw, A + (long long)S[k] * lda + c0, (unsigned)w * 8u, bar);
      }
    }
    if (msrc && mcount > 0 && lane == 0) bulk_g2s(mdst, msrc, (unsigned)mcount * 8u, bar);
  } else {
    if (slab)
      for (int k = 0; k < s; ++k) {
        const double* src = A + (long long)S[k] * lda + c0;
        double* d = adst + (long long)k * sw;
        for (int j = lane; j < w; j += 32) cp_async8(d + j, src + j);
      }
    if (msrc)
      for (int e = lane; e < mcount; e += 32) cp_async8(mdst + e, msrc + e);
    cp_async_commit();
  }
}

// First-pass loads of the streaming kernel: CD++ streams (evict-first), K++ tags the part of the
// block its second pass should find in L2 with an evict_last policy.
template <int CDT>
__device__ __forceinline__ double2 ld_pass1(const double2* ptr, unsigned long long pol) {
  if constexpr (CDT) return __ldcs(ptr);
  double2 v;
  asm volatile("ld.global.nc.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;\n" : "=d"(v.x), "=d"(v.y) : "l"(ptr), "l"(pol));
  return v;
}
template <int CDT>
__device__ __forceinline__ double ld_pass1(const double* ptr, unsigned long long pol) {
  if constexpr (CDT) return __ldcs(ptr);
  double v;
  asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;\n" : "=d"(v) : "l"(ptr), "l"(pol));
  return v;
}

#define TRACE(e)                                                                              \
  do {                                                                                        \
    if (p.trace && tid == 0 && it >= 64 && it < 64 + 16)                                      \
      p.trace[(((long long)(it - 64) * gridDim.x) + blockIdx.x) * 8 + (e)] = (long long)globaltimer(); \
  } while (0)

#define PHASE_MARK(i)                   \
  do {                                  \
    if (prof_on) {                      \
      const long long now_ = clock64(); \
      prof_acc[i] += now_ - prof_last;  \
      prof_last = now_;                 \
    }                                   \
  } while (0)

// Butterfly reduce-scatter of RPW per-lane values over the 32 lanes of a warp: afterwards
// v[0] of lane l is the full warp sum of value index rs_row<RPW>(l) (fixed order: deterministic).
template <int RPW>
__device__ __forceinline__ void warp_reduce_scatter(double (&v)[RPW], int lane) {
  int o = 16;
#pragma unroll
  for (int cnt = RPW; cnt > 1; cnt >>= 1, o >>= 1) {
    const int half = cnt >> 1;
    const bool upper = (lane & o) != 0;
#pragma unroll
    for (int i = 0; i < half; ++i) {
      const double send = upper ? v[i] : v[i + half];
      const double keep = upper ? v[i + half] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
  }
  for (; o >= 1; o >>= 1) v[0] += __shfl_xor_sync(0xffffffffu, v[0], o);
}
template <int RPW>
__device__ __forceinline__ int rs_row(int lane) {
  int r = 0, o = 16;
#pragma unroll
  for (int cnt = RPW; cnt > 1; cnt >>= 1, o >>= 1)
    if (lane & o) r += cnt >> 1;
  return r;
}


}  // namespace itk
}  // namespace kpp
