// schedule.cu -- the data-independent block schedule.
//
// Online block selection with memoization (Alg 5 l.6-8 P:1342-1345;
// Alg 3 l.6-9 P:750-754).  The paper leaves the random generator unspecified; the
// binding convention (readings Q4-Q7) is counter-based Philox-4x32-10
// (Salmon et al., SC'11), so any iteration's decision can be computed independently:
//   decision at t  : counter (lo32 t, hi32 t, 1, 0), key (lo32 seed, hi32 seed)
//                    fresh  <=>  t == 0 || !memo || word0 * 2^-32 < min(1, C/t)
//                    reuse  ->  block floor(word1 * nb / 2^32) of the nb created before t
//   fresh block k  : partial Fisher-Yates over [0, pop), draw i from word (i mod 4) of
//                    counter (i/4, lo32 k, 2, hi32 k); S = sorted first s entries.
#include <cstdint>

#include "kpp_internal.h"

namespace kpp {
namespace {

__device__ __forceinline__ void philox4x32_10(uint32_t c[4], uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int round = 0; round < 10; ++round) {
    const uint32_t hi0 = __umulhi(0xD2511F53u, c[0]);
    const uint32_t lo0 = 0xD2511F53u * c[0];
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c[2]);
    const uint32_t lo1 = 0xCD9E8D57u * c[2];
    const uint32_t n0 = hi1 ^ c[1] ^ k0;
    const uint32_t n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0;
    c[1] = lo1;
    c[2] = n2;
    c[3] = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
}

// One thread per iteration t: Bernoulli draw and reuse word.
__global__ void sched_flags_kernel(uint64_t seed, double C, int memo, long long t0, int count,
                                   uint8_t* fresh, uint32_t* word1) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  const unsigned long long t = (unsigned long long)(t0 + i);
  uint32_t c[4] = {(uint32_t)(t & 0xffffffffull), (uint32_t)(t >> 32), 1u, 0u};
  philox4x32_10(c, (uint32_t)(seed & 0xffffffffull), (uint32_t)(seed >> 32));
  bool f;
  if (t == 0 || !memo) {
    f = true;
  } else {
    const double p = fmin(1.0, __ddiv_rn(C, (double)t));
    const double u = (double)c[0] * 0x1p-32;
    f = u < p;
  }
  fresh[i] = f ? 1 : 0;
  word1[i] = c[1];
}

// Single CTA: exclusive scan of the fresh flags with the carried count, then block ids.
__global__ void __launch_bounds__(1024) sched_scan_kernel(int count, long long* nb_io,
                                                          const uint8_t* fresh,
                                                          const uint32_t* word1, int32_t* bid) {
  __shared__ int warp_sums[32];
  __shared__ long long carry_sh;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) carry_sh = *nb_io;
  __syncthreads();
  for (int base = 0; base < count; base += 1024) {
    const int i = base + tid;
    const int f = (i < count) ? fresh[i] : 0;
    int incl = f;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    if (lane == 31) warp_sums[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      int ws = warp_sums[lane];
      int wi = ws;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, wi, o);
        if (lane >= o) wi += v;
      }
      warp_sums[lane] = wi - ws;  // exclusive prefix of warp totals
    }
    __syncthreads();
    const long long carry = carry_sh;
    const long long before = carry + warp_sums[warp] + (incl - f);  // fresh blocks created before t
    if (i < count) {
      if (f) {
        bid[i] = (int32_t)before;
      } else {
        bid[i] = (int32_t)(((unsigned long long)word1[i] * (unsigned long long)before) >> 32);
      }
    }
    __syncthreads();
    if (tid == 1023) carry_sh = before + f;
    __syncthreads();
  }
  if (tid == 0) *nb_io = carry_sh;
}

// One CTA per fresh block: thread 0 runs the partial Fisher-Yates shuffle with a sparse
// swap map (positions >= s live in an open-addressing table), then all threads rank-sort.
constexpr int FB_THREADS = 256;
constexpr int FB_MAXS = 1024;
constexpr int FB_HASH = 4096;  // >= 2 * FB_MAXS, power of two

__global__ void __launch_bounds__(FB_THREADS) fresh_blocks_kernel(uint64_t seed, long long pop, int s,
                                                                  long long k0, int32_t* S_pool) {
  __shared__ int32_t P[FB_MAXS];
  __shared__ int32_t hkey[FB_HASH];
  __shared__ int32_t hval[FB_HASH];
  const long long k = k0 + blockIdx.x;
  for (int i = threadIdx.x; i < FB_HASH; i += blockDim.x) hkey[i] = -1;
  for (int i = threadIdx.x; i < s; i += blockDim.x) P[i] = i;
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned long long uk = (unsigned long long)k;
    const uint32_t key0 = (uint32_t)(seed & 0xffffffffull), key1 = (uint32_t)(seed >> 32);
    uint32_t w[4] = {0, 0, 0, 0};
    for (int i = 0; i < s; ++i) {
      if ((i & 3) == 0) {
        w[0] = (uint32_t)(i >> 2);
        w[1] = (uint32_t)(uk & 0xffffffffull);
        w[2] = 2u;
        w[3] = (uint32_t)(uk >> 32);
        philox4x32_10(w, key0, key1);
      }
      const uint32_t u = w[i & 3];
      const long long j = i + (long long)(((unsigned long long)u * (unsigned long long)(pop - i)) >> 32);
      if (j == i) continue;
      const int32_t vi = P[i];
      if (j < s) {
        P[i] = P[j];
        P[j] = vi;
      } else {
        // look up / insert position j in the sparse map (default value j)
        uint32_t h = ((uint32_t)j * 2654435761u) & (FB_HASH - 1);
        while (hkey[h] != -1 && hkey[h] != (int32_t)j) h = (h + 1) & (FB_HASH - 1);
        const int32_t vj = (hkey[h] == -1) ? (int32_t)j : hval[h];
        hkey[h] = (int32_t)j;
        hval[h] = vi;
        P[i] = vj;
      }
    }
  }
  __syncthreads();
  // rank sort (values are distinct)
  int32_t* S = S_pool + (size_t)k * s;
  for (int i = threadIdx.x; i < s; i += blockDim.x) {
    const int32_t v = P[i];
    int rank = 0;
    for (int q = 0; q < s; ++q) rank += (P[q] < v);
    S[rank] = v;
  }
}

}  // namespace

void launch_schedule(cudaStream_t st, uint64_t seed, double C, int memo, long long t0, int count,
                     long long* nb_io, uint32_t* word1_ws, uint8_t* fresh_out, int32_t* bid_out) {
  if (count <= 0) return;
  sched_flags_kernel<<<(count + 255) / 256, 256, 0, st>>>(seed, C, memo, t0, count, fresh_out, word1_ws);
  sched_scan_kernel<<<1, 1024, 0, st>>>(count, nb_io, fresh_out, word1_ws, bid_out);
  count_launches(2);
}

void launch_fresh_blocks(cudaStream_t st, uint64_t seed, long long pop, int s, long long k0,
                         long long k1, int32_t* S_pool) {
  if (k1 <= k0) return;
  long long nblk = k1 - k0;
  while (nblk > 0) {
    const int g = (int)(nblk > 65535 ? 65535 : nblk);
    fresh_blocks_kernel<<<g, FB_THREADS, 0, st>>>(seed, pop, s, k0, S_pool);
    count_launches(1);
    k0 += g;
    nblk -= g;
  }
}

}  // namespace kpp
