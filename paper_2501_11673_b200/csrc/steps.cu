// steps.cu -- Phase 2 as step kernels (engine "graph").
//
// Same arithmetic as the persistent kernel in iterate.cu, split at the one exchange
// point of the column-sharded layout: every rank computes its partial
// A_S[:, cols_p] x[cols_p]; an NCCL allreduce (fp64 sum, in place) combines the
// s-vector; then every rank applies the replicated solve y = M (r - b_S) and updates its
// own columns.  The current iteration index lives in device memory (DevStep), so one
// captured CUDA graph of U iterations is replayed for every window without re-capture.
#include <cmath>
#include <cstdint>

#include "kpp_internal.h"
#include "window.cuh"

namespace kpp {
namespace {

constexpr int ST_THREADS = 512;
constexpr int ST_WARPS = ST_THREADS / 32;

__device__ __forceinline__ double wsum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ bool step_active(const DevState* st, const DevStep* sp, long long* t) {
  const long long tt = sp->t_cur;
  *t = tt;
  return st->stopped == 0 && tt < sp->t_end;
}

__global__ void __launch_bounds__(ST_THREADS) step_partial_kernel(StepParams p) {
  long long t;
  if (!step_active(p.st, p.sp, &t)) return;
  const int s = p.s;
  const long long k = p.bid[t - p.sp->t_base];
  const int32_t* S = p.S_pool + k * s;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = blockIdx.x;
  const long long c0 = (long long)g * p.slab;
  const long long c1 = (c0 + p.slab < p.n) ? c0 + p.slab : p.n;
  for (int kk = warp; kk < s; kk += ST_WARPS) {
    const double* row = p.A + (long long)S[kk] * p.lda;
    double acc = 0.0;
    for (long long j = c0 + lane; j < c1; j += 32) acc = fma(row[j], p.x[j], acc);
    acc = wsum(acc);
    if (lane == 0) p.part[(long long)g * s + kk] = acc;
  }
}

__device__ __noinline__ void peer_fail(int* err) {
  atomicExch(err, 4);
  __trap();
}

// rsum[k] = sum_g part[g][k] (fixed order).  Peer mode (the B200-native replacement of the NCCL
// allreduce between this kernel and the solve): lane 0 publishes the rank's sum as two
// tagged 8-byte words (32 data bits + 32-bit tag t+1; an aligned 8-byte store is single-copy atomic,
// so seeing the tag means seeing the data) into slot [t mod 2][rank][k] of EVERY rank's receive
// buffer over NVLink (system-scope stores to the peers' mapped memory), then lanes r < nranks poll
// slot [t mod 2][r][k] of the local buffer and the warp sums the ranks in rank order -- the same
// bits on every rank.  Two parity slots suffice: a rank can only publish t+2 after every rank has
// published t+1, i.e. after every rank has consumed t.
__global__ void __launch_bounds__(ST_THREADS) step_reduce_kernel(StepParams p) {
  long long t;
  if (!step_active(p.st, p.sp, &t)) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kk = blockIdx.x * ST_WARPS + warp;
  if (kk >= p.s) return;
  double acc = 0.0;
  for (int q = lane; q < p.grid; q += 32) acc += p.part[(long long)q * p.s + kk];
  acc = wsum(acc);
  if (!p.peer) {
    if (lane == 0) p.rsum[kk] = acc;
    return;
  }
  const unsigned tag = (unsigned)(t + 1);
  const long long slot = ((long long)(t & 1) * p.nranks) * p.s;
  if (lane < p.nranks) {  // lane r stores into rank r's buffer
    const unsigned long long u = (unsigned long long)__double_as_longlong(acc);
    const unsigned long long tg = (unsigned long long)tag << 32;
    unsigned long long* dst = p.peer_recv[lane] + 2 * (slot + (long long)p.rank * p.s + kk);
    asm volatile("st.relaxed.sys.global.v2.u64 [%0], {%1, %2};\n" ::"l"(dst), "l"(tg | (u & 0xffffffffull)),
                 "l"(tg | (u >> 32))
                 : "memory");
  }
  double v = 0.0;
  if (lane < p.nranks) {
    const unsigned long long* src = p.peer_recv[p.rank] + 2 * (slot + (long long)lane * p.s + kk);
    unsigned long long a, b;
    unsigned long long t0 = 0;
    unsigned n = 0;
    for (;;) {
      asm volatile("ld.relaxed.sys.global.v2.u64 {%0, %1}, [%2];\n" : "=l"(a), "=l"(b) : "l"(src) : "memory");
      if ((unsigned)(a >> 32) == tag && (unsigned)(b >> 32) == tag) break;
      if (n == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
      if ((++n & 1023u) == 0) {
        unsigned long long now;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
        if (now - t0 > 20000000000ull) peer_fail(p.err);
      }
    }
    v = __longlong_as_double((long long)((a & 0xffffffffull) | (b << 32)));
  }
  double tot = 0.0;  // ranks in order 0 .. nranks-1
  for (int r = 0; r < p.nranks; ++r) tot += __shfl_sync(0xffffffffu, v, r);
  if (lane == 0) p.rsum[kk] = tot;
}

__global__ void __launch_bounds__(ST_THREADS) step_solve_kernel(StepParams p) {
  long long t;
  if (!step_active(p.st, p.sp, &t)) return;
  const int s = p.s;
  const long long k = p.bid[t - p.sp->t_base];
  const int32_t* S = p.S_pool + k * s;
  const double* M = p.M_pool + k * (long long)s * s;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kk = blockIdx.x * ST_WARPS + warp;
  if (kk >= s) return;
  const double* Mrow = M + (long long)kk * s;
  double acc = 0.0;
  for (int l = lane; l < s; l += 32) acc = fma(Mrow[l], p.rsum[l] - p.b[S[l]], acc);
  acc = wsum(acc);
  if (lane == 0) p.y[kk] = acc;
}

__device__ __forceinline__ int find_sorted_s(const int32_t* S, int s, long long gj) {
  int lo = 0, hi = s - 1;
  while (lo <= hi) {
    const int mid = (lo + hi) >> 1;
    const long long v = S[mid];
    if (v == gj) return mid;
    if (v < gj) lo = mid + 1; else hi = mid - 1;
  }
  return -1;
}

__global__ void __launch_bounds__(ST_THREADS) step_update_kernel(StepParams p) {
  long long t;
  if (!step_active(p.st, p.sp, &t)) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int s = p.s;
  double* y_sh = reinterpret_cast<double*>(smem_raw);
  int32_t* S_sh = reinterpret_cast<int32_t*>(y_sh + s);
  const long long k = p.bid[t - p.sp->t_base];
  const int32_t* S = p.S_pool + k * s;
  for (int i = threadIdx.x; i < s; i += ST_THREADS) {
    y_sh[i] = p.y[i];
    S_sh[i] = S[i];
  }
  const double rho = p.st->rho;
  __syncthreads();
  const double c = (1.0 - rho) / (1.0 + rho);
  const long long c0 = (long long)blockIdx.x * p.slab;
  const long long c1 = (c0 + p.slab < p.n) ? c0 + p.slab : p.n;
  for (long long j = c0 + threadIdx.x; j < c1; j += ST_THREADS) {
    double w = 0.0;
    if (!p.cd) {
      for (int q = 0; q < s; ++q) w = fma(p.A[(long long)S_sh[q] * p.lda + j], y_sh[q], w);
    } else {
      const int pos = find_sorted_s(S_sh, s, p.col_base + j);
      if (pos >= 0) w = y_sh[pos];
    }
    const double mm = c * (p.mom[j] - w);
    p.mom[j] = mm;
    p.x[j] = p.x[j] - w + p.eta * mm;
  }
}

// One warp: ||r||^2 with the persistent kernel's summation order, then the window logic.
__global__ void step_window_kernel(StepParams p) {
  long long t;
  if (!step_active(p.st, p.sp, &t)) return;
  const int s = p.s, lane = threadIdx.x;
  const long long k = p.bid[t - p.sp->t_base];
  const int32_t* S = p.S_pool + k * s;
  double e = 0.0;
  for (int i = lane; i < s; i += 32) {
    const double r = p.rsum[i] - p.b[S[i]];
    e = fma(r, r, e);
  }
  e = wsum(e);
  if (lane == 0) {
    DevState st = *p.st;
    const int res = window_step_dev(st, t % (2 * p.zeta), e, p.zeta, p.tol2bb, p.bb, p.adaptive, p.writer,
                                    p.hist_res, p.hist_rho, p.hist_cap);
    if (res) st.stopped = res;
    st.t_done = t + 1;
    *p.st = st;
    p.sp->t_cur = t + 1;
  }
}

}  // namespace

size_t step_update_smem(int s) { return (size_t)s * (sizeof(double) + sizeof(int32_t)) + 16; }

void launch_step_partial(cudaStream_t st, const StepParams& p) {
  step_partial_kernel<<<p.grid, ST_THREADS, 0, st>>>(p);
  count_launches(1);
}
void launch_step_reduce(cudaStream_t st, const StepParams& p) {
  step_reduce_kernel<<<(p.s + ST_WARPS - 1) / ST_WARPS, ST_THREADS, 0, st>>>(p);
  count_launches(1);
}
void launch_step_solve(cudaStream_t st, const StepParams& p) {
  step_solve_kernel<<<(p.s + ST_WARPS - 1) / ST_WARPS, ST_THREADS, 0, st>>>(p);
  count_launches(1);
}
void launch_step_update(cudaStream_t st, const StepParams& p) {
  const size_t sm = step_update_smem(p.s);
  if (sm > 48 * 1024) cudaFuncSetAttribute(step_update_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  step_update_kernel<<<p.grid, ST_THREADS, sm, st>>>(p);
  count_launches(1);
}
void launch_step_window(cudaStream_t st, const StepParams& p) {
  step_window_kernel<<<1, 32, 0, st>>>(p);
  count_launches(1);
}

}  // namespace kpp
