// dist.cu -- the fused compute + exchange Phase-2 kernel (engine 2; default for column-sharded
// contexts, SURVEY 8(e) "B200-native upgrade").
//
// One persistent cooperative kernel per window, one CTA per SM.  Per block iteration (Alg 5 l.9-12
// P:1346-1349 / Alg 3 l.10-13 P:755-759) on rank p's column slab A[:, cols_p]:
//   (a) CTA g: row sums of its slab, part[g][k] = sum_{j in slab g} A[S_k][j] x_j, as tagged LL
//       words in L2 (the slab sits in shared memory when it fits: double-buffered, the next block's
//       slab streaming in by cp.async behind the current iteration, or a single copy reused by (e));
//   (b) exchange: the owner warp of k (CTA k mod grid) sums the grid's words in a fixed order and
//       stores the rank's partial into slot [t mod 2][p][k] of EVERY rank's receive buffer -- over
//       NVLink for the peers (CUDA IPC mappings, system-scope stores of 32 data bits + 32-bit tag per
//       8-byte word) -- and every CTA gathers slot [t mod 2][0..P-1][k] of its own buffer, summing
//       the ranks in rank order: the same bits on every rank, no NCCL call and no kernel boundary
//       between the partial products and the solve;
//   (c) r = (A_S x)_total - b_S, e = ||r||^2;  (d) y = M r: by every CTA from M staged in shared
//       memory when it fits, else row k by CTA k mod grid and gathered through L2 (one more hop);
//       bit-identical on every CTA of every rank either way;
//   (e) w = A_S^T y on the slab (K++) or the scatter of y (CD++), m <- c (m - w), x <- x - w + eta m;
//   (f) window logic (row 8), replicated.
// Two parity slots suffice for the peer buffers: a rank publishes t+2 only after every rank has
// published t+1, i.e. consumed t.  Tags are t+1; every rank clears its buffer at the start of a
// solve, followed by a barrier, before anyone publishes.
#include <cmath>
#include <cstdint>

#include "grid_common.cuh"
#include "kpp_internal.h"
#include "window.cuh"

namespace kpp {
namespace {
using namespace gx;

constexpr int NT = 512, NW = NT / 32, RW = 8, YR = 8, DC = 2, TW = 32 * DC;

// Sorted S: position of global column gj, or -1.
__device__ __forceinline__ int find_sorted(const int32_t* S, int s, long long gj) {
  int lo = 0, hi = s - 1;
  while (lo <= hi) {
    const int mid = (lo + hi) >> 1;
    const long long v = S[mid];
    if (v == gj) return mid;
    if (v < gj) lo = mid + 1;
    else hi = mid - 1;
  }
  return -1;
}

__device__ __forceinline__ void cp_async8(void* smem, const void* g) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(g) : "memory");
}
// Copy the CTA's slab of A_S (rows S, columns [c0, c1)) into dst (row stride sl), asynchronously.
__device__ __forceinline__ void prefetch_slab(const XParams& p, const int32_t* S, double* dst, long long c0,
                                              long long c1) {
  const int w = (int)(c1 - c0);
  if (w <= 0) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int k = warp; k < p.s; k += NW) {  // a warp per row, lanes across the slab (no divisions)
    const double* src = p.A + (long long)S[k] * p.lda + c0;
    double* d = dst + (long long)k * p.sl;
    for (int c = lane; c < w; c += 32) cp_async8(d + c, src + c);
  }
  asm volatile("cp.async.commit_group;\n" ::: "memory");
}

// MODE 0: A_S from global; 1: from global, filling As; 2: from As (prefetched)
template <int MODE>
__device__ __forceinline__ void rowsums(const XParams& p, const int32_t* S_sh, double* As, long long c0, long long c1,
                                        unsigned long long* ll_part, unsigned tag, int g) {
  const int s = p.s, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int k0 = warp * RW; k0 < s; k0 += NW * RW) {
    double acc[RW];
    const double* rows[RW];
#pragma unroll
    for (int r = 0; r < RW; ++r) {
      acc[r] = 0.0;
      const int kr = k0 + r < s ? k0 + r : k0;
      rows[r] = MODE == 2 ? As + (long long)kr * p.sl - c0 : p.A + (long long)S_sh[kr] * p.lda;
    }
#pragma unroll 2
    for (long long j = c0 + lane; j < c1; j += 32) {
      const double xj = p.x[j];
#pragma unroll
      for (int r = 0; r < RW; ++r)
        if (k0 + r < s) {
          const double a = rows[r][j];
          if (MODE == 1) As[(long long)(k0 + r) * p.sl + (j - c0)] = a;
          acc[r] = fma(a, xj, acc[r]);
        }
    }
    const double tot = warp_multi_sum<RW>(acc);
    const int r = warp_multi_index<RW>();
    if ((lane & (32 / RW - 1)) == 0 && k0 + r < s) ll_put(ll_part + 2LL * ((long long)g * s + k0 + r), tot, tag);
  }
}

// MS: M staged in shared memory (p.m_smem) as a template parameter, so that the y products read it
// with shared-memory loads rather than generic ones
template <bool MS>
__global__ void __launch_bounds__(NT, 1) xeng_kernel(XParams p) {
  extern __shared__ double sm[];
  __shared__ DevState st_sh;
  __shared__ double red_sh[128];
  int bs = 0;
  const int s = p.s, SP = (s + 31) & ~31, G = p.grid, R = p.nranks;
  double* tot = sm;  // r
  double* bS = tot + SP;
  double* yv = bS + SP;
  double(*part_sh)[TW] = reinterpret_cast<double(*)[TW]>(yv + SP);
  int32_t* S_sh = reinterpret_cast<int32_t*>(yv + SP + NW * TW);
  int32_t* Sn_sh = S_sh + SP;  // the next block's rows (prefetch mode)
  double* As0 = yv + SP + NW * TW + SP;
  double* As1 = As0 + (p.a_smem == 2 ? (long long)s * p.sl : 0);
  double* Ms = As1 + (p.a_smem ? (long long)s * p.sl : 0);
  // virtual rank vr of this CTA (one rank per launch unless emulated, see XParams::vranks)
  const int vr = (int)blockIdx.x / G;
  const int rank = p.rank + vr;
  const bool lead = vr == 0;  // the CTAs of the first rank of the launch write the shared state
  unsigned long long* llr = p.ll + (long long)vr * 2LL * ((long long)G * s + s);
  unsigned long long* ll_y = llr + 2LL * G * s;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = (int)blockIdx.x - vr * G;
  const long long cr1 = p.vcol[vr + 1];
  const long long c0 = min(p.vcol[vr] + (long long)g * p.slab, cr1);
  const long long c1 = (c0 + p.slab < cr1) ? c0 + p.slab : cr1;
  if (tid == 0) st_sh = *p.st;
  int cur = 0;
  if (p.a_smem == 2 && p.t0 < p.t1) {  // prefetch mode: the first block of the window, synchronously
    const long long kb0 = p.bid[0];
    for (int i = tid; i < s; i += NT) Sn_sh[i] = p.S_pool[kb0 * s + i];
    __syncthreads();
    prefetch_slab(p, Sn_sh, As0, c0, c1);
    asm volatile("cp.async.wait_all;\n" ::: "memory");
  }
  __syncthreads();
  long long tm = p.t0 % (2 * p.zeta);
  const bool prof = p.prof != nullptr && g == 0 && lead && tid == 0;
  long long tp = prof ? clock64() : 0;
  long long pr[6] = {0, 0, 0, 0, 0, 0};
  auto mark = [&](int i) {
    if (prof) {
      const long long now = clock64();
      pr[i] += now - tp;
      tp = now;
    }
  };
  for (long long t = p.t0; t < p.t1; ++t) {
    if (st_sh.stopped) break;
    const long long kb = p.bid[t - p.t_base];
    const double* Mg = p.M_pool + kb * (long long)s * s;
    if constexpr (MS) {  // asynchronous copy, overlapped with (a) and (b)
      const long long nm = (long long)s * s;
      for (long long i = 2LL * tid; i < nm; i += 2LL * NT) cp_async16(Ms + i, Mg + i);
      asm volatile("cp.async.commit_group;\n" ::: "memory");
    }
    const double* M = MS ? Ms : Mg;
    for (int i = tid; i < s; i += NT) {
      const int32_t row = p.S_pool[kb * s + i];
      S_sh[i] = row;
      bS[i] = p.b[row];
    }
    __syncthreads();
    const unsigned tag = (unsigned)(t + 1);
    double* As = cur ? As1 : As0;
    // (a)
    if (p.a_smem == 2) rowsums<2>(p, S_sh, As, c0, c1, llr, tag, g);
    else if (p.a_smem == 1) rowsums<1>(p, S_sh, As, c0, c1, llr, tag, g);
    else rowsums<0>(p, S_sh, As, c0, c1, llr, tag, g);
    mark(0);
    auto issue_prefetch = [&]() {  // the next block's slab streams in behind this iteration
      if (p.a_smem == 2 && t + 1 < p.t1) {
        const long long kbn = p.bid[t + 1 - p.t_base];
        for (int i = tid; i < s; i += NT) Sn_sh[i] = p.S_pool[kbn * s + i];
        __syncthreads();
        prefetch_slab(p, Sn_sh, cur ? As0 : As1, c0, c1);
      }
    };
    if (p.pf_at == 0) issue_prefetch();
    // (b) grid reduce by the owner warps, publish to every rank, gather
    const long long slot = (long long)(t & 1) * R * s;
    for (int k = g + warp * G; k < s; k += NW * G) {
      double a = 0.0;
      for (int q0 = lane; q0 < G; q0 += 32 * 8) a += ll_sum<8>(llr + 2LL * k, 2LL * s, q0, G, tag, p.err);
      a = wsum(a);
      // system scope: the destination may be a peer GPU's memory (one rank runs the same code)
      if (lane < R) ll_put_sys(p.peer_recv[lane] + 2 * (slot + (long long)rank * s + k), a, tag);
    }
    double e = 0.0;
    for (int k = tid; k < s; k += NT) {
      double v = 0.0;
      for (int r = 0; r < R; ++r) {
        v += ll_get_sys(p.peer_recv[rank] + 2 * (slot + (long long)r * s + k), tag, p.err);
      }
      const double rk = v - bS[k];
      tot[k] = rk;
      e = fma(rk, rk, e);
    }
    if constexpr (MS) asm volatile("cp.async.wait_all;\n" ::: "memory");
    e = block_sum(e, red_sh, bs);  // (its barrier publishes r and the staged M)
    mark(1);
    if (p.pf_at == 1) issue_prefetch();
    // (d) y = M r.  M staged in shared memory: every CTA computes all of y; else the rows are spread
    // over the grid (row k by CTA k mod grid) and gathered through L2 like (b)
    if (!MS) {
      for (int k = g + warp * G; k < s; k += NW * G) {
        const double* Mrow = M + (long long)k * s;
        double a = 0.0;
#pragma unroll 4
        for (int l = lane; l < s; l += 32) a = fma(Mrow[l], tot[l], a);
        a = wsum(a);
        if (lane == 0) ll_put(ll_y + 2LL * k, a, tag);
      }
      for (int k = tid; k < s; k += NT) yv[k] = ll_sum<1>(ll_y + 2LL * k, 0, 0, 1, tag, p.err);
    }
    for (int r0 = warp * YR; MS && r0 < s; r0 += NW * YR) {
      double a[YR];
#pragma unroll
      for (int r = 0; r < YR; ++r) a[r] = 0.0;
      for (int l = lane; l < s; l += 32) {
        const double rl = tot[l];
#pragma unroll
        for (int r = 0; r < YR; ++r)
          if (r0 + r < s) a[r] = fma(M[(long long)(r0 + r) * s + l], rl, a[r]);
      }
      const double y = warp_multi_sum<YR>(a);
      const int row = r0 + warp_multi_index<YR>();
      if ((lane & (32 / YR - 1)) == 0 && row < s) yv[row] = y;
    }
    __syncthreads();
    mark(2);
    if (p.pf_at == 2) issue_prefetch();
    // (e) w on the slab, momentum, x
    const double rho = st_sh.rho, cm = (1.0 - rho) / (1.0 + rho);
    if (!p.cd) {
      for (long long jb = c0; jb < c1; jb += TW) {
        double acc[DC];
#pragma unroll
        for (int c = 0; c < DC; ++c) acc[c] = 0.0;
#pragma unroll 4
        for (int k = warp; k < s; k += NW) {
          const double* row = p.a_smem ? As + (long long)k * p.sl - c0 : p.A + (long long)S_sh[k] * p.lda;  // current slab
          const double yk = yv[k];
#pragma unroll
          for (int c = 0; c < DC; ++c) {
            const long long j = jb + c * 32 + lane;
            if (j < c1) acc[c] = fma(row[j], yk, acc[c]);
          }
        }
#pragma unroll
        for (int c = 0; c < DC; ++c) part_sh[warp][c * 32 + lane] = acc[c];
        __syncthreads();
        if (tid < TW) {
          const long long j = jb + tid;
          if (j < c1) {
            double h0 = 0.0, h1 = 0.0;
#pragma unroll
            for (int w = 0; w < NW; w += 2) {
              h0 += part_sh[w][tid];
              h1 += part_sh[w + 1][tid];
            }
            const double wj = h0 + h1;
            const double mm = cm * (p.mom[j] - wj);
            p.mom[j] = mm;
            p.x[j] = p.x[j] - wj + p.eta * mm;
          }
        }
        __syncthreads();
      }
    } else {
      for (long long j = c0 + tid; j < c1; j += NT) {
        const int pos = find_sorted(S_sh, s, p.col_base + j);
        const double wj = pos >= 0 ? yv[pos] : 0.0;
        const double mm = cm * (p.mom[j] - wj);
        p.mom[j] = mm;
        p.x[j] = p.x[j] - wj + p.eta * mm;
      }
    }
    mark(3);
    // (f)
    __syncthreads();
    if (tid == 0) {
      const int res = window_step_dev(st_sh, tm, e, p.zeta, p.tol2bb, p.bb, p.adaptive, p.writer && g == 0 && lead,
                                      p.hist_res, p.hist_rho, p.hist_cap);
      if (res) st_sh.stopped = res;
      st_sh.t_done = t + 1;
    }
    if (++tm == 2 * p.zeta) tm = 0;
    if (p.a_smem == 2) {
      asm volatile("cp.async.wait_all;\n" ::: "memory");
      cur ^= 1;
    }
    __syncthreads();
    mark(4);
  }
  if (g == 0 && lead && tid == 0) *p.st = st_sh;
  if (prof)
    for (int i = 0; i < 6; ++i) p.prof[i] += pr[i];
}

}  // namespace

size_t xeng_smem_bytes(int s, int a_smem, int sl, int m_smem) {
  const int SP = (s + 31) & ~31;
  size_t d = (size_t)(3 * SP + NW * TW + SP);
  d += (size_t)a_smem * s * sl;  // 1: one slab buffer, 2: double-buffered (prefetch)
  if (m_smem) d += (size_t)s * s;
  return d * sizeof(double);
}

size_t xeng_ll_words(int s, int grid) { return 2 * ((size_t)grid * s + s); }

cudaError_t launch_xeng_window(cudaStream_t st, const XParams& p) {
  static int attr_smem[2] = {0, 0};
  const int ms = p.m_smem ? 1 : 0;
  const void* fn = ms ? (const void*)xeng_kernel<true> : (const void*)xeng_kernel<false>;
  const size_t smem = xeng_smem_bytes(p.s, p.a_smem, p.sl, p.m_smem);
  if ((int)smem > attr_smem[ms]) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr_smem[ms] = (int)smem;
  }
  if (p.nranks > KPP_MAX_PEERS || p.nranks > 32 || p.vranks < 1 || p.rank + p.vranks > p.nranks)
    return cudaErrorInvalidValue;
  cudaError_t e = cudaMemsetAsync(p.ll, 0, (size_t)p.vranks * xeng_ll_words(p.s, p.grid) * sizeof(unsigned long long), st);
  if (e != cudaSuccess) return e;
  XParams q = p;
  void* args[] = {&q};
  e = cudaLaunchCooperativeKernel(fn, dim3(p.grid * p.vranks), dim3(NT), args, smem, st);
  count_launches(1);
  return e;
}

}  // namespace kpp
