// iterate.cu -- Phase 2: the per-iteration memoized block update.
//
// For each iteration t of a window (Alg 5 l.9-18 P:1346-1357 / Alg 3 l.10-20 P:755-766):
//   r   = A_S x - b_S                                        (row 3)
//   y   = M r,  M = (A_S A_S^T + lam I)^{-1}  memoized (K++)  / (A_SS + lam I)^{-1} (CD++)  (row 4)
//   w   = A_S^T y (K++, Eq (bk))  |  I_S^T y (CD++, Alg 3 l.11)            (row 5)
//   m   = (1-rho)/(1+rho) (m - w);  x = x - w + eta m        (row 6, Eq (momentum))
//   E0/E1 window sums; checkpoint every 2 zeta: stop test, adaptive rho   (row 8)
//
// Engine "persistent" (one launch per window, one CTA per SM, thread-block clusters of C CTAs):
//  * CTA g owns the column slab [g*slab, (g+1)*slab) of A, x and m; x and m live in shared
//    memory for the whole launch.
//  * Resident mode (the s x slab block fits on chip): the slab of the NEXT block is copied
//    HBM -> shared memory with cp.async while the current iteration runs (the schedule is
//    data independent, so block t+1 is known); both passes (A_S x and A_S^T y) read shared
//    memory, and A_S crosses HBM once per iteration.  Streaming mode (c4/c5-sized blocks):
//    both passes stream from HBM/L2 with 16-byte loads.
//  * Exchange of the s-vector partials: inside a cluster through distributed shared memory
//    (DSMEM); across clusters CTA rank c of every cluster owns row slice c of the s-vector,
//    writes its cluster's partial of that slice to global memory and waits on a per-slice
//    arrival counter -- C independent barriers of G/C CTAs instead of one grid barrier.
//    Each slice owner then forms r for its slice (fixed summation order), all-gathers r in
//    the cluster (DSMEM), computes its slice of y = M r from a shared-memory copy of its M
//    rows (prefetched for the next block), and all-gathers y.  Every CTA ends up with the
//    identical r and y, so the scalar window logic is replicated bit-for-bit and no CTA
//    needs to broadcast a decision.  No floating-point atomics: runs are bit-reproducible.
#include <cooperative_groups.h>

#include <cmath>
#include <cstdint>

#include "kpp_internal.h"
#include "window.cuh"

namespace cg = cooperative_groups;

namespace kpp {
namespace {

constexpr int T2 = 512;
constexpr int NW2 = T2 / 32;

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

__device__ __forceinline__ void red_release_add(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ void cp_async16(void* smem, const void* g) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async8(void* smem, const void* g) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

// Copy rows S[0..s) x columns [c0, c0+w) of A into dst (row stride sw doubles) with cp.async:
// warp per row, lanes over 16-byte chunks (8-byte chunks when the row is not 16-byte aligned).
__device__ __forceinline__ void prefetch_slab(const double* A, long long lda, const int32_t* S_sh, int s,
                                              long long c0, int w, double* dst, int sw) {
  if (w <= 0) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool vec = ((lda & 1) == 0) && ((c0 & 1) == 0) && ((w & 1) == 0) && ((sw & 1) == 0) &&
                   ((reinterpret_cast<uintptr_t>(A) & 15) == 0);
  if (vec) {
    const int hw = w >> 1;  // 16-byte chunks per row
    for (int k = warp; k < s; k += T2 / 32) {
      const double* src = A + (long long)S_sh[k] * lda + c0;
      double* d = dst + (long long)k * sw;
      for (int j = lane; j < hw; j += 32) cp_async16(d + 2 * j, src + 2 * j);
    }
  } else {
    for (int k = warp; k < s; k += T2 / 32) {
      const double* src = A + (long long)S_sh[k] * lda + c0;
      double* d = dst + (long long)k * sw;
      for (int j = lane; j < w; j += 32) cp_async8(d + j, src + j);
    }
  }
}

__device__ __forceinline__ void prefetch_rows(const double* src, int count, double* dst) {
  const bool vec = ((reinterpret_cast<uintptr_t>(src) & 15) == 0) && ((count & 1) == 0);
  if (vec) {
    for (int e = threadIdx.x * 2; e < count; e += 2 * T2) cp_async16(dst + e, src + e);
  } else {
    for (int e = threadIdx.x; e < count; e += T2) cp_async8(dst + e, src + e);
  }
}

__device__ __forceinline__ void spin_until(const unsigned* cnt, unsigned target, int* err_flag) {
  const unsigned long long t0 = globaltimer();
  unsigned it = 0;
  while (ld_acquire(cnt) < target) {
    if ((++it & 1023u) == 0 && globaltimer() - t0 > 20000000000ull) {  // 20 s: co-residency lost
      atomicExch(err_flag, 1);
      __trap();
    }
  }
}

// Optional phase timers (CTA 0, thread 0): cumulative clock64 cycles per phase -> p.prof[8].
#define PHASE_MARK(i)                                   \
  do {                                                  \
    if (prof_on) {                                      \
      const long long now_ = clock64();                 \
      prof_acc[i] += now_ - prof_last;                  \
      prof_last = now_;                                 \
    }                                                   \
  } while (0)

__global__ void __launch_bounds__(T2, 1) iterate_kernel(IterParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int s = p.s;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  cg::cluster_group cluster = cg::this_cluster();
  const int C = (int)cluster.num_blocks();
  const int c = (int)cluster.block_rank();
  const int q = blockIdx.x / C;   // cluster index
  const int NQ = gridDim.x / C;   // clusters
  // slice of the s-vector owned by this rank
  const int sl = (s + C - 1) / C;
  const int r0 = min(s, c * sl), r1 = min(s, r0 + sl);

  // ---- shared memory carve-up (must match iterate_smem_bytes) ----
  const int sp = (s + 1) & ~1;
  const int wpad = p.slab;  // multiple of 4
  double* x_sm = reinterpret_cast<double*>(smem_raw);
  double* m_sm = x_sm + wpad;
  double* w_sm = m_sm + wpad;
  double* part_sm = w_sm + wpad;
  double* r_sm = part_sm + sp;
  double* y_sm = r_sm + sp;
  double* red_sm = y_sm + sp;                                      // [T2] column-partial scratch
  int32_t* S_sh = reinterpret_cast<int32_t*>(red_sm + T2);         // [2][sp]
  double* Msl = reinterpret_cast<double*>(S_sh + 2 * sp);          // [sl][s] if m_in_smem
  double* Abuf = Msl + (p.m_in_smem ? (((long long)sl * s + 1) & ~1LL) : 0);  // [2][s][sw] if resident (16B aligned)
  const long long absz = (long long)s * p.sw;
  __shared__ DevState st;
  __shared__ int stop_sh;

  const long long c0 = (long long)blockIdx.x * p.slab;
  const long long c1 = (c0 + p.slab < p.n) ? c0 + p.slab : p.n;
  const int w = (int)(c1 > c0 ? c1 - c0 : 0);

  if (tid == 0) {
    st = *p.st;
    stop_sh = 0;
  }
  for (int j = tid; j < w; j += T2) {
    x_sm[j] = p.x[c0 + j];
    m_sm[j] = p.mom[c0 + j];
  }
  // prefetch the first block (index set, slab, M slice)
  {
    const long long k0 = p.bid[0];
    for (int i = tid; i < s; i += T2) S_sh[i] = p.S_pool[k0 * s + i];
    __syncthreads();
    if (p.resident) prefetch_slab(p.A, p.lda, S_sh, s, c0, w, Abuf, p.sw);
    if (p.m_in_smem && r1 > r0)
      prefetch_rows(p.M_pool + k0 * (long long)s * s + (long long)r0 * s, (r1 - r0) * s, Msl);
    cp_async_commit();
  }
  cluster.sync();  // peers' shared memory is live before any DSMEM access

  const bool prof_on = p.prof != nullptr && blockIdx.x == 0 && threadIdx.x == 0;
  long long prof_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long prof_last = prof_on ? clock64() : 0;
  long long t = p.t0;
  unsigned it = 0;
  for (; t < p.t1; ++t, ++it) {
    const int buf = it & 1;
    const int32_t* Sc = S_sh + buf * sp;
    const long long kb = p.bid[t - p.t0];
    const double* Mg = p.M_pool + kb * (long long)s * s;
    cp_async_wait_all();
    __syncthreads();
    PHASE_MARK(0);  // wait for this iteration's prefetched slab + previous iteration tail
    const double rho = st.rho;  // set at the last checkpoint strictly before t (reading Q11)
    // ---- prefetch block t+1 (index set, then its slab) into the other buffer
    if (t + 1 < p.t1) {
      const long long kn = p.bid[t + 1 - p.t0];
      int32_t* Sn = S_sh + (buf ^ 1) * sp;
      for (int i = tid; i < s; i += T2) Sn[i] = p.S_pool[kn * s + i];
      if (p.resident) {
        __syncthreads();
        prefetch_slab(p.A, p.lda, Sn, s, c0, w, Abuf + (buf ^ 1) * absz, p.sw);
        cp_async_commit();
      }
    }
    const double* Ac = Abuf + buf * absz;
    PHASE_MARK(1);  // issue of the next prefetch

    // ---- row 3: partial block residual over the slab -> part_sm[k]
    if (p.resident) {
      // tpr threads per row, rows in passes of T2/tpr
      const int tpr = p.tpr;
      const int rows_per_pass = T2 / tpr;
      const int sub = tid & (tpr - 1);
      for (int kp = 0; kp < s; kp += rows_per_pass) {
        const int k = kp + tid / tpr;
        double acc = 0.0;
        if (k < s) {
          const double* arow = Ac + (long long)k * p.sw;
          for (int j = sub; j < w; j += tpr) acc = fma(arow[j], x_sm[j], acc);
        }
        for (int o = tpr >> 1; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (k < s && sub == 0) part_sm[k] = acc;
      }
    } else {
      // streaming: warp per row, 4 rows in flight, 16-byte loads when aligned
      const bool vec = ((p.lda & 1) == 0) && ((c0 & 1) == 0);
      for (int kbase = warp * 4; kbase < s; kbase += NW2 * 4) {
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
        const double* rows[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int k = min(kbase + u, s - 1);
          rows[u] = p.A + (long long)Sc[k] * p.lda + c0;
        }
        if (vec) {
          const int w2 = w >> 1;
          for (int j2 = lane; j2 < w2; j2 += 32) {
            const double2 xv = *reinterpret_cast<const double2*>(x_sm + 2 * j2);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const double2 a = __ldcs(reinterpret_cast<const double2*>(rows[u]) + j2);
              acc[u] = fma(a.x, xv.x, acc[u]);
              acc[u] = fma(a.y, xv.y, acc[u]);
            }
          }
          if ((w & 1) && lane == 0) {
#pragma unroll
            for (int u = 0; u < 4; ++u) acc[u] = fma(__ldcs(rows[u] + w - 1), x_sm[w - 1], acc[u]);
          }
        } else {
          for (int j = lane; j < w; j += 32) {
            const double xv = x_sm[j];
#pragma unroll
            for (int u = 0; u < 4; ++u) acc[u] = fma(__ldcs(rows[u] + j), xv, acc[u]);
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const double v = warp_sum(acc[u]);
          if (lane == 0 && kbase + u < s) part_sm[kbase + u] = v;
        }
      }
    }
    PHASE_MARK(2);  // row 3 (A_S x partials)
    cluster.sync();  // [A] every rank's part_sm is complete

    // ---- cluster partial of my slice -> global (double-buffered by parity), arrive, wait
    double* pcl = p.part + (long long)(it & 1) * NQ * s;
    for (int kk = r0 + tid; kk < r1; kk += T2) {
      double v = 0.0;
      for (int cc = 0; cc < C; ++cc) v += *cluster.map_shared_rank(part_sm + kk, cc);
      pcl[(long long)q * s + kk] = v;
    }
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      PHASE_MARK(3);  // cluster barrier A + cluster partial of the slice
      red_release_add(p.cnt + c, 1u);
      spin_until(p.cnt + c, (it + 1) * (unsigned)NQ, p.err);
      PHASE_MARK(4);  // cross-cluster arrival wait
    }
    __syncthreads();
    // ---- r for my slice: fixed-order sum over clusters, minus b_S; all-gather in the cluster.
    // Every (row, cluster-group) pair loads at once; groups are then summed in a fixed order.
    const int R = r1 - r0;
    if (R > 0) {
      const int G2 = R <= T2 ? T2 / R : 1;
      for (int e = tid; e < R * G2 && e < T2; e += T2) {
        const int row = e % R, grp = e / R;
        double v = 0.0;
        for (int qq = grp; qq < NQ; qq += G2) v += __ldcg(pcl + (long long)qq * s + r0 + row);
        red_sm[grp * R + row] = v;
      }
      if (R > T2) {  // very large slices (s > T2 * C): one thread per row, all clusters
        for (int row = tid; row < R; row += T2) {
          double v = 0.0;
          for (int qq = 0; qq < NQ; qq += 1) v += __ldcg(pcl + (long long)qq * s + r0 + row);
          r_sm[r0 + row] = v;  // local staging; subtract b and scatter below
        }
      }
      __syncthreads();
      for (int row = tid; row < R; row += T2) {
        double v;
        if (R <= T2) {
          v = 0.0;
          for (int grp = 0; grp < G2; ++grp) v += red_sm[grp * R + row];
        } else {
          v = r_sm[r0 + row];
        }
        v -= p.b[Sc[r0 + row]];
        for (int cc = 0; cc < C; ++cc) *cluster.map_shared_rank(r_sm + r0 + row, cc) = v;
      }
    }
    cluster.sync();  // [B] r complete everywhere
    PHASE_MARK(5);  // r slice gather + all-gather + barrier B
    // ---- row 4: my slice of y = M r (tq threads per row, shuffle-combined); all-gather
    if (R > 0) {
      int tq = 1;
      while (tq < 32 && tq * 2 * R <= T2) tq *= 2;
      const int rows_per_pass = T2 / tq;
      const int sub = tid & (tq - 1);
      for (int rp = 0; rp < R; rp += rows_per_pass) {
        const int row = rp + tid / tq;
        double v = 0.0;
        if (row < R) {
          const double* Mrow = p.m_in_smem ? Msl + (long long)row * s : Mg + (long long)(r0 + row) * s;
          for (int l = sub; l < s; l += tq) v = fma(Mrow[l], r_sm[l], v);
        }
        for (int o = tq >> 1; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (row < R)
          for (int cc = sub; cc < C; cc += tq) *cluster.map_shared_rank(y_sm + r0 + row, cc) = v;
      }
    }
    cluster.sync();  // [C] y complete everywhere
    PHASE_MARK(6);  // y slice + all-gather + barrier C
    // M slice of block t+1 into shared memory (mine is consumed)
    if (p.m_in_smem && t + 1 < p.t1 && r1 > r0) {
      const long long kn = p.bid[t + 1 - p.t0];
      prefetch_rows(p.M_pool + kn * (long long)s * s + (long long)r0 * s, (r1 - r0) * s, Msl);
      cp_async_commit();
    }

    // ---- rows 5-6: w on the slab, momentum, x
    const double cm = (1.0 - rho) / (1.0 + rho);
    if (!p.cd) {
      if (p.resident) {
        // ng groups of cw threads: group g sums rows [g*rg, (g+1)*rg) of column j; then a
        // fixed-order sum over the groups (w <= cw is guaranteed by the host)
        const int cw = p.cw, ng = T2 / cw, rg = (s + ng - 1) / ng;
        const int g = tid / cw, j = tid - g * cw;
        const int ka = min(s, g * rg), kz = min(s, ka + rg);
        double a = 0.0;
        if (j < w)
          for (int k = ka; k < kz; ++k) a = fma(Ac[(long long)k * p.sw + j], y_sm[k], a);
        red_sm[g * cw + j] = a;
        __syncthreads();
        for (int jj = tid; jj < w; jj += T2) {
          double v = 0.0;
          for (int gg = 0; gg < ng; ++gg) v += red_sm[gg * cw + jj];
          w_sm[jj] = v;
        }
      } else {
        for (int jj = tid; jj < w; jj += T2) {
          double a = 0.0;
          const double* col = p.A + c0 + jj;
#pragma unroll 8
          for (int k = 0; k < s; ++k) a = fma(__ldcg(col + (long long)Sc[k] * p.lda), y_sm[k], a);
          w_sm[jj] = a;
        }
      }
    } else {
      for (int jj = tid; jj < w; jj += T2) w_sm[jj] = 0.0;
      __syncthreads();
      for (int k = tid; k < s; k += T2) {
        const long long gj = (long long)Sc[k] - p.col_base;
        if (gj >= c0 && gj < c1) w_sm[gj - c0] = y_sm[k];
      }
    }
    __syncthreads();
    for (int jj = tid; jj < w; jj += T2) {
      const double wv = w_sm[jj];
      const double mm = cm * (m_sm[jj] - wv);
      m_sm[jj] = mm;
      x_sm[jj] = x_sm[jj] - wv + p.eta * mm;
    }
    // ---- row 8: ||r||^2 (fixed order, identical in every CTA) and the window logic
    if (warp == 0) {
      double e = 0.0;
      for (int i = lane; i < s; i += 32) e = fma(r_sm[i], r_sm[i], e);
      e = warp_sum(e);
      if (lane == 0) {
        const int res = window_step_dev(st, t, e, p.zeta, p.tol2bb, p.bb, p.adaptive,
                                        blockIdx.x == 0 && p.writer, p.hist_res, p.hist_rho,
                                        p.hist_cap);
        if (res) {
          st.stopped = res;
          stop_sh = 1;
        }
      }
    }
    __syncthreads();
    PHASE_MARK(7);  // rows 5-6 (A_S^T y, momentum) + window logic
    if (stop_sh) {
      ++t;
      break;
    }
  }
  if (prof_on)
    for (int i = 0; i < 8; ++i) p.prof[i] += prof_acc[i];
  cp_async_wait_all();
  for (int j = tid; j < w; j += T2) {
    p.x[c0 + j] = x_sm[j];
    p.mom[c0 + j] = m_sm[j];
  }
  if (blockIdx.x == 0 && tid == 0) {
    st.t_done = t;
    *p.st = st;
  }
  cluster.sync();  // keep shared memory alive until every peer is done with DSMEM
}

}  // namespace

int iterate_block_threads() { return T2; }

size_t iterate_smem_bytes(const IterParams& p, int C) {
  const int s = p.s;
  const int sp = (s + 1) & ~1;
  const int sl = (s + C - 1) / C;
  size_t bytes = 0;
  bytes += 3ull * p.slab * sizeof(double);
  bytes += 3ull * sp * sizeof(double);
  bytes += (size_t)T2 * sizeof(double);
  bytes += 2ull * sp * sizeof(int32_t);
  if (p.m_in_smem) bytes += (size_t)(((long long)sl * s + 1) & ~1LL) * sizeof(double);
  if (p.resident) bytes += 2ull * s * p.sw * sizeof(double);
  return bytes + 64;
}

static void set_attrs(size_t smem, int C) {
  cudaFuncSetAttribute(iterate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (C > 8) cudaFuncSetAttribute(iterate_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
}

cudaError_t launch_iterate(cudaStream_t stream, const IterParams& p, int grid, int C, size_t smem) {
  set_attrs(smem, C);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(T2);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  count_launches(1);
  return cudaLaunchKernelEx(&cfg, iterate_kernel, p);
}

// Largest number of co-resident clusters of size C at this shared-memory size.
int iterate_max_clusters(int C, size_t smem) {
  set_attrs(smem, C);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C * 256);
  cfg.blockDim = dim3(T2);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, iterate_kernel, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

}  // namespace kpp
