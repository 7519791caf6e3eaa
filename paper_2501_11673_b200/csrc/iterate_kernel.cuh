// iterate_kernel.cuh -- Phase 2: the per-iteration memoized block update.
//
// For each iteration t of a window (Alg 5 l.9-18 P:1346-1357 / Alg 3 l.10-20 P:755-766):
//   r   = A_S x - b_S                                        (row 3)
//   y   = M r,  M = (A_S A_S^T + lam I)^{-1}  memoized (K++)  / (A_SS + lam I)^{-1} (CD++)  (row 4)
//   w   = A_S^T y (K++, Eq (bk))  |  I_S^T y (CD++, Alg 3 l.11)            (row 5)
//   m   = (1-rho)/(1+rho) (m - w);  x = x - w + eta m        (row 6, Eq (momentum))
//   E0/E1 window sums; checkpoint every 2 zeta: stop test, adaptive rho   (row 8)
//
// Engine "persistent": one launch per window, one CTA per SM, thread-block clusters of C CTAs.
//  * CTA g owns the column slab [g*slab, (g+1)*slab) of A, x and m; x and m stay in shared
//    memory for the whole launch.
//  * Resident mode (the s x slab block fits on chip): the block schedule is data independent,
//    so while iteration t runs, the TMA engine (cp.async.bulk, one bulk copy per row segment,
//    completion on an mbarrier) brings the slab of block t+1 into the other half of a
//    double buffer, and the M rows this CTA needs for t+1 into a staging buffer.  Both
//    passes (A_S x and A_S^T y) read shared memory and A_S crosses HBM once per iteration.
//    Streaming mode (c4/c5-sized blocks): both passes stream 16-byte loads from HBM/L2.
//  * The one all-reduce of the iteration (the s-vector A_S x) is a barrier-free dataflow
//    exchange.  Inside a cluster values move by st.async (DSMEM stores that complete bytes on
//    the receiver's mbarrier, so the receiver sleeps on its barrier instead of polling);
//    across clusters through L2 as two 8-byte words, each carrying 32 data bits and a 32-bit
//    iteration tag (the "LL" protocol of NCCL): an 8-byte store is single-copy atomic, so a
//    consumer that sees the current tag has the data -- no flag round trip.
//      partials --st.async--> slice owner in the cluster (rank c owns rows slice c)
//      cluster partial of the slice --L2 (LL)--> the slice owners of every cluster
//      r slice (fixed-order sum, - b_S) --st.async--> every CTA of the cluster
//      y slice = M[slice] r --st.async--> every CTA of the cluster
//    Every CTA then holds identical r and y, so the scalar window logic is replicated
//    bit-for-bit and nobody broadcasts a decision.  No floating-point atomics anywhere.
#pragma once
#include "kernel_common.cuh"

namespace kpp {
namespace itk {

// Register tile of the resident A_S x / A_S^T y passes: warp wi holds rows wi + 16 i (i < RPW),
// lane l holds columns l + 32 c (c < CPL).  RPW = 0: shared-memory path.
// Compile-time mode (each launch plan runs an instantiation holding only its own code: the loop
// body must stay within the instruction caches -- a 240 KB all-modes kernel was i-cache bound):
//   RES  1: block slab resident in shared memory (TMA-prefetched), 0: streamed from HBM
//   YG   where y = M r is computed: 0 per cluster from staged M rows (DSMEM all-gather of y),
//        1 once per GPU (rows spread over all CTAs, LL all-gather through L2),
//        4 per cluster as the sum of the ranks' partials M[slice,:]^T r_slice (no all-gather of r)
//   CDT  1: CD++ (w = I_S^T y), 0: K++ (w = A_S^T y)
template <int RES, int RPW, int CPL, int YG, int CDT>
__global__ void __launch_bounds__(T2, 1) iterate_kernel(const __grid_constant__ IterParams p) {
  static_assert(RES || RPW == 0, "register tile needs the resident slab");
  constexpr bool yred = YG == 4;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int s = p.s;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  cg::cluster_group cluster = cg::this_cluster();
  const int C = (int)cluster.num_blocks();
  const int c = (int)cluster.block_rank();
  // rank of this CTA: several ranks per launch when emulated (IterParams::vranks), cluster boundaries
  // align with them; with one rank per launch vr = 0 and gb = blockIdx.x
  const int gpr = (int)gridDim.x / p.vranks;
  const int vr = (int)blockIdx.x / gpr, gb = (int)blockIdx.x - vr * gpr;
  const int rank = p.rank + vr, P = p.nranks;
  const bool lead = vr == 0;
  const int q = gb / C;             // cluster index within the rank
  const int NQ = gpr / C;           // clusters per rank
  const int sl = (s + C - 1) / C;  // rank cc owns rows [cc*sl, min(s, cc*sl + sl))
  const int r0 = min(s, c * sl), r1 = min(s, r0 + sl);
  const int R = r1 - r0;

  // ---- shared memory carve-up (must match iterate_smem_bytes) ----
  const int sp = (s + 1) & ~1;
  // mbarriers: [0],[1] slab buffers (TMA); [2] partials of my slice arrived; [3] r arrived;
  // [4] y arrived (the DSMEM exchanges are st.async stores completing bytes on these)
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(smem_raw);
  double* rp_sm = reinterpret_cast<double*>(bars + 8);  // [C][sl] partials of my slice, from each rank
  double* x_sm = rp_sm + ((C * sl + 1) & ~1);
  double* m_sm = x_sm + p.slab;
  double* w_sm = m_sm + p.slab;
  double* r_sm = w_sm + p.slab;
  double* y_sm = r_sm + sp;
  double* red_sm = y_sm + sp;                                   // [2*T2] reduction scratch
  double* bS_sh = red_sm + 2 * T2;                              // [3][sp] b_S of blocks t, t+1, t+2
  int32_t* S_sh = reinterpret_cast<int32_t*>(bS_sh + 3 * sp);   // [3][sp]
  // ygl 4: partial y (and ||r_slice||^2) from every rank of the cluster, [C][s+1]
  double* yp_sm = reinterpret_cast<double*>(S_sh + 3 * sp);
  unsigned char* tail = reinterpret_cast<unsigned char*>(yp_sm + (yred ? ((C * (s + 1) + 1) & ~1) : 0));
  {
    // 128-byte alignment of the TMA buffers, applied as an offset to a pointer derived from
    // smem_raw: the compiler then keeps the shared address space (LDS, not generic loads)
    const unsigned a0 = (unsigned)__cvta_generic_to_shared(tail);
    tail += ((a0 + 127u) & ~127u) - a0;
  }
  double* Abuf = reinterpret_cast<double*>(tail);               // [2][s4][sw] (128B aligned)
  const long long absz = (long long)((s + 3) & ~3) * p.sw;
  const long long mslz = ((long long)sl * s + 15) & ~15LL;
  // a_single: the register tile holds the slab during the iteration, so one shared buffer suffices
  // (block t+1 is gathered into it as soon as the tile of block t is in registers)
  const bool a_single = p.a_single != 0;
  double* Mbuf = Abuf + (RES ? (a_single ? 1 : 2) * absz : 0);  // [2][sl][s] staged rows of M
  __shared__ DevState st;
  __shared__ int stop_sh;
  __shared__ long long tmod_sh;

  const long long cr1 = p.vcol[vr + 1];
  const long long c0 = min(p.vcol[vr] + (long long)gb * p.slab, cr1);
  const long long c1 = (c0 + p.slab < cr1) ? c0 + p.slab : cr1;
  unsigned long long* const llr = p.ll + (long long)vr * p.ll_vstride;  // this rank's grid exchange
  unsigned long long* const ylr = p.yll + (long long)vr * p.ll_vstride;
  const int w = (int)(c1 > c0 ? c1 - c0 : 0);
  // TMA eligibility: 16-byte aligned row segments of a multiple of 16 bytes, aligned M slices
  const bool bulkA = ((p.lda & 1) == 0) && ((c0 & 1) == 0) && ((w & 1) == 0) && ((p.sw & 1) == 0) &&
                     ((reinterpret_cast<uintptr_t>(p.A) & 15) == 0);
  const bool bulkM = ((s & 1) == 0) && ((reinterpret_cast<uintptr_t>(p.M_pool) & 15) == 0);
  const bool bulk = (!RES || bulkA || p.tma) && (!p.m_in_smem || bulkM);
  const CUtensorMap* tm = p.tma ? &p.tmA : nullptr;
  const long long ss = (long long)s * s;
  const bool stageM = p.m_in_smem && R > 0;
  const bool m2 = p.m_in_smem == 2;  // single buffer: M rows of t+1 are loaded once y(t) is complete
  const int nops = (s + 3) >> 2;
  // bytes landing on bars[buf] per iteration: the slab (resident) + this rank's M rows (staged)
  const unsigned slab_bytes = RES ? (tm ? (unsigned)nops * 4u * (unsigned)p.sw * 8u : (unsigned)s * (unsigned)w * 8u) : 0u;
  const unsigned m_bytes = stageM ? (unsigned)(R * s) * 8u : 0u;
  const unsigned m_bytes_slab = m2 ? 0u : m_bytes;  // part of the per-buffer barrier's byte count
  // warps that issue the prefetch (the others do the slice-owner work in the same window)
  // (at most half the warps: the others must remain to issue the prefetch of block t+1)
  const int own_warps = min((R + 31) / 32, NW2 / 2);
  const int pf_tid = tid - 32 * own_warps;
  const int pf_n = T2 - 32 * own_warps;

  if (tid == 0) {
    st = *p.st;
    stop_sh = 0;
    tmod_sh = p.t0 % (2 * p.zeta);
    for (int i = 0; i < 6; ++i) mbar_init(bars + i, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  for (int j = tid; j < w; j += T2) {
    x_sm[j] = p.x[c0 + j];
    m_sm[j] = p.mom[c0 + j];
  }
  for (int i = tid; i < s; i += T2) {
    const int32_t v = p.S_pool[(long long)p.bid[0] * s + i];
    S_sh[i] = v;
    bS_sh[i] = p.b[v];
  }
  if (p.t0 + 1 < p.t1)
    for (int i = tid; i < s; i += T2) S_sh[sp + i] = p.S_pool[(long long)p.bid[1] * s + i];
  // block ids of t+1 and t+2 in registers (each loaded an iteration before it is needed)
  long long qb1 = (p.t0 + 1 < p.t1) ? p.bid[1] : 0;
  long long qb2 = (p.t0 + 2 < p.t1) ? p.bid[2] : 0;
  long long qb3 = 0;
  __syncthreads();
  if (warp == 0)  // block t0: slab + M rows on bars[0]
    issue_loads(bulk, tm, p.A, p.lda, S_sh, s, c0, w, Abuf, p.sw, RES != 0,
                stageM ? p.M_pool + (long long)p.bid[0] * ss + (long long)r0 * s : nullptr, R * s, Mbuf, bars + 0);
  cluster.sync();  // every peer's LL buffers are zeroed before any DSMEM store
  long long tmod = tmod_sh;

  const unsigned la_rp = smem_u32(rp_sm), la_r = smem_u32(r_sm), la_y = smem_u32(y_sm);
  const unsigned lb_rp = smem_u32(bars + 2), lb_r = smem_u32(bars + 3), lb_y = smem_u32(bars + 4);
  const bool prof_on = p.prof != nullptr && blockIdx.x == 0 && threadIdx.x == 0;
  long long prof_acc[16] = {};
  long long prof_last = prof_on ? clock64() : 0;
  long long t = p.t0;
  unsigned it = 0;
  unsigned phA0 = 0, phA1 = 0;  // mbarrier parities of bars[0], bars[1]
  for (; t < p.t1; ++t, ++it) {
    const int buf = it & 1;
    const int par = it & 1;
    const unsigned tag = it + 1;
    const int32_t* Sc = S_sh + (it % 3) * sp;
    const double* bSc = bS_sh + (it % 3) * sp;
    const int sb = a_single ? 0 : buf;        // slab buffer / barrier of this iteration
    const int nbf = a_single ? 0 : (buf ^ 1);  // ... of the prefetch of iteration t+1
    const double* Ac = Abuf + sb * absz;
    const double* Msl = Mbuf + (m2 ? 0 : buf * mslz);
    if constexpr (YG == 0) {
      // Measured (c2, one box, A/B): this plan runs faster with the slab and the M rows read by
      // generic loads (5.81 vs 6.05 us/iteration with LDS) -- its y step issues the M-row loads
      // next to the DSMEM stores and shuffles of the exchange; the other plans use LDS (c3 8.45 ->
      // 7.76 us).  The no-op move hides the shared address space from the compiler.
      asm volatile("mov.b64 %0, %0;" : "+l"(Msl));
      asm volatile("mov.b64 %0, %0;" : "+l"(Ac));
    }
    const bool pf = t + 1 < p.t1;
    // ---- top: this iteration's slab and M rows have landed; this thread's cp.async loads
    //      (S, b_S) of the previous iteration have landed; arm the barrier of the next buffer
    if (bulk) {
      if (sb == 0) { mbar_wait(bars + 0, phA0, 10); phA0 ^= 1u; }
      else         { mbar_wait(bars + 1, phA1, 11); phA1 ^= 1u; }
    }
    // register tile of the slab (rows wi + 16 i, columns lane + 32 c): loaded as soon as the slab
    // has landed, before the barrier (it does not depend on x)
    constexpr bool regpath = RPW > 0;  // pick_kernel guarantees s <= 16 RPW, w <= 32 CPL
    double ar[RPW > 0 ? RPW : 1][CPL > 0 ? CPL : 1];
    if constexpr (regpath) {
#pragma unroll
      for (int i = 0; i < RPW; ++i) {
        const int k = warp + 16 * i;
        const double* arow = Ac + k * p.sw;
#pragma unroll
        for (int cc = 0; cc < CPL; ++cc) ar[i][cc] = (k < s && lane + 32 * cc < w) ? arow[lane + 32 * cc] : 0.0;
      }
    }
    cp_async_wait_all();
    if (tid == 0) {
      if (pf && bulk) mbar_expect_tx(bars + nbf, slab_bytes + m_bytes_slab);
      // this iteration's DSMEM exchanges (phase `it` of bars[2..4])
      if (R > 0) mbar_expect_tx(bars + 2, (unsigned)(C * R) * 8u);
      if constexpr (!yred) mbar_expect_tx(bars + 3, (unsigned)s * 8u);
      if constexpr (YG == 0) mbar_expect_tx(bars + 4, (unsigned)s * 8u);
      if constexpr (yred) mbar_expect_tx(bars + 4, (unsigned)(C * (s + 1)) * 8u);
    }
    __syncthreads();
    PHASE_MARK(0);
    TRACE(0);
    const double rho = st.rho;  // set at the last checkpoint strictly before t (reading Q11)

    // ---- row 3: partial block residual over the slab; each value goes (LL) to its slice owner
    if constexpr (RES) {
      if constexpr (regpath) {
        // register tile: rows wi + 16 i, columns lane + 32 c, kept until the A_S^T y pass
        double xr[CPL > 0 ? CPL : 1];
#pragma unroll
        for (int cc = 0; cc < CPL; ++cc) xr[cc] = (lane + 32 * cc < w) ? x_sm[lane + 32 * cc] : 0.0;
        double v[RPW > 0 ? RPW : 1];
#pragma unroll
        for (int i = 0; i < RPW; ++i) {
          v[i] = 0.0;
#pragma unroll
          for (int cc = 0; cc < CPL; ++cc) v[i] = fma(ar[i][cc], xr[cc], v[i]);
        }
        if constexpr (RPW > 0) warp_reduce_scatter<RPW>(v, lane);
        const int k = warp + 16 * rs_row<RPW>(lane);
        if ((lane & (32 / (RPW > 0 ? RPW : 1) - 1)) == 0 && k < s) {
          const int owner = k / sl;
          st_async_f64(mapa_u32(la_rp + (unsigned)(c * sl + k - owner * sl) * 8u, owner), v[0], mapa_u32(lb_rp, owner));
        }
      } else {  // generic resident path (shared-memory rows)
        const int tpr = p.tpr;
        const int rows_per_pass = T2 / tpr;
        const int sub = tid & (tpr - 1);
        for (int kp = 0; kp < s; kp += rows_per_pass) {
          const int k = kp + tid / tpr;
          double acc = 0.0;
          if (k < s && !(p.dbg_skip & 1)) {
            const double* arow = Ac + k * p.sw;
            for (int j = sub; j < w; j += tpr) acc = fma(arow[j], x_sm[j], acc);
          }
          for (int o = tpr >> 1; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
          if (k < s && sub == 0) {
            const int owner = k / sl;
            st_async_f64(mapa_u32(la_rp + (unsigned)(c * sl + k - owner * sl) * 8u, owner), acc, mapa_u32(lb_rp, owner));
          }
        }
      }
    } else {
      // K++ reads the block twice: the first pass leaves it in L2 (normal eviction) so that the
      // reversed second pass hits L2 for the last rows; CD++ streams it once (evict-first)
      // (rows k >= keep0, ~35% of the block, with an evict_last L2 policy, the rest evict_first)
      const int keep0 = s - (s * 35) / 100;
      unsigned long long pol_first, pol_last;
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol_first));
      asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(pol_last));
      // streaming: a warp takes 2 rows at a time; each lane keeps 4 x 2 sixteen-byte loads in
      // flight (64 KB per SM) so HBM stays saturated
      const bool vec = ((p.lda & 1) == 0) && ((c0 & 1) == 0) && ((reinterpret_cast<uintptr_t>(p.A) & 15) == 0);
      constexpr int UR = 2, UQ = 8;  // latency-bound per warp: a whole row segment per round
      for (int kbase = warp * UR; kbase < s; kbase += NW2 * UR) {
        double acc[UR] = {0.0, 0.0};
        const double* rows[UR];
#pragma unroll
        for (int u = 0; u < UR; ++u) rows[u] = p.A + (long long)Sc[min(kbase + u, s - 1)] * p.lda + c0;
        if (vec) {
          const int w2 = w >> 1;
          const double2* x2 = reinterpret_cast<const double2*>(x_sm);
          for (int jb = lane; jb < w2; jb += 32 * UQ) {
            double2 a[UR][UQ], xv[UQ];
#pragma unroll
            for (int q = 0; q < UQ; ++q) {
              const int j2 = jb + 32 * q;
              xv[q] = j2 < w2 ? x2[j2] : make_double2(0.0, 0.0);
#pragma unroll
              for (int u = 0; u < UR; ++u)
                a[u][q] = j2 < w2 ? ld_pass1<CDT>(reinterpret_cast<const double2*>(rows[u]) + j2, kbase + u >= keep0 ? pol_last : pol_first) : make_double2(0.0, 0.0);
            }
#pragma unroll
            for (int q = 0; q < UQ; ++q)
#pragma unroll
              for (int u = 0; u < UR; ++u) {
                acc[u] = fma(a[u][q].x, xv[q].x, acc[u]);
                acc[u] = fma(a[u][q].y, xv[q].y, acc[u]);
              }
          }
          if ((w & 1) && lane == 0) {
#pragma unroll
            for (int u = 0; u < UR; ++u) acc[u] = fma(ld_pass1<CDT>(rows[u] + w - 1, kbase + u >= keep0 ? pol_last : pol_first), x_sm[w - 1], acc[u]);
          }
        } else {
          for (int j = lane; j < w; j += 32) {
            const double xv = x_sm[j];
#pragma unroll
            for (int u = 0; u < UR; ++u) acc[u] = fma(ld_pass1<CDT>(rows[u] + j, kbase + u >= keep0 ? pol_last : pol_first), xv, acc[u]);
          }
        }
#pragma unroll
        for (int u = 0; u < UR; ++u) {
          const double v = warp_sum(acc[u]);
          const int k = kbase + u;
          if (lane == 0 && k < s) {
            const int owner = k / sl;
            st_async_f64(mapa_u32(la_rp + (unsigned)(c * sl + k - owner * sl) * 8u, owner), v, mapa_u32(lb_rp, owner));
          }
        }
      }
    }
    PHASE_MARK(2);
    TRACE(1);

    unsigned long long* gll = llr + (long long)par * NQ * s * 2;
    if (pf_tid < 0) {
      // ---- slice owner warps: cluster partial of my slice -> L2 (LL) for every cluster's owner
      if (R > 0) mbar_wait_cluster(bars + 2, it & 1u, 12);
      TRACE(2);
      for (int row = tid; row < R; row += 32 * own_warps) {
        double v = 0.0;
        for (int cc = 0; cc < C; ++cc) v += rp_sm[cc * sl + row];
        ll_store_global(gll + ((long long)q * s + r0 + row) * 2, v, tag);
      }
    } else {
      // ---- the other warps: prefetch block t+1 (slab by TMA gather4, M rows by one bulk copy)
      //      and b_S(t+1), S(t+2) by cp.async -- spread so no warp serialises many TMA issues
      const int32_t* S1 = S_sh + ((it + 1) % 3) * sp;
      if (pf) {
        double* adst = Abuf + nbf * absz;
        if constexpr (RES) {
          if (bulk && tm) {
            const int stride = pf_n / nops >= 1 ? pf_n / nops : 1;
            if (pf_tid % stride == 0)
              for (int j = pf_tid / stride; j < nops; j += pf_n / stride) {
                const int k = 4 * j;
                fence_proxy_async();
                tma_gather4(adst + (long long)k * p.sw, tm, (int)c0, S1[k], S1[min(k + 1, s - 1)],
                            S1[min(k + 2, s - 1)], S1[min(k + 3, s - 1)], bars + nbf);
              }
          } else if (bulk) {
            for (int k = pf_tid; k < s; k += pf_n) {
              fence_proxy_async();
              bulk_g2s(adst + (long long)k * p.sw, p.A + (long long)S1[k] * p.lda + c0, (unsigned)w * 8u, bars + nbf);
            }
          } else {
            for (long long e = pf_tid; e < (long long)s * w; e += pf_n) {
              const int k = (int)(e / w), j = (int)(e - (long long)k * w);
              cp_async8(adst + (long long)k * p.sw + j, p.A + (long long)S1[k] * p.lda + c0 + j);
            }
          }
        }
        if (stageM && !m2) {
          const double* msrc = p.M_pool + qb1 * ss + (long long)r0 * s;
          double* mdst = Mbuf + (buf ^ 1) * mslz;
          if (bulk) {
            if (pf_tid == pf_n - 1) {
              fence_proxy_async();
              bulk_g2s(mdst, msrc, m_bytes, bars + nbf);
            }
          } else {
            for (int e = pf_tid; e < R * s; e += pf_n) cp_async8(mdst + e, msrc + e);
          }
        }
        double* b1 = bS_sh + ((it + 1) % 3) * sp;
        for (int i = pf_tid; i < s; i += pf_n) cp_async8(b1 + i, p.b + S1[i]);
        if (YG == 1 && pf_tid == 0) {
          // rows [yg0, yg1) of M(t+1) into L2 ahead of the y pass of the next iteration
          const int yg0 = (int)((long long)gb * s / gpr);
          const int yg1 = (int)((long long)(gb + 1) * s / gpr);
          const double* src = p.M_pool + qb1 * ss + (long long)yg0 * s;
          const unsigned bytes = (unsigned)(yg1 - yg0) * (unsigned)s * 8u;
          if (bytes > 0 && (s & 1) == 0 && (reinterpret_cast<uintptr_t>(p.M_pool) & 15) == 0)
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(src), "r"(bytes) : "memory");
        }
      }
      if (t + 2 < p.t1) {
        int32_t* S2 = S_sh + ((it + 2) % 3) * sp;
        const int32_t* src = p.S_pool + qb2 * s;
        for (int i = pf_tid; i < s; i += pf_n) cp_async4(S2 + i, src + i);
      }
      cp_async_commit();
    }
    if (t + 3 < p.t1) qb3 = p.bid[t + 3 - p.t0];
    PHASE_MARK(3);
    TRACE(3);
    // ---- r slice: every (row, cluster-group) polls at once; fixed-order combine over the groups
    const int G2 = (R > 0 && R <= T2) ? min(p.g2max > 0 ? min(p.g2max, 16) : 16, T2 / R) : 1;
    if (R > 0 && R <= T2) {
      if (tid < R * G2) {
        const int row = tid % R, grp = tid / R;
        double v = 0.0;
        if ((NQ - grp + G2 - 1) / G2 <= 4) {
          v = ll_gather_sum<4>(gll + (long long)(r0 + row) * 2, (long long)s * 2, grp, G2, NQ, tag, p.err, p.poll_ns);
        } else {
          // many clusters per thread: batches of 8 loads in flight (one L2 round trip per batch)
          for (int q0 = grp; q0 < NQ; q0 += 8 * G2)
            v += ll_gather_sum<8>(gll + (long long)(r0 + row) * 2, (long long)s * 2, q0, G2, NQ, tag, p.err, p.poll_ns);
        }
        red_sm[grp * R + row] = v;
      }
      PHASE_MARK(14);  // this thread's polls done
    } else if (R > T2) {
      for (int row = tid; row < R; row += T2) {
        double v = 0.0;
        for (int qq = 0; qq < NQ; ++qq) v += ll_wait_global(gll + ((long long)qq * s + r0 + row) * 2, tag, p.err);
        red_sm[row] = v;  // R <= 2 * T2
      }
    }
    __syncthreads();
    PHASE_MARK(4);
    TRACE(4);
    // ---- r = A_S x - b_S for my slice; all-gather to the cluster (LL over DSMEM)
    for (int row = tid; row < R; row += T2) {
      double v;
      if (R <= T2) {
        double g[16];  // G2 <= 16 partial sums: all loads at once, fixed pairwise tree
#pragma unroll
        for (int i = 0; i < 16; ++i) g[i] = (i < G2) ? red_sm[i * R + row] : 0.0;
#pragma unroll
        for (int h = 8; h >= 1; h >>= 1)
#pragma unroll
          for (int i = 0; i < h; ++i) g[i] += g[i + h];
        v = g[0];
      } else {
        v = red_sm[row];
      }
      // rank stage (row 9): the P ranks' partials of the row, summed in rank order
      if (P > 1) v = rank_stage_sum(v, q == 0, p.peer_recv, rank, P, s, r0 + row, t, p.err);
      v -= bSc[r0 + row];
      if constexpr (yred) r_sm[r0 + row] = v;
      else for (int cc = 0; cc < C; ++cc) st_async_f64(mapa_u32(la_r + (unsigned)(r0 + row) * 8u, cc), v, mapa_u32(lb_r, cc));
    }
    PHASE_MARK(15);  // r slice combined and sent
    if constexpr (yred) __syncthreads();  // my slice of r
    else mbar_wait_cluster(bars + 3, it & 1u, 13);  // r complete (every rank's slice)
    PHASE_MARK(5);
    TRACE(5);
    // ---- row 8 (off the critical path of the others): ||r||^2 in a fixed order (identical in
    //      every CTA) and the replicated window logic; rho for t+1 is read after the next barrier
    if (warp == NW2 - 1 && !yred) {
      double e = 0.0;
      for (int i = lane; i < s; i += 32) e = fma(r_sm[i], r_sm[i], e);
      e = warp_sum(e);
      if (lane == 0) {
        const int res = window_step_dev(st, tmod, e, p.zeta, p.tol2bb, p.bb, p.adaptive,
                                        gb == 0 && lead && p.writer, p.hist_res, p.hist_rho, p.hist_cap);
        if (res) {
          st.stopped = res;
          stop_sh = 1;
        }
      }
    }
    const long long tmod_prev = tmod;
    tmod = (tmod + 1 == 2 * p.zeta) ? 0 : tmod + 1;
    if (m2 && stageM && it > 0) {  // M rows of block t, loaded after y(t-1) completed
      // Only threads that read the rows wait: thread 0 reissues the buffer once every reader has
      // sent its y values (bars[4] complete), and a thread that had not yet waited for phase it-1
      // (e.g. the window-logic warp at a checkpoint) could otherwise see phase it+1 and hang.
      const bool m_reader = yred ? tid < s : warp < min(NW2 - 1, (R + 3) / 4);
      if (bulk) {
        if (m_reader) mbar_wait(bars + 5, (it - 1) & 1u, 15);
      } else {
        if (warp == 0) cp_async_wait_all();
        __syncthreads();  // warp 0's cp.async rows visible to every reader
      }
    }
    if constexpr (yred) {
      // ---- row 4: partial y over my slice, sent to every rank of the cluster with ||r_slice||^2
      const unsigned la_yp = smem_u32(yp_sm);
      for (int l = tid; l < s; l += T2) {
        double v = 0.0;
        if (!(p.dbg_skip & 1))
          for (int k = 0; k < R; ++k) v = fma(Msl[k * s + l], r_sm[r0 + k], v);
        for (int cc = 0; cc < C; ++cc)
          st_async_f64(mapa_u32(la_yp + (unsigned)(c * (s + 1) + l) * 8u, cc), v, mapa_u32(lb_y, cc));
      }
      if (warp == NW2 - 1) {
        double e = 0.0;
        for (int k = lane; k < R; k += 32) e = fma(r_sm[r0 + k], r_sm[r0 + k], e);
        e = warp_sum(e);
        if (lane < C) st_async_f64(mapa_u32(la_yp + (unsigned)(c * (s + 1) + s) * 8u, lane), e, mapa_u32(lb_y, lane));
      }
    } else if constexpr (YG == 1) {
      // ---- row 4, large blocks: y rows [yg0, yg1) of this CTA (every M element read once per
      //      iteration on the whole GPU), published to L2 as LL words; all CTAs gather y below
      const int yg0 = (int)((long long)gb * s / gpr);
      const int yg1 = (int)((long long)(gb + 1) * s / gpr);
      if (warp < NW2 - 1) {
        const double* Mb = p.M_pool + (long long)p.bid[t - p.t0] * ss;
        for (int k = yg0 + warp; k < yg1; k += NW2 - 1) {
          double v = 0.0;
          const double* Mrow = Mb + (long long)k * s;
#pragma unroll 4
          for (int l = lane; l < s; l += 32) v = fma(__ldg(Mrow + l), r_sm[l], v);
          v = warp_sum(v);
          if (lane == 0) ll_store_global(ylr + ((long long)par * s + k) * 2, v, tag);
        }
      }
    } else {
    // ---- row 4: my slice of y = M r; warps 0..14 take groups of RY rows (lanes over columns,
      //      conflict-free shared-memory reads, butterfly reduce-scatter); lanes of each group then
      //      send the row to peer (lane & 7) by st.async.  The last warp runs the window logic.
      if (R > 0 && warp < NW2 - 1) {
        constexpr int RY = 4;
        const int ngroups = (R + RY - 1) / RY;
        const double* Mg = p.M_pool + (long long)p.bid[t - p.t0] * ss + (long long)r0 * s;
        for (int gi = warp; gi < ngroups; gi += NW2 - 1) {
          const int rb = gi * RY;
          double v[RY] = {0.0, 0.0, 0.0, 0.0};
          if (!(p.dbg_skip & 1)) {
            if (p.m_in_smem && regpath) {
              // s <= 16 RPW: at most RPW / 2 column chunks per lane, fully unrolled
#pragma unroll
              for (int jc = 0; jc < (RPW + 1) / 2; ++jc) {
                const int l = lane + 32 * jc;
                if (l < s) {
                  const double rl = r_sm[l];
#pragma unroll
                  for (int i = 0; i < RY; ++i)
                    if (rb + i < R) v[i] = fma(Msl[(rb + i) * s + l], rl, v[i]);
                }
              }
            } else if (p.m_in_smem) {
#pragma unroll 4
              for (int l = lane; l < s; l += 32) {
                const double rl = r_sm[l];
#pragma unroll
                for (int i = 0; i < RY; ++i)
                  if (rb + i < R) v[i] = fma(Msl[(rb + i) * s + l], rl, v[i]);
              }
            } else {
#pragma unroll 4
              for (int l = lane; l < s; l += 32) {
                const double rl = r_sm[l];
#pragma unroll
                for (int i = 0; i < RY; ++i)
                  if (rb + i < R) v[i] = fma(__ldg(Mg + (long long)(rb + i) * s + l), rl, v[i]);
              }
            }
          }
          warp_reduce_scatter<RY>(v, lane);
          const int row = rb + rs_row<RY>(lane);
          const int cc = lane & 7;  // lanes of a row group share the value; lane & 7 picks the peer
          if (row < R && cc < C) st_async_f64(mapa_u32(la_y + (unsigned)(r0 + row) * 8u, cc), v[0], mapa_u32(lb_y, cc));
          if (row < R && C > 8)
            for (int c2 = cc + 8; c2 < C; c2 += 8) st_async_f64(mapa_u32(la_y + (unsigned)(r0 + row) * 8u, c2), v[0], mapa_u32(lb_y, c2));
        }
      }
    }
    PHASE_MARK(13);  // y slice computed and sent
    if constexpr (YG == 1) {
      for (int l = tid; l < s; l += T2) y_sm[l] = ll_wait_global(ylr + ((long long)par * s + l) * 2, tag, p.err);
      __syncthreads();
    } else if constexpr (YG == 0) {
      mbar_wait_cluster(bars + 4, it & 1u, 14);  // y complete
    } else {
      mbar_wait_cluster(bars + 4, it & 1u, 24);  // every rank's partial y arrived
      for (int l = tid; l < s; l += T2) {
        double v = 0.0;
        for (int cc = 0; cc < C; ++cc) v += yp_sm[cc * (s + 1) + l];  // fixed order: same bits everywhere
        y_sm[l] = v;
      }
      if (tid == 0) {
        double e = 0.0;
        for (int cc = 0; cc < C; ++cc) e += yp_sm[cc * (s + 1) + s];
        const int res = window_step_dev(st, tmod_prev, e, p.zeta, p.tol2bb, p.bb, p.adaptive,
                                        gb == 0 && lead && p.writer, p.hist_res, p.hist_rho, p.hist_cap);
        if (res) {
          st.stopped = res;
          stop_sh = 1;
        }
      }
      __syncthreads();
    }
    // single-buffered M rows: every reader of Msl in this CTA has sent its y rows (they all
    // arrived), so the rows of block t+1 can be brought in now
    if (m2 && stageM && pf && tid == 0) {
      const double* msrc = p.M_pool + qb1 * ss + (long long)r0 * s;
      fence_proxy_async();
      if (bulk) {
        mbar_expect_tx(bars + 5, m_bytes);
        bulk_g2s(Mbuf, msrc, m_bytes, bars + 5);
      }
    }
    if (m2 && stageM && pf && !bulk && warp == 0) {
      const double* msrc = p.M_pool + qb1 * ss + (long long)r0 * s;
      for (int e = lane; e < R * s; e += 32) cp_async8(Mbuf + e, msrc + e);
      cp_async_commit();
    }
    PHASE_MARK(6);
    TRACE(6);

    // ---- rows 5-6: w on the slab, momentum, x (the next iteration's first barrier orders
    //      these shared-memory updates before its A_S x pass)
    const double cm = (1.0 - rho) / (1.0 + rho);
    if constexpr (!CDT && regpath) {
      // w_j = sum_k A[k][j] y_k: the warp's rows from registers, then a fixed-order sum over warps
#pragma unroll
      for (int cc = 0; cc < CPL; ++cc) {
        double a = 0.0;
#pragma unroll
        for (int i = 0; i < RPW; ++i) {
          const int k = warp + 16 * i;
          if (k < s) a = fma(ar[i][cc], y_sm[k], a);
        }
        if (lane + 32 * cc < w) red_sm[warp * p.slab + lane + 32 * cc] = a;
      }
      __syncthreads();
      PHASE_MARK(11);
      for (int jj = tid; jj < w; jj += T2) {
        double wv = 0.0;
        for (int ww = 0; ww < NW2; ++ww) wv += red_sm[ww * p.slab + jj];
        const double mm = cm * (m_sm[jj] - wv);
        m_sm[jj] = mm;
        x_sm[jj] = x_sm[jj] - wv + p.eta * mm;
      }
    } else {
      if constexpr (!CDT) {
        if constexpr (RES) {
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
          const bool vec = ((p.lda & 1) == 0) && ((c0 & 1) == 0) && ((reinterpret_cast<uintptr_t>(p.A) & 15) == 0);
          if (vec) {
            // second pass: a thread owns a column pair, 8 sixteen-byte row loads in flight
            for (int j2 = tid; 2 * j2 < w; j2 += T2) {
              double ax = 0.0, ay = 0.0;
              const double* col = p.A + c0 + 2 * j2;
              const bool pair = 2 * j2 + 1 < w;
              // rows in reverse order: the last rows of the first pass are still in L2
#pragma unroll 16
              for (int k = s - 1; k >= 0; --k) {
                const double yk = y_sm[k];
                if (pair) {
                  const double2 a = __ldcs(reinterpret_cast<const double2*>(col + (long long)Sc[k] * p.lda));
                  ax = fma(a.x, yk, ax);
                  ay = fma(a.y, yk, ay);
                } else {
                  ax = fma(__ldcs(col + (long long)Sc[k] * p.lda), yk, ax);
                }
              }
              w_sm[2 * j2] = ax;
              if (pair) w_sm[2 * j2 + 1] = ay;
            }
          } else {
            for (int jj = tid; jj < w; jj += T2) {
              double a = 0.0;
              const double* col = p.A + c0 + jj;
#pragma unroll 8
              for (int k = s - 1; k >= 0; --k) a = fma(__ldcs(col + (long long)Sc[k] * p.lda), y_sm[k], a);
              w_sm[jj] = a;
            }
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
    }
    PHASE_MARK(7);
    TRACE(7);
    qb1 = qb2;
    qb2 = qb3;
    if (stop_sh) {  // written before the y barrier of this iteration: every thread sees it
      ++t;
      break;
    }
  }
  // drain copies still in flight after an early stop (their barriers must complete before exit)
  if (bulk && t < p.t1) {
    if (a_single || (it & 1)) mbar_wait(bars + 0, phA0, 30); else mbar_wait(bars + 1, phA1, 31);
    if (m2 && stageM) mbar_wait(bars + 5, it & 1u, 35);
  }
  cp_async_wait_all();
  __syncthreads();
  for (int j = tid; j < w; j += T2) {
    p.x[c0 + j] = x_sm[j];
    p.mom[c0 + j] = m_sm[j];
  }
  if (gb == 0 && lead && tid == 0) {
    st.t_done = t;
    *p.st = st;
  }
  if (prof_on)
    for (int i = 0; i < 16; ++i) p.prof[i] += prof_acc[i];
  cluster.sync();  // keep shared memory alive until every peer is done with DSMEM
}

}  // namespace itk
}  // namespace kpp
