// iterate_lean.cu -- the persistent Phase-2 kernel for Kaczmarz++ blocks held in a register tile
// (the c1/c2 launch plans), written for the shortest loop body.
//
// Same method and same exchange as iterate_kernel.cuh (Alg 5 l.9-18 P:1346-1357):
//   r = A_S x - b_S (row 3), y = M r with the memoized M = (A_S A_S^T + lam I)^{-1} (row 4),
//   w = A_S^T y (row 5), m <- c (m - w), x <- x - w + eta m (row 6), window sums / checkpoint (row 8),
// with the s-vector all-reduce as partials --st.async--> slice owner --LL words in L2--> every
// cluster's slice owner --st.async--> r, then y slices --st.async--> every CTA of the cluster.
// What differs is the code, not the arithmetic: every plan decision of this instantiation is
// compile-time (TMA gather4 slabs, M rows double-buffered in shared memory, y per cluster, one slab
// buffer under a register tile), the rare paths (watchdog time-outs, the checkpoint's log/exp/pow)
// are out of line, and each prefetch duty has its own warp.  The generic kernel's loop body spans
// ~165 KB of SASS (instruction fetches on every stage of the critical path); measured on B200, its
// exchange skeleton alone runs at 2.2 us per iteration against 5.9 us for the whole iteration.
#include <cstdlib>

#include "kernel_common.cuh"

// M1 plans (c3): the register tile of block t+1 is loaded from shared memory at the end of iteration t,
// as soon as tile t's registers are dead (after the w partials), so its shared-memory latency overlaps
// the w barrier and the x update instead of heading the next iteration.  Measured (us / iteration,
// early / at the top): c3 6.46 / 6.68; on the double-buffered plans it loses (c2 4.79 / 4.73, c1 2.82 /
// 2.71), so they keep the load at the top.  KPP_LEAN_EARLY_TILE=0: at the top for every plan (A/B).
#ifndef KPP_LEAN_EARLY_TILE
#define KPP_LEAN_EARLY_TILE 1
#endif

namespace kpp {
namespace itk {
namespace {

// try_wait with a suspend-time hint: the waiting warp sleeps until the phase completes (or 0.2 ms
// pass) instead of re-issuing the test -- waiting warps share the SMSP issue slots with the warps on
// the critical path (ncu: the spin loop was ~20 % of all instructions issued per iteration)
__device__ __forceinline__ bool mbar_try_sleep(unsigned long long* bar, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n .reg .pred p;\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n"
      " selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity), "r"(200000u)
      : "memory");
  return ok != 0;
}
static __device__ __noinline__ void lean_wait_slow(unsigned long long* bar, unsigned parity, int code) {
  const unsigned long long t0 = globaltimer();
  while (!mbar_try_sleep(bar, parity))
    if (globaltimer() - t0 > 10000000000ull) mbar_hang(code, parity);
}
__device__ __forceinline__ void lwait(unsigned long long* bar, unsigned parity, int code) {
  if (!mbar_try_cta(bar, parity)) lean_wait_slow(bar, parity, code);
}
// Waits that spin on test_wait (no suspension): KPP_LEAN_SPIN bit 1 the r barrier, 2 the y barrier,
// 4 the owner's partials barrier, 8 the slab barrier (A/B of the wake-up latency of a suspended warp)
#ifndef KPP_LEAN_SPIN
#define KPP_LEAN_SPIN 0
#endif
__device__ __forceinline__ bool mbar_test_cta(unsigned long long* bar, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n .reg .pred p;\n"
      " mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
static __device__ __noinline__ void lean_spin_slow(unsigned long long* bar, unsigned parity, int code) {
  const unsigned long long t0 = globaltimer();
  unsigned n = 0;
  while (!mbar_test_cta(bar, parity))
    if ((++n & 1023u) == 0 && globaltimer() - t0 > 10000000000ull) mbar_hang(code, parity);
}
template <int BIT>
__device__ __forceinline__ void lwait_k(unsigned long long* bar, unsigned parity, int code) {
  if constexpr ((KPP_LEAN_SPIN & BIT) != 0) {
    if (!mbar_test_cta(bar, parity)) lean_spin_slow(bar, parity, code);
  } else {
    lwait(bar, parity, code);
  }
}

struct LeanLayout {
  int sp, sl, s4, red, mslz;
  size_t o_rp, o_x, o_m, o_r, o_y, o_red, o_bS, o_S, o_A, o_M, bytes;
};
__host__ __device__ inline LeanLayout lean_layout(int s, int slab, int sw, int C, bool m1 = false) {
  LeanLayout L{};
  L.sp = (s + 1) & ~1;
  L.sl = (s + C - 1) / C;
  L.s4 = (s + 3) & ~3;
  // gather partials [row][RS] and w partials [column][RS] (RS = 17: conflict-free, compile-time offsets)
  L.red = (slab > L.sl ? slab : L.sl) * 17;
  L.red = (L.red + 1) & ~1;
  L.mslz = (L.sl * s + 15) & ~15;
  size_t o = 64;  // 8 mbarriers
  L.o_rp = o; o += (size_t)((C * L.sl + 1) & ~1) * 8;
  L.o_x = o; o += (size_t)slab * 8;
  L.o_m = o; o += (size_t)slab * 8;
  L.o_r = o; o += (size_t)L.sp * 8;
  L.o_y = o; o += (size_t)L.sp * 8;
  L.o_red = o; o += (size_t)L.red * 8;
  L.o_bS = o; o += 3 * (size_t)L.sp * 8;
  L.o_S = o; o += 3 * (size_t)L.sp * 4;
  o = (o + 127) & ~(size_t)127;  // TMA destinations: 128-byte aligned
  L.o_A = o; o += (size_t)L.s4 * sw * 8;
  L.o_M = o; o += (m1 ? 1 : 2) * (size_t)L.mslz * 8;  // M rows: double-buffered, or one buffer (m1)
  L.bytes = o;
  return L;
}

// RPW: rows per warp of the register tile (warp wi holds rows wi + 16 i), CPL: columns per lane
// (lane l holds columns l + 32 c).  PROF: globaltimer stamps (p.trace) compiled in.
// M1: one M-row buffer (slices of 64 rows x s = 256: 128 KB); block t+1's rows are requested once y(t)
// is complete and land on their own barrier (bars[5]).  Slices of up to 64 rows: two owner warps.
template <int RPW, int CPL, bool PROF, bool M1>
__global__ void __launch_bounds__(T2, 1) iterate_lean_kernel(const __grid_constant__ IterParams p) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int s = p.s;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  cg::cluster_group cluster = cg::this_cluster();
  const int C = (int)cluster.num_blocks();
  const int c = (int)cluster.block_rank();
  const int q = blockIdx.x / C;
  const int NQ = gridDim.x / C;
  const LeanLayout L = lean_layout(s, p.slab, p.sw, C, M1);
  const int sl = L.sl, sp = L.sp;
  const int r0 = min(s, c * sl), r1 = min(s, r0 + sl);
  const int R = r1 - r0;  // rows of the slice this CTA owns (<= 64)
  // PROF: cycle counters of thread 0 of CTA 0 per stage (p.prof[16]), printed by the host
  const bool lprof = PROF && p.prof != nullptr && blockIdx.x == 0 && tid == 0;
  long long lacc[14] = {};
  long long llast = lprof ? clock64() : 0;
#define LM(i)                                   \
  do {                                          \
    if constexpr (PROF) {                       \
      if (lprof) {                              \
        const long long now_ = clock64();       \
        lacc[i] += now_ - llast;                \
        llast = now_;                           \
      }                                         \
    }                                           \
  } while (0)

  // shared memory: offsets derived from smem_raw keep the shared address space (LDS / STS)
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(smem_raw);  // [0] slab + M rows of
  // block t landed (TMA), [2] partials of my slice, [3] r, [4] y (DSMEM st.async transactions)
  double* rp_sm = reinterpret_cast<double*>(smem_raw + L.o_rp);  // [C][sl]
  double* x_sm = reinterpret_cast<double*>(smem_raw + L.o_x);
  double* m_sm = reinterpret_cast<double*>(smem_raw + L.o_m);
  double* r_sm = reinterpret_cast<double*>(smem_raw + L.o_r);
  double* y_sm = reinterpret_cast<double*>(smem_raw + L.o_y);
  double* red_sm = reinterpret_cast<double*>(smem_raw + L.o_red);  // gather [R][17], then w [slab][17]
  constexpr int RS = 17;
  double* bS_sh = reinterpret_cast<double*>(smem_raw + L.o_bS);    // [3][sp] b_S of t, t+1, t+2
  int32_t* S_sh = reinterpret_cast<int32_t*>(smem_raw + L.o_S);    // [3][sp]
  double* Abuf = reinterpret_cast<double*>(smem_raw + L.o_A);      // [s4][sw] slab of the next block
  double* Mbuf = reinterpret_cast<double*>(smem_raw + L.o_M);      // [M1 ? 1 : 2][sl][s] my rows of M
  __shared__ DevState st;
  __shared__ int stop_sh;

  const long long c0 = (long long)blockIdx.x * p.slab;
  const int w = (int)max(0LL, min((long long)p.slab, p.n - c0));
  const long long ss = (long long)s * s;
  const CUtensorMap* tm = &p.tmA;
  const int nops = (s + 3) >> 2;
  // (timing experiments only, results wrong: p.dbg_skip & 2 skips the slab copies of t+1, & 4 the M rows)
  // & 16: the slab rows of t+1 are prefetched into L2 only (gather4 prefetch), not copied to shared memory
  const bool no_slab = (p.dbg_skip & 18) != 0, no_m = (p.dbg_skip & 4) != 0, l2_only = (p.dbg_skip & 16) != 0;
  const unsigned slab_bytes = no_slab ? 0u : (unsigned)nops * 4u * (unsigned)p.sw * 8u;
  const unsigned m_bytes = no_m ? 0u : (unsigned)(R * s) * 8u;
  const bool full = (s == 16 * RPW) && (w == 32 * CPL);  // the tile needs no bounds predicates

  if (tid == 0) {
    st = *p.st;
    stop_sh = 0;
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
  long long qb1 = (p.t0 + 1 < p.t1) ? p.bid[1] : 0;
  long long qb2 = (p.t0 + 2 < p.t1) ? p.bid[2] : 0;
  long long qb3 = 0;
  __syncthreads();
  if (warp == 0)  // block t0: slab (gather4) + my M rows on bars[0]
    issue_loads(true, tm, p.A, p.lda, S_sh, s, c0, w, Abuf, p.sw, true,
                R > 0 ? p.M_pool + (long long)p.bid[0] * ss + (long long)r0 * s : nullptr, R * s, Mbuf, bars + 0);

  cluster.sync();  // every peer's barriers are initialised before any DSMEM store
  long long tmod = p.t0 % (2 * p.zeta);

  const unsigned la_rp = smem_u32(rp_sm), la_r = smem_u32(r_sm), la_y = smem_u32(y_sm);
  const unsigned lb_rp = smem_u32(bars + 2), lb_r = smem_u32(bars + 3), lb_y = smem_u32(bars + 4);
  // pollers per row of my slice: warps 0..14 only -- the last warp issues block t+1's copies (a
  // warp issuing 32 serialised TMA gathers must not hold up a polling group) and runs row 8
  const int G2 = R > 0 ? min(15, (T2 - 32) / R) : 1;
  const int ngroups = (R + 3) >> 2;              // groups of 4 rows of y, over warps 0..14
  const int nown = (R + 31) >> 5;                // owner warps (<= 2)
  long long t = p.t0;
  unsigned it = 0, ph0 = 0;
  constexpr bool early = KPP_LEAN_EARLY_TILE && M1;
  double ar[RPW][CPL];  // register tile of the slab of the current block (rows warp + 16 i, columns lane + 32 c)
  auto load_tile = [&](double (&a)[RPW][CPL]) {
    if (full) {  // (uniform per CTA) no bounds predicates
      const double* a0 = Abuf + warp * p.sw + lane;
#pragma unroll
      for (int i = 0; i < RPW; ++i)
#pragma unroll
        for (int cc = 0; cc < CPL; ++cc) a[i][cc] = a0[16 * i * p.sw + 32 * cc];
    } else {
#pragma unroll
      for (int i = 0; i < RPW; ++i) {
        const int k = warp + 16 * i;
#pragma unroll
        for (int cc = 0; cc < CPL; ++cc)
          a[i][cc] = (k < s && lane + 32 * cc < w) ? Abuf[k * p.sw + lane + 32 * cc] : 0.0;
      }
    }
  };
  for (; t < p.t1; ++t, ++it) {
    const int buf = it & 1;
    const unsigned tag = it + 1;
    const int32_t* Sc = S_sh + (it % 3) * sp;
    const double* bSc = bS_sh + (it % 3) * sp;
    const double* Msl = Mbuf + (M1 ? 0 : buf * L.mslz);
    const bool pf = t + 1 < p.t1;
    (void)Sc;
    // ---- top: slab + M rows of block t have landed; register tile of the slab
    LM(13);
    if (!early || it == 0) {
      lwait_k<8>(bars + 0, ph0, 10);
      ph0 ^= 1u;
      load_tile(ar);
    }
    LM(0);
    cp_async_wait_all();  // this thread's b_S(t) / S(t+1) copies
    if (tid == 0) {
      if (pf) mbar_expect_tx(bars + 0, slab_bytes + (M1 ? 0u : m_bytes));  // (0 bytes: the arrive completes the phase)
      if (R > 0) mbar_expect_tx(bars + 2, (unsigned)(C * R) * 8u);
      mbar_expect_tx(bars + 3, (unsigned)s * 8u);
      mbar_expect_tx(bars + 4, (unsigned)s * 8u);
    }
    __syncthreads();
    if constexpr (PROF) TRACE(0);
    LM(1);
    const double rho = st.rho;  // set at the last checkpoint strictly before t (reading Q11)

    // ---- row 3: partial block residual over the slab, row k to its slice owner
    {
      double xr[CPL];
#pragma unroll
      for (int cc = 0; cc < CPL; ++cc) xr[cc] = (lane + 32 * cc < w) ? x_sm[lane + 32 * cc] : 0.0;
      double v[RPW];
#pragma unroll
      for (int i = 0; i < RPW; ++i) {
        v[i] = 0.0;
#pragma unroll
        for (int cc = 0; cc < CPL; ++cc) v[i] = fma(ar[i][cc], xr[cc], v[i]);
      }
      warp_reduce_scatter<RPW>(v, lane);
      const int k = warp + 16 * rs_row<RPW>(lane);
      if ((lane & (32 / RPW - 1)) == 0 && k < s) {
        const int owner = k / sl;
        st_async_f64(mapa_u32(la_rp + (unsigned)(c * sl + k - owner * sl) * 8u, owner), v[0], mapa_u32(lb_rp, owner));
      }
    }
    if constexpr (PROF) TRACE(1);
    LM(2);

    unsigned long long* gll = p.ll + (long long)(it & 1) * NQ * s * 2;
    if (warp < nown) {
      // ---- owner warps: cluster partial of my slice -> L2 (LL words) for every cluster
      if (R > 0) lwait_k<4>(bars + 2, it & 1u, 12);
      if constexpr (PROF) TRACE(2);
      LM(3);
      const int row = warp * 32 + lane;
      if (row < R) {
        double v = 0.0;
        for (int cc = 0; cc < C; ++cc) v += rp_sm[cc * sl + row];
        ll_store_global(gll + ((long long)q * s + r0 + row) * 2, v, tag);
      }
    } else if (warp == NW2 - 1) {
      // ---- the last warp requests block t+1 behind this iteration (M rows first: one bulk copy)
      if (pf) {
        const int32_t* S1 = S_sh + ((it + 1) % 3) * sp;
        if (!M1 && lane == 0 && R > 0 && !no_m) {
          fence_proxy_async();
          bulk_g2s(Mbuf + (buf ^ 1) * L.mslz, p.M_pool + qb1 * ss + (long long)r0 * s, m_bytes, bars + 0);
        }
        if (l2_only) {
#pragma unroll 1
          for (int j = lane; j < nops; j += 32) {
            const int k = 4 * j;
            tma_prefetch_gather4(tm, (int)c0, S1[k], S1[min(k + 1, s - 1)], S1[min(k + 2, s - 1)], S1[min(k + 3, s - 1)]);
          }
        }
#pragma unroll 1
        for (int j = lane; j < (no_slab ? 0 : nops); j += 32) {  // (no unrolling: a TMA issue is a per-lane waterfall)
          const int k = 4 * j;
          fence_proxy_async();
          tma_gather4(Abuf + (long long)k * p.sw, tm, (int)c0, S1[k], S1[min(k + 1, s - 1)], S1[min(k + 2, s - 1)],
                      S1[min(k + 3, s - 1)], bars + 0);
        }
        double* b1 = bS_sh + ((it + 1) % 3) * sp;
#pragma unroll 1
        for (int i = lane; i < s; i += 32) cp_async8(b1 + i, p.b + S1[i]);
      }
      if (t + 2 < p.t1) {
        int32_t* S2 = S_sh + ((it + 2) % 3) * sp;
        const int32_t* src = p.S_pool + qb2 * s;
#pragma unroll 1
        for (int i = lane; i < s; i += 32) cp_async4(S2 + i, src + i);
      }
      cp_async_commit();
    }
    if (t + 3 < p.t1) qb3 = p.bid[t + 3 - p.t0];
    if constexpr (PROF) TRACE(3);
    LM(4);

    // ---- the slice over all clusters: G2 pollers per row, fixed-order sums
    if (tid < R * G2) {
      const int row = tid % R, grp = tid / R;
      double v = 0.0;
      if ((NQ - grp + G2 - 1) / G2 <= 4) {
        v = ll_gather_sum<4>(gll + (long long)(r0 + row) * 2, (long long)s * 2, grp, G2, NQ, tag, p.err);
      } else {
        for (int q0 = grp; q0 < NQ; q0 += 8 * G2)
          v += ll_gather_sum<8>(gll + (long long)(r0 + row) * 2, (long long)s * 2, q0, G2, NQ, tag, p.err);
      }
      red_sm[row * RS + grp] = v;
    }
    LM(5);
    // warps 0..14 only (named barrier 1): the last warp may still be issuing block t+1's copies
    // (a serialised TMA issue of ~2000 cycles) and joins at the r barrier below
    if (warp < NW2 - 1) asm volatile("bar.sync 1, %0;\n" ::"r"(T2 - 32) : "memory");
    if constexpr (PROF) TRACE(4);
    LM(6);
    // ---- r = A_S x - b_S for my slice (fixed-order tree over the pollers' partial sums)
    double rv = 0.0;
    if (tid < R) {
      double g[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) g[i] = (i < G2) ? red_sm[tid * RS + i] : 0.0;
#pragma unroll
      for (int h = 8; h >= 1; h >>= 1)
#pragma unroll
        for (int i = 0; i < h; ++i) g[i] += g[i + h];
      rv = g[0] - bSc[r0 + tid];
    }
    // ---- r slice to every CTA of the cluster
    if (tid < R)
      for (int cc = 0; cc < C; ++cc) st_async_f64(mapa_u32(la_r + (unsigned)(r0 + tid) * 8u, cc), rv, mapa_u32(lb_r, cc));
    LM(7);
    lwait_k<1>(bars + 3, it & 1u, 13);
    LM(8);
    if constexpr (PROF) TRACE(5);
    // ---- row 8 (last warp, beside y): ||r||^2 in a fixed order and the replicated window logic
    if (warp == NW2 - 1) {
      double e = 0.0;
      for (int i = lane; i < s; i += 32) e = fma(r_sm[i], r_sm[i], e);
      e = warp_sum(e);
      if (lane == 0) {
        const int res = window_step_dev(st, tmod, e, p.zeta, p.tol2bb, p.bb, p.adaptive, blockIdx.x == 0 && p.writer,
                                        p.hist_res, p.hist_rho, p.hist_cap);
        if (res && !(res == 2 && (p.dbg_skip & 22))) {  // (timing experiments run on stale data)
          st.stopped = res;
          stop_sh = 1;
        }
      }
    }
    tmod = (tmod + 1 == 2 * p.zeta) ? 0 : tmod + 1;
    // ---- row 4: my slice of y = M r (groups of 4 rows over warps 0..14 from the staged M rows), to
    //      every CTA (M1: the rows of block t were requested after y(t-1), on bars[5])
    if (M1 && it > 0 && warp < min(NW2 - 1, ngroups)) lwait(bars + 5, (it - 1) & 1u, 15);
    for (int gi = warp; gi < ngroups && warp < NW2 - 1; gi += NW2 - 1) {
      const int rb = gi * 4;
      double v[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int jc = 0; jc < (RPW + 1) / 2; ++jc) {  // s <= 16 RPW: at most RPW / 2 column chunks
        const int l = lane + 32 * jc;
        if (l < s) {
          const double rl = r_sm[l];
#pragma unroll
          for (int i = 0; i < 4; ++i)
            if (rb + i < R) v[i] = fma(Msl[(rb + i) * s + l], rl, v[i]);
        }
      }
      warp_reduce_scatter<4>(v, lane);
      const int row = rb + rs_row<4>(lane);
      const int cc = lane & 7;  // the 8 lanes holding a row send it to peer (lane & 7), C <= 8
      if (row < R && cc < C) st_async_f64(mapa_u32(la_y + (unsigned)(r0 + row) * 8u, cc), v[0], mapa_u32(lb_y, cc));
    }
    LM(9);
    lwait_k<2>(bars + 4, it & 1u, 14);
    LM(10);
    if (M1 && pf && tid == 0 && R > 0 && !no_m) {
      // every reader of the M rows of t has sent its y rows (they all arrived): block t+1's rows
      fence_proxy_async();
      mbar_expect_tx(bars + 5, m_bytes);
      bulk_g2s(Mbuf, p.M_pool + qb1 * ss + (long long)r0 * s, m_bytes, bars + 5);
    } else if (M1 && pf && tid == 0) {
      mbar_arrive(bars + 5);
    }
    if constexpr (PROF) TRACE(6);

    // ---- rows 5-6: w = A_S^T y from the register tile, fixed-order sum over warps, momentum, x
    const double cm = (1.0 - rho) / (1.0 + rho);
    {
      double yk[RPW];  // y rows of this warp's tile rows (tile rows past s are zero: any value works)
#pragma unroll
      for (int i = 0; i < RPW; ++i) {
        yk[i] = y_sm[min(warp + 16 * i, s - 1)];
      }
#pragma unroll
      for (int cc = 0; cc < CPL; ++cc) {
        double a = 0.0;
#pragma unroll
        for (int i = 0; i < RPW; ++i) a = fma(ar[i][cc], yk[i], a);
        if (lane + 32 * cc < w) red_sm[(lane + 32 * cc) * RS + warp] = a;
      }
    }
    if (early && pf) {
      // tile t is dead: block t+1's slab (requested during this iteration) into the registers now.
      // (Not conditional on stop_sh: the window warp may still be writing it -- the flag is only
      // read after the w barrier; a stopping iteration waits for the slab here instead of at exit.)
      lwait(bars + 0, ph0, 10);
      ph0 ^= 1u;
      load_tile(ar);
    }

    LM(11);
    __syncthreads();
    LM(12);
    for (int jj = tid; jj < w; jj += T2) {
      double wv = 0.0;
#pragma unroll
      for (int ww = 0; ww < NW2; ++ww) wv += red_sm[jj * RS + ww];
      const double mm = cm * (m_sm[jj] - wv);
      m_sm[jj] = mm;
      x_sm[jj] = x_sm[jj] - wv + p.eta * mm;
    }
    if constexpr (PROF) TRACE(7);
    qb1 = qb2;
    qb2 = qb3;
    if (stop_sh) {  // written before the y barrier of this iteration: every thread sees it
      ++t;
      break;
    }
  }
  // an early stop leaves block t's slab / M rows in flight: they must land before exit
  if (t < p.t1) {
    if (!early) lwait(bars + 0, ph0, 30);  // (early: waited for at the end of the last iteration)
    if (M1) lwait(bars + 5, (it & 1u), 35);  // the M rows requested after y of the last iteration run
  }
  cp_async_wait_all();
  __syncthreads();
  for (int j = tid; j < w; j += T2) {
    p.x[c0 + j] = x_sm[j];
    p.mom[c0 + j] = m_sm[j];
  }
  if (blockIdx.x == 0 && tid == 0) {
    st.t_done = t;
    *p.st = st;
  }
  if constexpr (PROF)
    if (lprof)
      for (int i = 0; i < 14; ++i) p.prof[i] += lacc[i];
#undef LM
  cluster.sync();  // keep shared memory alive until every peer is done with DSMEM
}

}  // namespace
}  // namespace itk

using KernelFn = void (*)(const IterParams);

// M rows double-buffered when they fit in shared memory, else one buffer
static bool lean_m1(const IterParams& p, int C) {
  return itk::lean_layout(p.s, p.slab, p.sw, C, false).bytes + 128 > 227 * 1024;
}

// The lean kernel serves K++ plans with the slab in a register tile, TMA gather4, the M rows staged
// in shared memory (its y is computed per cluster whatever the plan's y placement), clusters of at
// most 8 and slices of at most 64 rows; nullptr otherwise.
KernelFn iterate_pick_lean(const IterParams& p, int C, int rpw, int cpl) {
  if (p.cd || !p.resident || !p.a_single || !p.tma || (p.ygl != 0 && p.ygl != 4) || p.m_in_smem == 0 || C > 8)
    return nullptr;
  if ((p.s + C - 1) / C > 64 || (p.s & 1)) return nullptr;
  if (itk::lean_layout(p.s, p.slab, p.sw, C, true).bytes + 128 > 227 * 1024) return nullptr;
  static const int sl64 = getenv("KPP_LEAN64") ? atoi(getenv("KPP_LEAN64")) : 1;  // 0: slices <= 32 only
  if (!sl64 && (p.s + C - 1) / C > 32) return nullptr;
  const bool prof = p.trace != nullptr || p.prof != nullptr;
  const bool m1 = lean_m1(p, C);
#define K(R, CP)                                                                                       \
  if (rpw == R && cpl == CP)                                                                           \
    return prof ? (m1 ? itk::iterate_lean_kernel<R, CP, true, true> : itk::iterate_lean_kernel<R, CP, true, false>) \
                : (m1 ? itk::iterate_lean_kernel<R, CP, false, true> : itk::iterate_lean_kernel<R, CP, false, false>);
  K(2, 1) K(4, 1) K(8, 1) K(16, 1) K(2, 2) K(4, 2) K(8, 2) K(16, 2)
#undef K
  return nullptr;
}

size_t iterate_lean_smem_bytes(const IterParams& p, int C) {
  return itk::lean_layout(p.s, p.slab, p.sw, C, lean_m1(p, C)).bytes + 128;
}

}  // namespace kpp
