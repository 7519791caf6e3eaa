// cdpp_stream.cu -- CD++ Phase 2 for blocks that stream from HBM (c5-sized), with the residual
// of iteration t+1 re-associated so that its dense pass overlaps the exchange / projection chain
// of iteration t.
//
// CD++ (Alg 3 l.10-13) with c_t = (1 - rho_t)/(1 + rho_t):
//   r_t = A_{S_t} x_t - b_{S_t},  y_t = M_t r_t,  w_t = I_{S_t}^T y_t
//   m_{t+1} = c_t (m_t - w_t),    x_{t+1} = x_t - w_t + eta m_{t+1}
// so with z_t = x_t + eta c_t m_t (known before y_t):  x_{t+1} = z_t - (1 + eta c_t) w_t  and
//   A_{S_{t+1}} x_{t+1} = A_{S_{t+1}} z_t - (1 + eta c_t) A[S_{t+1}, S_t] y_t.
// The dense product D_{t+1} = A_{S_{t+1}} z_t (272 MB per iteration on c5) does not need y_t: it
// streams while the chain of t (cluster reduction, L2 exchange, window logic, y_t = M_t r_t, L2
// gather of y_t) runs on other warps.  The small correction A[S_{t+1}, S_t] y_t needs only the
// columns of S_t inside each CTA's slab; they are captured ("stash") while D_{t+1} streams.
//
// Slot t of a CTA (columns [c0, c1) of A, x, m):
//   A (all threads, short): apply w_{t-1} to x, m; r_t partial = D_t - (1 + eta c_{t-1}) *
//     A[S_t, S_{t-1} in slab] y_{t-1} -> its cluster slice owner (DSMEM); z_t; list S_t in slab
//   B  warps 0..11: stream D_{t+1} = A[S_{t+1}, slab] z_t (+ stash A[S_{t+1}, S_t in slab])
//      warps 12..15: chain of t -- slice owner sums the cluster's partials -> L2 (LL words);
//      gather the slice from every cluster; r slice -> every CTA of the cluster (DSMEM);
//      ||r||^2 and the window logic (stop test, adaptive rho); rows [yg0, yg1) of y_t = M_t r_t
//      -> L2; gather y_t
// Every sum has a fixed order, so r, y and the window decisions are bit-identical in every CTA.
#include "kernel_common.cuh"

#include <cstdlib>

namespace kpp {
namespace itk {
namespace {

constexpr int STASH = 16;            // stashed columns of S_t per slab (more fall back to global loads)

struct Smem {
  // offsets in doubles from the 128-byte aligned base (bars first)
  int rp, x, m, z, r, y, yprev, dcur, dnext, bS, stash0, stash1, ints;
  int cmap0, cmap1, lj, lk, S;  // int offsets from `ints`; lj/lk hold 3 lists of lcap
  int lcap;
  size_t bytes;
};

__host__ __device__ inline Smem cs_layout(int s, int slab, int C) {
  Smem L;
  const int sp = (s + 1) & ~1;
  const int sl = (s + C - 1) / C;
  L.lcap = (s < slab ? s : slab + 1) & ~1;
  L.lcap += 2;
  int o = 8;  // 8 mbarriers (8 bytes each)
  L.rp = o; o += (C * sl + 1) & ~1;
  L.x = o; o += (slab + 1) & ~1;
  L.m = o; o += (slab + 1) & ~1;
  L.z = o; o += (slab + 1) & ~1;
  L.r = o; o += sp;
  L.y = o; o += sp;
  L.yprev = o; o += sp;
  L.dcur = o; o += sp;
  L.dnext = o; o += sp;
  L.bS = o; o += 3 * sp;
  L.stash0 = o; o += sp * STASH;
  L.stash1 = o; o += sp * STASH;
  L.ints = o;
  int q = 0;
  L.cmap0 = q; q += (slab + 1) & ~1;
  L.cmap1 = q; q += (slab + 1) & ~1;
  L.lj = q; q += 3 * L.lcap;
  L.lk = q; q += 3 * L.lcap;
  L.S = q; q += 3 * sp;
  L.bytes = (size_t)o * 8 + (size_t)q * 4 + 128;
  return L;
}

// Stream rows of A[S, c0:c0+w] against zv (warps 0..NSW-1): out[k] = sum_j A[S_k, c0+j] zv[j]
// (fixed order: lane-strided 16-byte chunks, then a butterfly).  The first ns <= STASH columns of the
// list sl (local columns of S_t in the slab, in list order) are copied to stash[k][i]: lane i loads
// A[S_k, c0 + sl[i]] beside the row's stream (same sectors: an L1/L2 hit), so the stream itself
// carries no per-element column test.
// Row pairs are taken dynamically from *ctr (shared memory), so warps that join late (the chain
// warps, once the chain of the slot is done) take a share; each row's dot product is computed by
// one warp in a fixed order, so the result does not depend on which warp takes it.
__device__ __forceinline__ void stream_pass(const IterParams& p, const int32_t* S, long long c0, int w,
                                            const double* zv, double* out, const int* sl, int ns, double* stash,
                                            bool vec, int* ctr) {
  const int s = p.s;
  const int lane = threadIdx.x & 31;
  constexpr int UR = 2, UQ = 8;  // a whole 444-column row segment per round: 16 loads in flight per lane
  const bool stl = lane < ns;
  const int scol = stl ? sl[lane] : 0;
  for (;;) {
    int kbase = 0;
    if (lane == 0) kbase = atomicAdd(ctr, UR);
    kbase = __shfl_sync(0xffffffffu, kbase, 0);
    if (kbase >= s) break;
    double acc[UR] = {0.0, 0.0};
    const double* rows[UR];
#pragma unroll
    for (int u = 0; u < UR; ++u) rows[u] = p.A + (long long)S[min(kbase + u, s - 1)] * p.lda + c0;
    double sv[UR];
#pragma unroll
    for (int u = 0; u < UR; ++u) sv[u] = stl ? __ldg(rows[u] + scol) : 0.0;
    if (vec) {
      const int w2 = w >> 1;
      const double2* z2 = reinterpret_cast<const double2*>(zv);
      for (int jb = lane; jb < w2; jb += 32 * UQ) {
        double2 a[UR][UQ], zq[UQ];
#pragma unroll
        for (int q = 0; q < UQ; ++q) {
          const int j2 = jb + 32 * q;
          zq[q] = j2 < w2 ? z2[j2] : make_double2(0.0, 0.0);
#pragma unroll
          for (int u = 0; u < UR; ++u)
            a[u][q] = j2 < w2 ? __ldcs(reinterpret_cast<const double2*>(rows[u]) + j2) : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int q = 0; q < UQ; ++q) {
#pragma unroll
          for (int u = 0; u < UR; ++u) {
            acc[u] = fma(a[u][q].x, zq[q].x, acc[u]);
            acc[u] = fma(a[u][q].y, zq[q].y, acc[u]);
          }
        }
      }
      if ((w & 1) && lane == 0) {
#pragma unroll
        for (int u = 0; u < UR; ++u) acc[u] = fma(__ldcs(rows[u] + w - 1), zv[w - 1], acc[u]);
      }
    } else {
      for (int j = lane; j < w; j += 32) {
        const double zj = zv[j];
#pragma unroll
        for (int u = 0; u < UR; ++u) acc[u] = fma(__ldcs(rows[u] + j), zj, acc[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < UR; ++u) {
      if (stl && kbase + u < s) stash[(kbase + u) * STASH + lane] = sv[u];
      const double v = warp_sum(acc[u]);
      if (lane == 0 && kbase + u < s) out[kbase + u] = v;
    }
  }
}

// chain threads: LL values src[l*2] -> dst[l] for l = t0, t0 + nt, ... < n; KQ loads in flight per
// batch, polled together (one L2 round trip once the data are there)
template <int KQ>
__device__ __forceinline__ void ll_gather_vec(double* dst, const unsigned long long* src, int n, unsigned tag,
                                              int* err, int t0, int nt) {
  for (int l0 = t0; l0 < n; l0 += KQ * nt) {
    unsigned long long a[KQ], b[KQ];
#pragma unroll
    for (int i = 0; i < KQ; ++i) {
      const int l = l0 + i * nt;
      if (l < n) {
        asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];\n" : "=l"(a[i]), "=l"(b[i]) : "l"(src + (long long)l * 2) : "memory");
      } else {
        a[i] = b[i] = (unsigned long long)tag << 32;
      }
    }
    const unsigned long long tstart = globaltimer();
    unsigned spins = 0;
    for (;;) {
      bool all = true;
#pragma unroll
      for (int i = 0; i < KQ; ++i) {
        if ((unsigned)(a[i] >> 32) != tag || (unsigned)(b[i] >> 32) != tag) {
          all = false;
          asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];\n" : "=l"(a[i]), "=l"(b[i]) : "l"(src + (long long)(l0 + i * nt) * 2) : "memory");
        }
      }
      if (all) break;
      __nanosleep(200);
      if ((++spins & 1023u) == 0 && globaltimer() - tstart > 20000000000ull) spin_fail(err);
    }
#pragma unroll
    for (int i = 0; i < KQ; ++i)
      if (l0 + i * nt < n) dst[l0 + i * nt] = __longlong_as_double((long long)((a[i] & 0xffffffffull) | (b[i] << 32)));
  }
}

// list of the entries of S (an index set, global columns) inside [gc0, gc1), in order of their
// position k in S: lj = local column, lk = k; cm[lj] = position in the list (one warp)
__device__ __forceinline__ int build_list(const int32_t* S, int s, long long gc0, long long gc1, int* lj, int* lk,
                                          int* cm, int lane) {
  int n = 0;
  for (int k0 = 0; k0 < s; k0 += 32) {
    const int k = k0 + lane;
    const long long g = k < s ? (long long)S[k] : -1;
    const bool in = k < s && g >= gc0 && g < gc1;
    const unsigned bal = __ballot_sync(0xffffffffu, in);
    if (in) {
      const int pos = n + __popc(bal & ((1u << lane) - 1u));
      lj[pos] = (int)(g - gc0);
      lk[pos] = k;
      cm[(int)(g - gc0)] = pos;
    }
    n += __popc(bal);
  }
  return n;
}

// NSW streaming warps; the other T2/32 - NSW warps run the chain
template <int NSW>
__global__ void __launch_bounds__(T2, 1) cdpp_stream_kernel(const __grid_constant__ IterParams p) {
  constexpr int CH0 = 32 * NSW;  // first chain thread
  constexpr int NCH = T2 - CH0;  // chain threads
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int s = p.s;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  cg::cluster_group cluster = cg::this_cluster();
  const int C = (int)cluster.num_blocks();
  const int c = (int)cluster.block_rank();
  // rank of this CTA (several ranks per launch when emulated; cluster boundaries align with them)
  const int gpr = (int)gridDim.x / p.vranks;      // CTAs per rank
  const int vr = (int)blockIdx.x / gpr, gb = (int)blockIdx.x - vr * gpr;
  const int rank = p.rank + vr, P = p.nranks;
  const bool lead = vr == 0;                       // the first rank of the launch writes shared state
  const int q = gb / C, NQ = gpr / C;              // cluster within the rank, clusters per rank
  const int sl = (s + C - 1) / C;
  const int r0 = min(s, c * sl), r1 = min(s, r0 + sl);
  const int R = r1 - r0;
  const int sp = (s + 1) & ~1;
  const Smem L = cs_layout(s, p.slab, C);
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(smem_raw);
  double* D = reinterpret_cast<double*>(smem_raw);
  double* rp_sm = D + L.rp;
  double* x_sm = D + L.x;
  double* m_sm = D + L.m;
  double* z_sm = D + L.z;
  double* r_sm = D + L.r;
  // double buffers picked by parity with selects, not arrays of pointers: the pointers stay
  // derived from smem_raw, so their accesses compile to shared-memory loads/stores (LDS/STS)
  auto ybuf = [&](int i) { return i ? D + L.yprev : D + L.y; };  // y_t of slot t in ybuf(it & 1)
  auto dbuf = [&](int i) { return i ? D + L.dnext : D + L.dcur; };
  double* bS_sh = D + L.bS;
  auto stash = [&](int i) { return i ? D + L.stash1 : D + L.stash0; };
  int* I = reinterpret_cast<int*>(D + L.ints);
  auto cmap = [&](int i) { return i ? I + L.cmap1 : I + L.cmap0; };  // cmap(it & 1): positions of S_t's entries in the slab
  int* ljb = I + L.lj;                       // lists of S_t, S_{t+1}, S_{t+2} entries: [it % 3]
  int* lkb = I + L.lk;
  int32_t* S_sh = I + L.S;
  __shared__ DevState st;
  __shared__ int stop_sh, nl_sh[3], row_ctr;
  __shared__ long long tmod_sh;

  const long long cr1 = p.vcol[vr + 1];            // end of the rank's local columns
  const long long c0 = min(p.vcol[vr] + (long long)gb * p.slab, cr1);
  const long long c1 = (c0 + p.slab < cr1) ? c0 + p.slab : cr1;
  const int w = (int)(c1 > c0 ? c1 - c0 : 0);
  const long long gc0 = p.col_base + c0, gc1 = p.col_base + c1;  // global columns of the slab
  unsigned long long* const llr = p.ll + (long long)vr * p.ll_vstride;   // this rank's grid exchange
  unsigned long long* const ylr = p.yll + (long long)vr * p.ll_vstride;
  unsigned long long* const ulr = p.yx ? p.ull + (long long)vr * p.ll_vstride : nullptr;
  const bool vec = ((p.lda & 1) == 0) && ((c0 & 1) == 0) && ((reinterpret_cast<uintptr_t>(p.A) & 15) == 0);
  const long long ss = (long long)s * s;
  const int yg0 = (int)((long long)gb * s / gpr);
  const int yg1 = (int)((long long)(gb + 1) * s / gpr);

  if (tid == 0) {
    st = *p.st;
    stop_sh = 0;
    tmod_sh = p.t0 % (2 * p.zeta);
    for (int i = 0; i < 4; ++i) mbar_init(bars + i, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  for (int j = tid; j < w; j += T2) {
    x_sm[j] = p.x[c0 + j];
    m_sm[j] = p.mom[c0 + j];
    cmap(0)[j] = -1;
    cmap(1)[j] = -1;
  }
  for (int i = tid; i < s; i += T2) {
    const int32_t v = p.S_pool[(long long)p.bid[0] * s + i];
    S_sh[i] = v;
    bS_sh[i] = p.b[v];
    if (p.t0 + 1 < p.t1) S_sh[sp + i] = p.S_pool[(long long)p.bid[1] * s + i];
  }
  __syncthreads();
  if (warp == 0) {
    const int n = build_list(S_sh, s, gc0, gc1, ljb, lkb, cmap(0), lane);
    if (lane == 0) nl_sh[0] = n;
  }
  if (tid == 0) row_ctr = 0;
  cluster.sync();
  // prologue: D_{t0} = A_{S_{t0}} x_{t0} (no correction: nothing was applied before t0 here)
  stream_pass(p, S_sh, c0, w, x_sm, dbuf(0), nullptr, 0, stash(0), vec, &row_ctr);
  __syncthreads();

  const unsigned la_rp = smem_u32(rp_sm), la_r = smem_u32(r_sm);
  const unsigned lb_rp = smem_u32(bars + 2), lb_r = smem_u32(bars + 3);
  long long tmod = tmod_sh;
  double rho_prev = 0.0;  // rho in force at t-1
  // optional phase timers (KPP_PHASE_PROFILE): CTA 0, thread 0 (phase A, stream) and the first
  // chain thread (chain), then the end-of-slot barrier wait of each
  const bool prof0 = p.prof != nullptr && blockIdx.x == 0 && (tid == 0 || tid == CH0);  // (rank 0's first CTA)
  long long pacc[8] = {};
  long long plast = prof0 ? clock64() : 0;
#define CS_MARK(i)                        \
  do {                                    \
    if (prof0) {                          \
      const long long now_ = clock64();   \
      pacc[i] += now_ - plast;            \
      plast = now_;                       \
    }                                     \
  } while (0)
  long long t = p.t0;
  unsigned it = 0;
  for (; t < p.t1; ++t, ++it) {
    const int cur = it & 1, prv = cur ^ 1;
    const int l0 = it % 3, lm = (it + 2) % 3, lp = (it + 1) % 3;  // lists of S_t, S_{t-1}, S_{t+1}
    const unsigned tag = it + 1;
    const int32_t* Sc = S_sh + (it % 3) * sp;
    const int32_t* Sn = S_sh + ((it + 1) % 3) * sp;
    const double* bSc = bS_sh + (it % 3) * sp;
    const bool pf = t + 1 < p.t1;
    const double rho = st.rho;                       // rho_t (set at the last checkpoint before t)
    const double c_prev = (1.0 - rho_prev) / (1.0 + rho_prev);
    const double c_cur = (1.0 - rho) / (1.0 + rho);
    const int nprev = it > 0 ? nl_sh[lm] : 0;
    const int* ljm = ljb + lm * L.lcap;
    const int* lkm = lkb + lm * L.lcap;
    const double* yprev = ybuf(prv);
    double* y_sm = ybuf(cur);
    if (tid == 0) {
      if (R > 0) mbar_expect_tx(bars + 2, (unsigned)(C * R) * 8u);
      mbar_expect_tx(bars + 3, (unsigned)s * 8u);
      row_ctr = 0;  // read only after the phase-A barrier
    }
    // ---- phase A (all threads): A1 only -- the stream of t+1 needs z_t; the residual partials of t
    // (A2) are formed by the chain threads while the stream runs
    // A1: x_t, m_t from w_{t-1} = I_{S_{t-1}}^T y_{t-1} (cmap(prv) holds S_{t-1}'s positions), z_t
    for (int j = tid; j < w; j += T2) {
      double xv = x_sm[j], mv = m_sm[j];
      if (it > 0) {
        const int pos = cmap(prv)[j];
        const double wv = pos >= 0 ? yprev[lkm[pos]] : 0.0;
        mv = c_prev * (mv - wv);
        xv = xv - wv + p.eta * mv;
        x_sm[j] = xv;
        m_sm[j] = mv;
      }
      z_sm[j] = fma(p.eta * c_cur, mv, xv);
    }
    __syncthreads();
    CS_MARK(0);  // phase A

    if (warp < NSW) {
      // ---- B (streaming warps): D_{t+1} = A[S_{t+1}, slab] z_t, stash A[S_{t+1}, S_t in slab]
      if (pf) stream_pass(p, Sn, c0, w, z_sm, dbuf(prv), ljb + l0 * L.lcap, min(nl_sh[l0], STASH), stash(prv), vec, &row_ctr);
      CS_MARK(1);  // stream (thread 0)
    } else {
      // ---- B (chain threads): exchange, window logic and projection of iteration t
      const int ct = tid - CH0;
      // A2 (chain threads, beside the stream of t+1): partial r_t = D_t - (1 + eta c_{t-1})
      // A[S_t, S_{t-1} in slab] y_{t-1} -> slice owner
      {
        const double* dcur = dbuf(cur);
        const double* stc = stash(cur);
        const double g = 1.0 + p.eta * c_prev;
        for (int k = ct; k < s; k += NCH) {
          double v = dcur[k];
          if (nprev > 0) {
            double corr = 0.0;
            for (int i = 0; i < nprev; ++i) {
              const double a = i < STASH ? stc[k * STASH + i] : __ldg(p.A + (long long)Sc[k] * p.lda + c0 + ljm[i]);
              corr = fma(a, yprev[lkm[i]], corr);
            }
            v = fma(-g, corr, v);
          }
          const int owner = k / sl;
          st_async_f64(mapa_u32(la_rp + (unsigned)(c * sl + k - owner * sl) * 8u, owner), v, mapa_u32(lb_rp, owner));
        }
      }
      unsigned long long* gll = llr + (long long)(it & 1) * NQ * s * 2;
      if (R > 0) mbar_wait_cluster(bars + 2, it & 1u, 42);
      for (int row = ct; row < R; row += NCH) {
        double v = 0.0;
        for (int cc = 0; cc < C; ++cc) v += rp_sm[cc * sl + row];
        ll_store_global(gll + ((long long)q * s + r0 + row) * 2, v, tag);
      }
      // gather my slice from every cluster (batches of 8 in flight), fixed-order sum
      for (int row = ct; row < R; row += NCH) {
        double v = 0.0;
        for (int q0 = 0; q0 < NQ; q0 += 8)
          v += ll_gather_sum<8, 500>(gll + (long long)(r0 + row) * 2, (long long)s * 2, q0, 1, NQ, tag, p.err);
        // rank stage (row 9): the P ranks' partials of the row, summed in rank order (the dense pass of
        // t+1 streams on the other warps meanwhile)
        if (P > 1) v = rank_stage_sum(v, q == 0, p.peer_recv, rank, P, s, r0 + row, t, p.err);
        v -= bSc[r0 + row];
        for (int cc = 0; cc < C; ++cc) st_async_f64(mapa_u32(la_r + (unsigned)(r0 + row) * 8u, cc), v, mapa_u32(lb_r, cc));
      }
      CS_MARK(2);  // chain: partials reduced, slice gathered and sent
      mbar_wait_cluster(bars + 3, it & 1u, 43);  // r_t complete in this CTA
      CS_MARK(3);
      if (ct < 32) {
        // window logic (row 8): ||r||^2 in a fixed order, replicated in every CTA
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
      } else if (ct < 64 && pf) {
        // map of S_{t+1} for the stream of slot t+1 (cmap(prv): clear S_{t-1}'s entries first)
        for (int i = lane; i < nprev; i += 32) cmap(prv)[ljm[i]] = -1;
        __syncwarp();
        const int n = build_list(Sn, s, gc0, gc1, ljb + lp * L.lcap, lkb + lp * L.lcap, cmap(prv), lane);
        if (lane == 0) nl_sh[lp] = n;
      }
      tmod = (tmod + 1 == 2 * p.zeta) ? 0 : tmod + 1;
      if (!p.yx) {
        // rows [yg0, yg1) of y_t = M_t r_t -> L2 (every element of M_t read once on the GPU)
        const double* Mb = p.M_pool + (long long)p.bid[t - p.t0] * ss;
        const int cw = ct >> 5;
        for (int k = yg0 + cw; k < yg1; k += NCH / 32) {
          const double* Mrow = Mb + (long long)k * s;
          double v = 0.0;
#pragma unroll 4
          for (int l = lane; l < s; l += 32) v = fma(__ldg(Mrow + l), r_sm[l], v);
          v = warp_sum(v);
          if (lane == 0) ll_store_global(ylr + ((long long)(it & 1) * s + k) * 2, v, tag);
        }
      } else {
        // y_t = X_t (X_t^T r_t) with X = R^{-1} upper (M_t = X X^T = (A_SS + lam I)^{-1}, Alg 3 l.8-10
        // P:754-758), read from Z = X + X^T - diag(X): row k of X^T is Z[k, 0..k], row k of X is
        // Z[k, k..s).  u rows [yg0, yg1) -> L2, gather u, then y rows [yg0, yg1) -> L2 (the rows are
        // the same, so the L2 prefetch of block t+1's rows serves both passes).  The chain runs beside
        // the stream of t+1, so the second exchange round is off the critical path.
        const double* Zb = p.M_pool + (long long)p.bid[t - p.t0] * ss;
        // u goes to y_{t-1}'s buffer: every read of y_{t-1} in this slot (phase A, the A2 partials of
        // this CTA, all sent before r_t could complete) is done.  (A buffer of its own would take c5's
        // shared memory past the 196 KB carveout, and the smaller L1 slows the stream by a third.)
        double* u_sm = ybuf(prv);
        const int cw = ct >> 5;
        for (int k = yg0 + cw; k < yg1; k += NCH / 32) {
          const double* Zrow = Zb + (long long)k * s;
          double v = 0.0;
#pragma unroll 4
          for (int l = lane; l <= k; l += 32) v = fma(__ldg(Zrow + l), r_sm[l], v);
          v = warp_sum(v);
          if (lane == 0) ll_store_global(ulr + ((long long)(it & 1) * s + k) * 2, v, tag);
        }
        ll_gather_vec<4>(u_sm, ulr + (long long)(it & 1) * s * 2, s, tag, p.err, ct, NCH);
        asm volatile("bar.sync 1, %0;\n" ::"r"(NCH) : "memory");  // u complete (chain threads only)
        for (int k = yg0 + cw; k < yg1; k += NCH / 32) {
          const double* Zrow = Zb + (long long)k * s;
          double v = 0.0;
#pragma unroll 4
          for (int l = k + lane; l < s; l += 32) v = fma(__ldg(Zrow + l), u_sm[l], v);
          v = warp_sum(v);
          if (lane == 0) ll_store_global(ylr + ((long long)(it & 1) * s + k) * 2, v, tag);
        }
      }
      CS_MARK(4);  // window logic + y rows
      if (pf && ct == 0 && (s & 1) == 0 && (reinterpret_cast<uintptr_t>(p.M_pool) & 15) == 0 && yg1 > yg0) {
        const double* src = p.M_pool + (long long)p.bid[t + 1 - p.t0] * ss + (long long)yg0 * s;
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(src), "r"((unsigned)((yg1 - yg0) * s * 8))
                     : "memory");
      }
      // next blocks' index sets and b_S (used from slot t+1 on)
      if (pf) {
        double* b1 = bS_sh + ((it + 1) % 3) * sp;
        for (int i = ct; i < s; i += NCH) b1[i] = p.b[Sn[i]];
      }
      if (t + 2 < p.t1) {
        int32_t* S2 = S_sh + ((it + 2) % 3) * sp;
        const int32_t* src = p.S_pool + (long long)p.bid[t + 2 - p.t0] * s;
        for (int i = ct; i < s; i += NCH) S2[i] = src[i];
      }
      // y_t from every CTA's rows
      ll_gather_vec<4>(y_sm, ylr + (long long)(it & 1) * s * 2, s, tag, p.err, ct, NCH);
      CS_MARK(5);  // y gathered
      // the chain of t is done: help stream D_{t+1}
      if (pf) stream_pass(p, Sn, c0, w, z_sm, dbuf(prv), ljb + l0 * L.lcap, min(nl_sh[l0], STASH), stash(prv), vec, &row_ctr);
    }
    __syncthreads();
    CS_MARK(6);  // end-of-slot barrier wait
    // hand over: y_t (ybuf(cur)) becomes y_prev, rho_t becomes rho_prev
    rho_prev = rho;
    if (stop_sh) {
      ++t;
      ++it;
      break;
    }
  }
  // apply the last w (y of the last iteration run) to x and m
  if (it > 0) {
    __syncthreads();
    const int lastm = (it - 1) & 1, lastl = (it - 1) % 3;
    const double* yprev = ybuf(lastm);
    const double c_last = (1.0 - rho_prev) / (1.0 + rho_prev);
    const int* lkl = lkb + lastl * L.lcap;
    for (int j = tid; j < w; j += T2) {
      const int pos = cmap(lastm)[j];
      const double wv = pos >= 0 ? yprev[lkl[pos]] : 0.0;
      const double mm = c_last * (m_sm[j] - wv);
      m_sm[j] = mm;
      x_sm[j] = x_sm[j] - wv + p.eta * mm;
    }
  }
  __syncthreads();
  for (int j = tid; j < w; j += T2) {
    p.x[c0 + j] = x_sm[j];
    p.mom[c0 + j] = m_sm[j];
  }
  if (gb == 0 && lead && tid == 0) {
    st.t_done = t;
    *p.st = st;
  }
  if (prof0)
    for (int i = 0; i < 7; ++i) p.prof[(tid == 0 ? 0 : 8) + i] += pacc[i];
#undef CS_MARK
  cluster.sync();  // keep shared memory alive until every peer is done with DSMEM
}

}  // namespace
}  // namespace itk

size_t cdpp_stream_smem_bytes(const IterParams& p, int C) { return itk::cs_layout(p.s, p.slab, C).bytes; }

cudaError_t launch_cdpp_stream(cudaStream_t stream, const IterParams& p, int grid, int C, size_t smem) {
  auto fn = itk::cdpp_stream_kernel<12>;  // 12 streaming warps (14 measured slower: 55 vs 51 us/it on c5)
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (C > 8) cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[2];
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(itk::T2);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return launch_coresident(cfg, attr, fn, p);
}

int cdpp_stream_max_clusters(const IterParams& p, int C, size_t smem) {
  auto fn = itk::cdpp_stream_kernel<12>;  // 12 streaming warps (14 measured slower: 55 vs 51 us/it on c5)
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (C > 8) cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  cfg.gridDim = dim3(C * 256);
  cfg.blockDim = dim3(itk::T2);
  cfg.dynamicSmemBytes = smem;
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, (const void*)fn, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

}  // namespace kpp
