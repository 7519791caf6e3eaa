// lsqr.cu -- sketch-and-precondition projection: Alg 6 as the
// Proj of Alg 5, "K++(LSQR-t_max)" of P:1317-1322.
//
// Phase 1 (per fresh block): A_hat = A_S Pi^T with the SRHT Pi = sqrt(n2/tau) I_T H D over the
// column space (n padded to n2; D = diag(d)/sqrt(n2), d = +-1 from Philox stream 4; T = tau indices of
// [0, n2) from a partial Fisher-Yates on stream 5; R5), R = chol(A_hat A_hat^T + lam I),
// memoized as X = R^{-1}.  On the device: the gathered rows of A_S are transposed into one n2 x (B s)
// matrix, H diag(d) is applied to its rows by the HBM butterfly passes of rht.cu, the tau rows T are
// selected (scaled by 1/sqrt(tau)), and A_hat A_hat^T goes through the batched DMMA GEMM.
//
// Phase 2 (per iteration): w_t = the first n entries of t_max steps of LSQR (Paige & Saunders) on
// M z = R^{-T} r_t with M = R^{-T} [A_S, sqrt(lam) I], from zero.  Every LSQR step needs M v and M^T u
// (products with A_S, reduced over all columns) plus a norm over n: one persistent cooperative kernel
// per window, t_max + 1 exchange rounds per iteration (see the Phase-2 section below and DESIGN.md
// section 7).  Every sum has a fixed order.
#include <cmath>
#include <cstdint>

#include "grid_common.cuh"
#include "kpp_internal.h"
#include "window.cuh"

namespace kpp {
namespace {
using namespace gx;

__device__ __forceinline__ void philox4(uint32_t c[4], uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int round = 0; round < 10; ++round) {
    const uint32_t hi0 = __umulhi(0xD2511F53u, c[0]), lo0 = 0xD2511F53u * c[0];
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c[2]), lo1 = 0xCD9E8D57u * c[2];
    const uint32_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0;
    c[1] = lo1;
    c[2] = n2;
    c[3] = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
}

// ---------------------------------------------------------------- SRHT parameters (reading R5)
__global__ void srht_signs_kernel(uint64_t seed, long long n2, double* d) {
  const long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (j >= n2) return;
  const unsigned long long c = (unsigned long long)j >> 2;
  uint32_t w[4] = {(uint32_t)(c & 0xffffffffull), (uint32_t)(c >> 32), 4u, 0u};
  philox4(w, (uint32_t)(seed & 0xffffffffull), (uint32_t)(seed >> 32));
  d[j] = (w[j & 3] & 1u) ? -1.0 : 1.0;
}
// one thread: partial Fisher-Yates over perm[0..n2) (identity on entry), tau draws, stream 5
__global__ void srht_rows_kernel(uint64_t seed, long long n2, int tau, int32_t* perm) {
  const uint32_t k0 = (uint32_t)(seed & 0xffffffffull), k1 = (uint32_t)(seed >> 32);
  uint32_t w[4] = {0, 0, 0, 0};
  for (int i = 0; i < tau; ++i) {
    if ((i & 3) == 0) {
      w[0] = (uint32_t)(i >> 2);
      w[1] = 0u;
      w[2] = 5u;
      w[3] = 0u;
      philox4(w, k0, k1);
    }
    const long long j = i + (long long)(((unsigned long long)w[i & 3] * (unsigned long long)(n2 - i)) >> 32);
    const int32_t a = perm[i];
    perm[i] = perm[j];
    perm[j] = a;
  }
}
__global__ void iota_kernel(int32_t* v, long long n) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) v[i] = (int32_t)i;
}
// T = sorted perm[0..tau) (one CTA: rank sort, tau <= 2048)
__global__ void sort_small_kernel(const int32_t* in, int tau, int32_t* out) {
  for (int i = threadIdx.x; i < tau; i += blockDim.x) {
    const int32_t v = in[i];
    int rank = 0;
    for (int j = 0; j < tau; ++j) rank += in[j] < v;
    out[rank] = v;
  }
}

// ---------------------------------------------------------------- Phase 1: sketch
// Y[j][b s + k] = A[S_b[k]][j] for j < n (32 x 32 tiles through shared memory)
__global__ void sketch_gather_t_kernel(const double* A, long long lda, long long n, const int32_t* S, int s,
                                       double* Y, long long ldy) {
  __shared__ double tile[32][33];
  const int b = blockIdx.z;
  const long long j0 = blockIdx.x * 32LL;
  const int k0 = blockIdx.y * 32;
  for (int kk = threadIdx.y; kk < 32; kk += 8) {
    const int k = k0 + kk;
    const long long j = j0 + threadIdx.x;
    tile[kk][threadIdx.x] = (k < s && j < n) ? A[(long long)S[(long long)b * s + k] * lda + j] : 0.0;
  }
  __syncthreads();
  for (int jj = threadIdx.y; jj < 32; jj += 8) {
    const long long j = j0 + jj;
    const int k = k0 + threadIdx.x;
    if (j < n && k < s) Y[j * ldy + (long long)b * s + k] = tile[threadIdx.x][jj];
  }
}
// Ah[b][q][k] = scale * Y[T_q][b s + k]
__global__ void sketch_select_kernel(const double* Y, long long ldy, const int32_t* T, int tau, int s, double scale,
                                     double* Ah) {
  const int b = blockIdx.y, q = blockIdx.x;
  const double* src = Y + (long long)T[q] * ldy + (long long)b * s;
  double* dst = Ah + ((long long)b * tau + q) * s;
  for (int k = threadIdx.x; k < s; k += blockDim.x) dst[k] = scale * src[k];
}

// ---------------------------------------------------------------- Phase 2: persistent LSQR kernel
// One CTA per SM (co-resident: cooperative launch), a window of block iterations per launch.  CTA g
// owns the column slab [g slab, (g+1) slab) of x, m and the n-parts of the LSQR vectors (v, w and
// the iterate), so the n-sized updates never leave the SM.  The t_max LSQR steps of Alg 6 l.6-8
// (Paige & Saunders on M z = R^{-T} r, M = R^{-T} [A_S, sqrt(lam) I]) are re-associated into
// t_max + 1 ROUNDS with ONE cross-SM exchange each:
//   round 0   slab row sums of A_S x                                   -> exchange -> r_t, u_1, y_1
//   round r   slab pass: finish v_{r-1} (v_n /= alpha_{r-1}) and the deferred w/x updates of step
//             r-2, then v_n <- A_S^T y_r - beta_r v_{r-1} (column sums) and, on the same tile
//             while it is on chip, the row sums A_S v_n and ||v_n||^2     -> exchange
//             s-part: alpha_r, rotation of step r-1, then the first half of step r
//             (beta_{r+1} u_{r+1} = X^T (A_S v_r + sqrt(lam) v_s) - alpha_r u_r, y = X u)
// The products A_S v and M^T u of one LSQR step therefore share one pass over A_S, and the
// normalisation by alpha (a global norm) is applied after the exchange to the reduced sums
// (linearity) instead of before the pass.  The last step needs no alpha_{t_max+1}: its x update
// only depends on rho_{t_max} = sqrt(rhobar^2 + beta^2) (P-S recurrences).
// Exchange: each CTA publishes s + 1 tagged LL words (row sums, ||v_n slab||^2); the owner warp of
// word k (CTA k mod grid) sums the grid's words in a fixed order and publishes the total; every
// CTA gathers the s + 1 totals.  The s-part is computed redundantly and bit-identically by every CTA.
// Exchange buffers are single: a CTA rewrites its words only after every CTA consumed the previous
// contents, which the data dependencies of the next exchange already guarantee.
constexpr int NT = 512, NW = NT / 32, RW = 8, YR = 8, DC = 2, TW = 32 * DC, RA = 16;

// Round 0: part[g][k] = sum_{j in slab} A[S_k][j] x_j as LL words: RW rows per warp at a time (all
// loads in flight), lanes across the slab.  MODE 0: A_S from global; 1: from global, filling the
// shared slab copy As.
template <int MODE>
__device__ __forceinline__ void slab_rowsums_x(const LsqrParams& p, const int32_t* S_sh, double* As, long long c0,
                                               long long c1, unsigned long long* ll_part, unsigned tag) {
  const int s = p.s, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int k0 = warp * RW; k0 < s; k0 += NW * RW) {
    double acc[RW];
    const double* rows[RW];
#pragma unroll
    for (int r = 0; r < RW; ++r) {
      acc[r] = 0.0;
      rows[r] = p.A + (long long)S_sh[k0 + r < s ? k0 + r : k0] * p.lda;
    }
#pragma unroll 2
    for (long long j = c0 + lane; j < c1; j += 32) {
      const double zj = p.x[j];
#pragma unroll
      for (int r = 0; r < RW; ++r)
        if (k0 + r < s) {
          const double a = rows[r][j];
          if (MODE == 1) As[(long long)(k0 + r) * p.sl + (j - c0)] = a;
          acc[r] = fma(a, zj, acc[r]);
        }
    }
    const double tot = warp_multi_sum<RW>(acc);
    const int r = warp_multi_index<RW>();
    if ((lane & (32 / RW - 1)) == 0 && k0 + r < s)
      ll_put(ll_part + 2LL * ((long long)blockIdx.x * (s + 1) + k0 + r), tot, tag);
  }
  if (threadIdx.x == 0) ll_put(ll_part + 2LL * ((long long)blockIdx.x * (s + 1) + s), 0.0, tag);
}

struct SlabScal {
  double ia;      // 1 / alpha_{r-1} (0 when alpha_{r-1} = 0): normalises the previous v_n
  int defer;      // 0 no previous v (round 1), 1 the initial w = v, x = 0 (step 1), 2 x += f1 w, w = v - f2 w
  double f1, f2;  // deferred coefficients
  double beta;    // beta_r of the C term (0 in round 1)
};

// The slab parts of the LSQR vectors: in shared memory when they fit (lsqr_plan), else global.
struct SlabVec {
  double* vn;  // indexed by the global column j
  double* wn;
  double* xn;
};

// Rounds >= 1: the fused slab pass.  Per tile of TW columns: (1) finish the previous v_n and the
// deferred w/x updates, (2) v_n = A_S^T y - beta v (warps split rows, lanes columns), (3) the row
// sums A_S v_n on the same tile (rows of warp w: k = w + NW i; per-lane partials kept in registers
// across tiles when s <= NW * RA, else folded into shared memory per tile).  ASM: A_S from the
// shared slab copy.  Also returns ||v_s||^2 of the (raw) s-part, reduced with the slab norm.
template <bool ASM, bool REG>
__device__ __forceinline__ double slab_fused(const LsqrParams& p, const int32_t* S_sh, const double* As,
                                             const double* yv, const double* vs, const SlabScal& sc, SlabVec sv,
                                             long long c0, long long c1, double (*part_sh)[TW], double* vt,
                                             double* pacc, double* red_sh, int& bs, unsigned long long* ll_part,
                                             unsigned tag) {
  const int s = p.s, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  double accA[RA];
#pragma unroll
  for (int i = 0; i < RA; ++i) accA[i] = 0.0;
  if (!REG)
    for (int k = tid; k < s; k += NT) pacc[k] = 0.0;
  double q2 = 0.0;
  auto row_ptr = [&](int k) -> const double* {
    return ASM ? As + (long long)k * p.sl - c0 : p.A + (long long)S_sh[k] * p.lda;
  };
  for (long long jb = c0; jb < c1; jb += TW) {
    // (1) previous v and deferred updates (threads tid < TW own column jb + tid)
    if (tid < TW) {
      const long long j = jb + tid;
      double v = 0.0;
      if (j < c1 && sc.defer != 0) {  // (not sc.ia: a zero alpha at an LSQR breakdown still defers)
        v = sv.vn[j] * sc.ia;
        if (sc.defer == 1) {
          sv.wn[j] = v;
          sv.xn[j] = 0.0;
        } else if (sc.defer == 2) {
          const double w = sv.wn[j];
          sv.xn[j] = fma(sc.f1, w, sv.xn[j]);
          sv.wn[j] = fma(-sc.f2, w, v);
        }
      }
      vt[TW + tid] = v;
    }
    // (2) column sums over the rows of this warp
    double acc[DC];
#pragma unroll
    for (int c = 0; c < DC; ++c) acc[c] = 0.0;
#pragma unroll 4
    for (int k = warp; k < s; k += NW) {
      const double* row = row_ptr(k);
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
      double a = 0.0;
      if (j < c1) {
        double h0 = 0.0, h1 = 0.0;  // two interleaved chains, fixed order
#pragma unroll
        for (int w = 0; w < NW; w += 2) {
          h0 += part_sh[w][tid];
          h1 += part_sh[w + 1][tid];
        }
        a = fma(-sc.beta, vt[TW + tid], h0 + h1);
        sv.vn[j] = a;
        q2 = fma(a, a, q2);
      }
      vt[tid] = a;
    }
    __syncthreads();
    // (3) row sums of the tile against the new v_n
    if (REG) {
#pragma unroll
      for (int i = 0; i < RA; ++i) {
        const int k = warp + NW * i;
        if (k < s) {
          const double* row = row_ptr(k);
#pragma unroll
          for (int c = 0; c < DC; ++c) {
            const long long j = jb + c * 32 + lane;
            if (j < c1) accA[i] = fma(row[j], vt[c * 32 + lane], accA[i]);
          }
        }
      }
    } else {
      for (int k = warp; k < s; k += NW) {
        const double* row = row_ptr(k);
        double a = 0.0;
#pragma unroll
        for (int c = 0; c < DC; ++c) {
          const long long j = jb + c * 32 + lane;
          if (j < c1) a = fma(row[j], vt[c * 32 + lane], a);
        }
        a = wsum(a);
        if (lane == 0) pacc[k] += a;
      }
    }
  }
  const long long base = (long long)blockIdx.x * (s + 1);
  if (REG) {
    const double a = warp_multi_sum<RA>(accA);
    const int k = warp + NW * warp_multi_index<RA>();
    if ((lane & (32 / RA - 1)) == 0 && k < s) ll_put(ll_part + 2LL * (base + k), a, tag);
  } else {
    __syncthreads();
    for (int k = tid; k < s; k += NT) ll_put(ll_part + 2LL * (base + k), pacc[k], tag);
  }
  double vq = 0.0;
  for (int k = tid; k < s; k += NT) vq = fma(vs[k], vs[k], vq);
  block_sum2(q2, vq, red_sh, bs);
  if (tid == 0) ll_put(ll_part + 2LL * (base + s), q2, tag);
  return vq;
}

// Exchange of round `tag`: totals of the s + 1 words into out[0..s] (every CTA).
__device__ __forceinline__ void exchange(const LsqrParams& p, unsigned long long* ll_part, unsigned long long* ll_red,
                                         double* out, unsigned tag) {
  const int s1 = p.s + 1, G = p.grid, warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = blockIdx.x;
  for (int k = g + warp * G; k < s1; k += NW * G) {
    double a = 0.0;
    for (int q0 = lane; q0 < G; q0 += 32 * 8) a += ll_sum<8>(ll_part + 2LL * k, 2LL * s1, q0, G, tag, p.err);
    a = wsum(a);
    if (lane == 0) ll_put(ll_red + 2LL * k, a, tag);
  }
  for (int k = threadIdx.x; k < s1; k += NT) out[k] = ll_sum<1>(ll_red + 2LL * k, 0, 0, 1, tag, p.err);
  __syncthreads();
}

// u = X^T vin (- alpha u when !init), beta = ||u||, u /= beta, y = X u, vs = sqrt(lam) y (- beta vs)
// -- one CTA, X upper s x s (shared or global).  Load balance over the triangle: X^T vin pairs
// column k with column SP-1-k (P row groups per pair), X u pairs row block b with block NB-1-b.
// buf: 2 NT doubles.  Returns beta.
__device__ __forceinline__ void xu_block(const LsqrParams& p, const double* X, const double* u, double ib, int r0,
                                         double beta, bool init, double* yv, double* vs) {
  const int s = p.s, lane = threadIdx.x & 31;
  double a[YR];
#pragma unroll
  for (int r = 0; r < YR; ++r) a[r] = 0.0;
  for (int l = (r0 & ~31) + lane; l < s; l += 32) {
    const double ul = u[l] * ib;
#pragma unroll
    for (int r = 0; r < YR; ++r) {
      const int row = r0 + r;
      if (row < s && l >= row) a[r] = fma(X[(long long)row * s + l], ul, a[r]);
    }
  }
  const double y = warp_multi_sum<YR>(a);
  const int row = r0 + warp_multi_index<YR>();
  if ((lane & (32 / YR - 1)) == 0 && row < s) {
    yv[row] = y;
    vs[row] = init ? p.lam_sqrt * y : fma(-beta, vs[row], p.lam_sqrt * y);
  }
}

__device__ __forceinline__ double s_products(const LsqrParams& p, const double* X, const double* vin, double* u,
                                             double* yv, double* vs, double* buf, double* red_sh, int& bs,
                                             double alpha, bool init) {
  const int s = p.s, SP = (s + 31) & ~31, tid = threadIdx.x, warp = tid >> 5;
  const int NPR = SP / 2, P = NT / NPR, cp = tid % NPR, grp = tid / NPR;
  if (grp < P) {
    const int k1 = cp, k2 = SP - 1 - cp;
    const bool v1 = k1 < s, v2 = k2 < s;
    const int iend = v2 ? k2 : (v1 ? k1 : -1);
    double a1 = 0.0, a2 = 0.0;
#pragma unroll 8
    for (int i = grp; i <= iend; i += P) {
      const double vi = vin[i];
      const double* xr = X + (long long)i * s;
      if (i <= k1) a1 = fma(xr[k1], vi, a1);
      if (v2) a2 = fma(xr[k2], vi, a2);
    }
    buf[grp * SP + k1] = a1;
    buf[grp * SP + k2] = a2;
  }
  __syncthreads();
  double uu = 0.0;
  for (int k = tid; k < s; k += NT) {
    double a = 0.0;
    for (int gg = 0; gg < P; ++gg) a += buf[gg * SP + k];
    a = init ? a : fma(-alpha, u[k], a);
    u[k] = a;
    uu = fma(a, a, uu);
  }
  const double beta = sqrt(block_sum(uu, red_sh, bs));
  const double ib = beta > 0.0 ? 1.0 / beta : 0.0;
  const int NB = (s + YR - 1) / YR;
  for (int bp = warp; bp < (NB + 1) / 2; bp += NW) {
    xu_block(p, X, u, ib, bp * YR, beta, init, yv, vs);
    if (NB - 1 - bp != bp) xu_block(p, X, u, ib, (NB - 1 - bp) * YR, beta, init, yv, vs);
  }
  __syncthreads();
  for (int k = tid; k < s; k += NT) u[k] *= ib;  // read by the next product after its barriers
  return beta;
}

// XS / VS: X and the slab vectors in shared memory (p.x_smem / p.v_smem), as template parameters so
// that their accesses compile to shared-memory loads rather than generic ones
template <bool REG, bool XS, bool VS>
__global__ void __launch_bounds__(NT, 1) lsqr_persistent_kernel(LsqrParams p) {
  extern __shared__ double sm[];
  __shared__ DevState st_sh;
  __shared__ double red_sh[128];
  int bs = 0;  // block_sum slot
  const int s = p.s, SP = (s + 31) & ~31;
  double* tot = sm;        // exchange totals [s + 1]
  double* u = tot + SP + 32;
  double* vs = u + SP;
  double* ws = vs + SP;
  double* xs = ws + SP;
  double* yv = xs + SP;
  double* vin = yv + SP;
  double* pacc = vin + SP;
  double* bS = pacc + SP;
  double* buf = bS + SP;           // [2 NT]
  double(*part_sh)[TW] = reinterpret_cast<double(*)[TW]>(buf + 2 * NT);
  double* vt = buf + 2 * NT + NW * TW;  // [2 TW]
  double* slv = vt + 2 * TW;        // [3 sl] when v_smem
  int32_t* S_sh = reinterpret_cast<int32_t*>(slv + (VS ? 3LL * p.sl : 0));
  // on-chip operands (lsqr_plan): the CTA's slab of A_S (s x sl) and X (s x s), reused by all
  // t_max + 1 rounds of the iteration
  double* As = reinterpret_cast<double*>(S_sh) + SP / 2;
  double* Xs = As + (p.a_smem ? (long long)s * p.sl : 0);
  const int tid = threadIdx.x, g = blockIdx.x;
  unsigned long long* ll_part = p.ll;
  unsigned long long* ll_red = p.ll + 2LL * p.grid * (s + 1);
  const long long c0 = (long long)g * p.slab;
  const long long c1 = (c0 + p.slab < p.n) ? c0 + p.slab : p.n;
  SlabVec sv;
  if constexpr (VS) {
    sv.vn = slv - c0;
    sv.wn = slv + p.sl - c0;
    sv.xn = slv + 2LL * p.sl - c0;
  } else {
    sv.vn = p.vn;
    sv.wn = p.wn;
    sv.xn = p.xn;
  }
  if constexpr (!XS) {
    // measured (c3, X in global memory): generic accesses to X and the slab vectors run faster
    // here than shared/global-specific ones (192.6 vs 212.1 us/iteration); the no-op moves hide
    // the address spaces.  With X in shared memory (c2) the specific loads win (119.1 -> 105.2).
    asm volatile("mov.b64 %0, %0;" : "+l"(sv.vn));
    asm volatile("mov.b64 %0, %0;" : "+l"(sv.wn));
    asm volatile("mov.b64 %0, %0;" : "+l"(sv.xn));
  }
  if (tid == 0) st_sh = *p.st;
  __syncthreads();
  unsigned tag = 0;
  long long tm = p.t0 % (2 * p.zeta);
  const bool prof = p.prof != nullptr && g == 0 && tid == 0;
  long long tp = prof ? clock64() : 0;
  long long pr[8] = {0, 0, 0, 0, 0, 0, 0, 0};
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
    const double* Xg = p.X_pool + kb * (long long)s * s;
    if constexpr (XS) {  // asynchronous copy, overlapped with round 0
      const long long nx = (long long)s * s;
      for (long long i = 2LL * tid; i < nx; i += 2LL * NT) cp_async16(Xs + i, Xg + i);
      asm volatile("cp.async.commit_group;\n" ::: "memory");
    }
    const double* X = XS ? Xs : Xg;
    if constexpr (!XS) asm volatile("mov.b64 %0, %0;" : "+l"(X));
    for (int i = tid; i < s; i += NT) {
      const int32_t row = p.S_pool[kb * s + i];
      S_sh[i] = row;
      bS[i] = p.b[row];
    }
    __syncthreads();
    // ---- round 0: r_t = A_S x_t - b_S, u_1 = R^{-T} r / beta_1, y_1 = R^{-1} u_1, v_s raw
    ++tag;
    if (p.a_smem) slab_rowsums_x<1>(p, S_sh, As, c0, c1, ll_part, tag);
    else slab_rowsums_x<0>(p, S_sh, As, c0, c1, ll_part, tag);
    mark(0);
    exchange(p, ll_part, ll_red, tot, tag);
    mark(1);
    double e = 0.0;
    for (int k = tid; k < s; k += NT) {
      const double r = tot[k] - bS[k];
      vin[k] = r;
      e = fma(r, r, e);
    }
    if constexpr (XS) asm volatile("cp.async.wait_all;\n" ::: "memory");
    e = block_sum(e, red_sh, bs);  // (its barrier also publishes vin and the copied X)
    double beta = s_products(p, X, vin, u, yv, vs, buf, red_sh, bs, 0.0, true);
    mark(2);
    double phibar = beta, rhobar = 0.0, alpha = 0.0, f1 = 0.0, f2 = 0.0;
    SlabScal sc{0.0, 0, 0.0, 0.0, 0.0};
    for (int r = 1; r <= p.tmax; ++r) {
      ++tag;
      const double vq = p.a_smem
                            ? slab_fused<true, REG>(p, S_sh, As, yv, vs, sc, sv, c0, c1, part_sh, vt, pacc, red_sh, bs,
                                                    ll_part, tag)
                            : slab_fused<false, REG>(p, S_sh, As, yv, vs, sc, sv, c0, c1, part_sh, vt, pacc, red_sh,
                                                     bs, ll_part, tag);
      mark(3);
      exchange(p, ll_part, ll_red, tot, tag);
      mark(4);
      // alpha_r, v_s = raw / alpha_r; rotation of step r - 1 (r >= 2) or the initial w (r = 1)
      alpha = sqrt(tot[s] + vq);
      const double ia = alpha > 0.0 ? 1.0 / alpha : 0.0;
      if (r == 1) {
        rhobar = alpha;
        f1 = f2 = 0.0;
      } else {
        const double rho = sqrt(rhobar * rhobar + beta * beta);
        const double c = rho > 0.0 ? rhobar / rho : 1.0, sn = rho > 0.0 ? beta / rho : 0.0;
        const double theta = sn * alpha, phi = c * phibar;
        f1 = rho > 0.0 ? phi / rho : 0.0;
        f2 = rho > 0.0 ? theta / rho : 0.0;
        rhobar = -c * alpha;
        phibar = sn * phibar;
      }
      for (int k = tid; k < s; k += NT) {
        const double v = vs[k] * ia;
        vs[k] = v;
        if (r == 1) {
          ws[k] = v;
          xs[k] = 0.0;
        } else {
          xs[k] = fma(f1, ws[k], xs[k]);
          ws[k] = fma(-f2, ws[k], v);
        }
        vin[k] = fma(p.lam_sqrt, v, tot[k] * ia);  // M v_r = R^{-T} (A_S v_n + sqrt(lam) v_s)
      }
      __syncthreads();
      mark(5);
      // step r, first half: beta_{r+1} u_{r+1} = M v_r - alpha_r u_r; y = R^{-1} u; v_s raw
      const double beta_next = s_products(p, X, vin, u, yv, vs, buf, red_sh, bs, alpha, false);
      mark(6);
      sc.ia = ia;
      sc.defer = r == 1 ? 1 : 2;
      sc.f1 = f1;
      sc.f2 = f2;
      sc.beta = beta_next;
      beta = beta_next;
    }
    // the x update of step t_max needs rho_{t_max} only (no alpha_{t_max + 1})
    double f1_last;
    {
      const double rho = sqrt(rhobar * rhobar + beta * beta);
      const double c = rho > 0.0 ? rhobar / rho : 1.0;
      f1_last = rho > 0.0 ? c * phibar / rho : 0.0;
    }
    // ---- slab: finish v_{t_max}, the deferred update of step t_max - 1, then w_t = x + f1 w;
    //      m = c (m - w_t), x = x - w_t + eta m
    {
      const double rho = st_sh.rho, cm = (1.0 - rho) / (1.0 + rho);
      for (long long j = c0 + tid; j < c1; j += NT) {
        const double v = sv.vn[j] * sc.ia;
        double xn, wn;
        if (sc.defer == 1) {
          wn = v;
          xn = 0.0;
        } else {
          const double w = sv.wn[j];
          xn = fma(sc.f1, w, sv.xn[j]);
          wn = fma(-sc.f2, w, v);
        }
        const double wt = fma(f1_last, wn, xn);
        const double mm = cm * (p.mom[j] - wt);
        p.mom[j] = mm;
        p.x[j] = p.x[j] - wt + p.eta * mm;
      }
    }
    __syncthreads();
    if (tid == 0) {
      const int res = window_step_dev(st_sh, tm, e, p.zeta, p.tol2bb, p.bb, p.adaptive, p.writer && g == 0,
                                      p.hist_res, p.hist_rho, p.hist_cap);
      if (res) st_sh.stopped = res;
      st_sh.t_done = t + 1;
    }
    if (++tm == 2 * p.zeta) tm = 0;
    __syncthreads();
    mark(7);
  }
  if (g == 0 && tid == 0) *p.st = st_sh;
  if (prof)
    for (int i = 0; i < 8; ++i) p.prof[i] += pr[i];
}

}  // namespace

size_t lsqr_smem_bytes(int s, int a_smem, int sl, int x_smem, int v_smem) {
  const int SP = (s + 31) & ~31;
  size_t d = (size_t)(9 * SP + 32 + 2 * NT + NW * TW + 2 * TW + SP / 2);
  if (v_smem) d += 3 * (size_t)sl;
  if (a_smem) d += (size_t)s * sl;
  if (x_smem) d += (size_t)s * s;
  return d * sizeof(double);
}

void launch_srht_setup(cudaStream_t st, uint64_t seed, long long n2, int tau, double* dsign, int32_t* T,
                       int32_t* perm_ws) {
  srht_signs_kernel<<<(unsigned)((n2 + 255) / 256), 256, 0, st>>>(seed, n2, dsign);
  iota_kernel<<<(unsigned)((n2 + 255) / 256), 256, 0, st>>>(perm_ws, n2);
  srht_rows_kernel<<<1, 1, 0, st>>>(seed, n2, tau, perm_ws);
  sort_small_kernel<<<1, 1024, 0, st>>>(perm_ws, tau, T);
  count_launches(4);
}

void launch_sketch_gather_t(cudaStream_t st, int batch, const double* A, long long lda, long long n,
                            const int32_t* S, int s, double* Y, long long ldy) {
  dim3 grid((unsigned)((n + 31) / 32), (unsigned)((s + 31) / 32), (unsigned)batch);
  sketch_gather_t_kernel<<<grid, dim3(32, 8), 0, st>>>(A, lda, n, S, s, Y, ldy);
  count_launches(1);
}

void launch_sketch_select(cudaStream_t st, int batch, const double* Y, long long ldy, const int32_t* T, int tau,
                          int s, double scale, double* Ah) {
  dim3 grid((unsigned)tau, (unsigned)batch);
  sketch_select_kernel<<<grid, 128, 0, st>>>(Y, ldy, T, tau, s, scale, Ah);
  count_launches(1);
}

size_t lsqr_ll_words(int s, int grid) { return 2 * ((size_t)grid * (s + 1) + s + 1); }

// One window [p.t0, p.t1) of K++ with Proj = Alg 6 (one cooperative launch: all CTAs co-resident).
cudaError_t launch_lsqr_window(cudaStream_t st, const LsqrParams& p) {
  static int attr_smem[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const bool reg = p.s <= NW * RA;
  static const void* const fns[8] = {
      (const void*)lsqr_persistent_kernel<false, false, false>, (const void*)lsqr_persistent_kernel<false, false, true>,
      (const void*)lsqr_persistent_kernel<false, true, false>,  (const void*)lsqr_persistent_kernel<false, true, true>,
      (const void*)lsqr_persistent_kernel<true, false, false>,  (const void*)lsqr_persistent_kernel<true, false, true>,
      (const void*)lsqr_persistent_kernel<true, true, false>,   (const void*)lsqr_persistent_kernel<true, true, true>};
  const int ki = (reg ? 4 : 0) + (p.x_smem ? 2 : 0) + (p.v_smem ? 1 : 0);
  const void* fn = fns[ki];
  const size_t smem = lsqr_smem_bytes(p.s, p.a_smem, p.sl, p.x_smem, p.v_smem);
  if ((int)smem > attr_smem[ki]) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr_smem[ki] = (int)smem;
  }
  if (p.grid > NT) return cudaErrorInvalidValue;
  cudaError_t e = cudaMemsetAsync(p.ll, 0, lsqr_ll_words(p.s, p.grid) * sizeof(unsigned long long), st);
  if (e != cudaSuccess) return e;
  LsqrParams q = p;
  void* args[] = {&q};
  e = cudaLaunchCooperativeKernel(fn, dim3(p.grid), dim3(NT), args, smem, st);
  count_launches(1);
  return e;
}

}  // namespace kpp
