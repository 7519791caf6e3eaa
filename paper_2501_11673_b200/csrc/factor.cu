// factor.cu -- small dense factorizations of Phase 1 (SURVEY 8(a) rows 2 and 2').
//
// One CTA per memoized block: Cholesky R^T R = G (G = A_S A_S^T + lam I for K++,
// P:140/P:1319; G = A_SS + lam I for CD++, Alg 3 l.8 P:753) followed by the triangular
// inverse X = R^{-1}, from which the runtime forms M = X X^T = G^{-1} on the tensor cores.
// Memoizing M (rather than R) turns the per-iteration solve into one s x s
// matvec; DESIGN.md records the parity measurement that justifies it.
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include <algorithm>

#include "kpp_internal.h"
#include "kernel_common.cuh"

namespace kpp {
namespace {

constexpr int CT = 256;

__device__ __forceinline__ double warp_sum_f(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ------------------------------------------------------------------ blocked Cholesky + R^{-1}
// One CTA per s x s matrix, NB-wide block steps (right-looking, upper: G = R^T R):
//   1. diagonal tile: unblocked Cholesky by one warp (lane = column) and its inverse Di
//   2. panel: R[k, k+1:] = Di^T G[k, k+1:]  (kept in shared memory for step 3)
//   3. trailing update of the upper triangle: G[i][j] -= sum_l P[l][i] P[l][j]
//      (4 x 4 register micro-tiles, shared-memory panel rows broadcast across a warp)
// then the column sweep of the triangular inverse (X = R^{-1}, upper):
//   X[0:j0, J] = -(X[0:j0, 0:j0] R[0:j0, J]) Di_J   for each NB-wide column block J.
// Every sum runs in a fixed order (no atomics), so the factor is reproducible bit for bit.
template <int NB>
struct CholSmem {
  static size_t bytes(int s) {
    return (size_t)(2 * NB * (NB + 1)) * sizeof(double) + (size_t)NB * (size_t)(((s + 3) & ~3) + 4) * sizeof(double) + 16;
  }
};

// Views: matrix b is G = Gall + b*gstride with element (i,j) at G[i*ldg + j] (likewise X), so the
// kernel also factors a diagonal tile of a larger matrix in place (blocked driver below).
template <int NB>
__global__ void __launch_bounds__(CT) chol_trtri_blocked_kernel(double* Gall, long long ldg, long long gstride,
                                                                double* Xall, long long ldx, long long xstride,
                                                                int s, int* info, int info_base) {
  extern __shared__ __align__(16) double csm[];
  double* D = csm;                      // [NB][NB+1] R_kk
  double* Di = D + NB * (NB + 1);       // [NB][NB+1] R_kk^{-1}
  double* P = Di + NB * (NB + 1);       // [NB][pld] panel rows
  const int pld = ((s + 3) & ~3) + 4;
  double* G = Gall + (long long)blockIdx.x * gstride;
  double* X = Xall + (long long)blockIdx.x * xstride;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  __shared__ int fail_sh;
  if (tid == 0) fail_sh = 0;
  for (long long e = tid; e < (long long)s * s; e += CT) X[(e / s) * ldx + e % s] = 0.0;
  __syncthreads();

  for (int k0 = 0; k0 < s; k0 += NB) {
    const int kb = min(NB, s - k0);
    const int c0 = k0 + kb;        // first trailing column
    const int rr = s - c0;         // trailing size
    // ---- 1. diagonal tile (warp 0; lane = column)
    if (warp == 0) {
      const int j = lane;
      for (int i = 0; i < kb; ++i)
        if (j < kb && j >= i) D[i * (NB + 1) + j] = G[(long long)(k0 + i) * ldg + k0 + j];
      __syncwarp();
      for (int i = 0; i < kb; ++i) {
        const double v = D[i * (NB + 1) + i];
        if (!(v > 0.0)) {
          if (lane == 0 && fail_sh == 0) fail_sh = k0 + i + 1;
        }
        const double d = (v > 0.0) ? sqrt(v) : 1.0;
        __syncwarp();
        if (j < kb && j > i) D[i * (NB + 1) + j] /= d;
        if (j == i) D[i * (NB + 1) + i] = d;
        __syncwarp();
        if (j < kb && j > i) {
          const double rij = D[i * (NB + 1) + j];
          for (int i2 = i + 1; i2 <= j; ++i2) D[i2 * (NB + 1) + j] = fma(-D[i * (NB + 1) + i2], rij, D[i2 * (NB + 1) + j]);
        }
        __syncwarp();
      }
      // Di = R_kk^{-1}: column j by back substitution
      if (j < kb) {
        for (int i = j + 1; i < NB; ++i) Di[i * (NB + 1) + j] = 0.0;
        Di[j * (NB + 1) + j] = 1.0 / D[j * (NB + 1) + j];
        for (int i = j - 1; i >= 0; --i) {
          double a = 0.0;
          for (int l = i + 1; l <= j; ++l) a = fma(D[i * (NB + 1) + l], Di[l * (NB + 1) + j], a);
          Di[i * (NB + 1) + j] = -a / D[i * (NB + 1) + i];
        }
        for (int i = 0; i < kb; ++i) {
          G[(long long)(k0 + i) * ldg + k0 + j] = (j >= i) ? D[i * (NB + 1) + j] : 0.0;
          X[(long long)(k0 + i) * ldx + k0 + j] = (j >= i) ? Di[i * (NB + 1) + j] : 0.0;
        }
      }
    }
    __syncthreads();
    if (rr <= 0) break;
    // ---- 2. panel P[i][c] = sum_{l <= i} Di[l][i] G[k0+l][c0+c]   (rows of R)
    for (int c = tid; c < ((rr + 3) & ~3); c += CT) {
      double g[NB];
#pragma unroll
      for (int l = 0; l < NB; ++l) g[l] = (l < kb && c < rr) ? G[(long long)(k0 + l) * ldg + c0 + c] : 0.0;
#pragma unroll 1
      for (int i = 0; i < NB; ++i) {
        double a = 0.0;
#pragma unroll
        for (int l = 0; l < NB; ++l)
          if (l <= i) a = fma(Di[l * (NB + 1) + i], g[l], a);
        if (i < kb) {
          P[i * pld + c] = a;
          if (c < rr) G[(long long)(k0 + i) * ldg + c0 + c] = a;
        }
      }
    }
    __syncthreads();
    // ---- 3. trailing update of the upper triangle in 4 x 4 micro-tiles
    const int T4 = (rr + 3) >> 2;
    const int ntiles = T4 * (T4 + 1) / 2;
    for (int idx = tid; idx < ntiles; idx += CT) {
      // column-major enumeration of the upper triangle: tb = column tile, ta <= tb
      int tb = (int)((sqrt(8.0 * (double)idx + 1.0) - 1.0) * 0.5);
      while ((tb + 1) * (tb + 2) / 2 <= idx) ++tb;
      while (tb * (tb + 1) / 2 > idx) --tb;
      const int ta = idx - tb * (tb + 1) / 2;
      const int a0 = 4 * ta, b0 = 4 * tb;
      double acc[4][4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = 0.0;
      for (int l = 0; l < kb; ++l) {
        const double2 pa0 = *reinterpret_cast<const double2*>(P + l * pld + a0);
        const double2 pa1 = *reinterpret_cast<const double2*>(P + l * pld + a0 + 2);
        const double2 pb0 = *reinterpret_cast<const double2*>(P + l * pld + b0);
        const double2 pb1 = *reinterpret_cast<const double2*>(P + l * pld + b0 + 2);
        const double pa[4] = {pa0.x, pa0.y, pa1.x, pa1.y}, pb[4] = {pb0.x, pb0.y, pb1.x, pb1.y};
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int v = 0; v < 4; ++v) acc[u][v] = fma(pa[u], pb[v], acc[u][v]);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = a0 + u;
        if (i >= rr) continue;
        double* grow = G + (long long)(c0 + i) * ldg + c0;
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const int j = b0 + v;
          if (j < rr && j >= i) grow[j] -= acc[u][v];
        }
      }
    }
    __syncthreads();
  }
  // zero the strictly lower part of R
  for (long long e = tid; e < (long long)s * s; e += CT) {
    const int i = (int)(e / s), j = (int)(e % s);
    if (i > j) G[(long long)i * ldg + j] = 0.0;
  }
  if (tid == 0 && fail_sh) info[blockIdx.x] = info_base + fail_sh;
  __syncthreads();
  if (fail_sh) return;

  // ---- X = R^{-1}: column blocks J = [j0, j0+kb); diagonal blocks are already in X
  for (int j0 = NB; j0 < s; j0 += NB) {
    const int kb = min(NB, s - j0);
    // stage R[0:j0, J] -> P[l][c] (row l, column c) and Di_J
    for (int e = tid; e < j0 * NB; e += CT) {
      const int l = e / NB, c = e - l * NB;
      P[l * NB + c] = c < kb ? G[(long long)l * ldg + j0 + c] : 0.0;
    }
    for (int e = tid; e < NB * NB; e += CT) {
      const int i = e / NB, c = e - i * NB;
      Di[i * (NB + 1) + c] = (i < kb && c < kb) ? X[(long long)(j0 + i) * ldx + j0 + c] : 0.0;
    }
    __syncthreads();
    for (int i = tid; i < j0; i += CT) {
      // T[c] = sum_{l=i}^{j0-1} X[i][l] R[l][j0+c]
      double t[NB];
#pragma unroll
      for (int c = 0; c < NB; ++c) t[c] = 0.0;
      const double* xrow = X + (long long)i * ldx;
      for (int l = i; l < j0; ++l) {
        const double xv = xrow[l];
#pragma unroll
        for (int c = 0; c < NB; ++c) t[c] = fma(xv, P[l * NB + c], t[c]);
      }
      // X[i][j0+c] = -sum_{c' <= c} T[c'] Di[c'][c]
#pragma unroll 1
      for (int c = 0; c < NB; ++c) {
        double a = 0.0;
#pragma unroll
        for (int c2 = 0; c2 < NB; ++c2)
          if (c2 <= c) a = fma(t[c2], Di[c2 * (NB + 1) + c], a);
        if (c < kb) X[(long long)i * ldx + j0 + c] = -a;
      }
    }
    __syncthreads();
  }
}

__global__ void gather_principal_kernel(const double* A, long long lda, const int32_t* Sall, int s,
                                        double lam, long long cb, long long ce, double* Gall) {
  const int32_t* S = Sall + (long long)blockIdx.y * s;
  double* G = Gall + (long long)blockIdx.y * s * s;
  // 4 rows per CTA (128 threads each), 4 independent gathered loads in flight per thread
  const int k = blockIdx.x * 4 + (threadIdx.x >> 7);
  if (k >= s) return;
  const double* row = A + (long long)S[k] * lda;
  const int t = threadIdx.x & 127;
  for (int l0 = t; l0 < s; l0 += 512) {
    double v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int l = l0 + 128 * u;
      const long long c = l < s ? (long long)S[l] : -1;
      v[u] = (l < s && c >= cb && c < ce) ? __ldg(row + (c - cb)) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int l = l0 + 128 * u;
      if (l < s) G[(long long)k * s + l] = v[u] + ((k == l) ? lam : 0.0);
    }
  }
}

// Symmetric gather: only the upper 32 x 32 tiles (k-tile <= l-tile) are read from A -- the upper
// triangle A[S_k][S_l], k <= l, is all the Cholesky of Alg 3 l.8 consumes (the oracle's factor reads
// exactly these entries) -- and each off-diagonal tile is written twice, as is and transposed
// through shared memory, so G is the full symmetric matrix.  ~Half the random 8-byte reads.
__global__ void __launch_bounds__(256) gather_sym_kernel(const double* A, long long lda, const int32_t* Sall, int s,
                                                         double lam, long long cb, long long ce, double* Gall) {
  __shared__ double tile[32][33];
  __shared__ long long rowoff[32];
  const int T = (s + 31) / 32;
  int idx = blockIdx.x, ti = 0;
  while (idx >= T - ti) {  // upper tile index -> (ti, tj), row-major over the upper triangle
    idx -= T - ti;
    ++ti;
  }
  const int tj = ti + idx;
  const int32_t* S = Sall + (long long)blockIdx.y * s;
  double* G = Gall + (long long)blockIdx.y * s * s;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  if (threadIdx.x < 32) {
    const int k = ti * 32 + threadIdx.x;
    rowoff[threadIdx.x] = k < s ? (long long)S[k] * lda : 0;
  }
  const int l = tj * 32 + tx;
  const long long c = l < s ? (long long)S[l] : -1;
  const bool own = l < s && c >= cb && c < ce;
  __syncthreads();
  double v[4];
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int kk = ty + 8 * r, k = ti * 32 + kk;
    v[r] = (k < s && own) ? __ldg(A + rowoff[kk] + (c - cb)) : 0.0;
  }
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int kk = ty + 8 * r, k = ti * 32 + kk;
    const double g = v[r] + ((k == l) ? lam : 0.0);
    tile[kk][tx] = g;
    if (k < s && l < s && (ti != tj || k <= l)) G[(long long)k * s + l] = g;
  }
  __syncthreads();
  // the mirror image (for the diagonal tile: its lower half, from the upper entries)
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int ll = ty + 8 * r, lr = tj * 32 + ll, k = ti * 32 + tx;
    if (lr < s && k < s && (ti != tj || lr > k)) G[(long long)lr * s + k] = tile[tx][ll];
  }
}

// M[l][k] = M[k][l] for l > k: the lower triangle from the upper one (tiled transpose).
__global__ void __launch_bounds__(256) mirror_upper_kernel(double* Mall, int s) {
  __shared__ double tile[32][33];
  const int T = (s + 31) / 32;
  int idx = blockIdx.x, ti = 0;
  while (idx >= T - ti) {
    idx -= T - ti;
    ++ti;
  }
  const int tj = ti + idx;
  double* M = Mall + (long long)blockIdx.y * s * s;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int kk = ty + 8 * r, k = ti * 32 + kk, l = tj * 32 + tx;
    tile[kk][tx] = (k < s && l < s) ? M[(long long)k * s + l] : 0.0;
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int ll = ty + 8 * r, lr = tj * 32 + ll, k = ti * 32 + tx;
    if (lr < s && k < s && (ti != tj || lr > k)) M[(long long)lr * s + k] = tile[tx][ll];
  }
}

__global__ void add_diag_kernel(double* Gall, int s, double lam) {
  double* G = Gall + (long long)blockIdx.x * s * s;
  for (int i = threadIdx.x; i < s; i += blockDim.x) G[(long long)i * s + i] += lam;
}

__global__ void sumsq_kernel(const double* b, long long m, double* out) {
  __shared__ double sh[1024];
  double a = 0.0;
  for (long long i = threadIdx.x; i < m; i += blockDim.x) a = fma(b[i], b[i], a);
  sh[threadIdx.x] = a;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = sh[0];
}

// ------------------------------------------------------------------ 64 x 64 diagonal tile
// One CTA (256 threads) per tile of size kb <= 64 (views with leading dimensions): right-looking
// Cholesky with one barrier per pivot (row i of R kept apart from the working copy so the trailing
// update of step i and the scaling of row i need no second barrier), then X = R^{-1} by rows from
// the bottom (4 threads per column, shuffle-reduced dots).  In place: G <- R (lower part zeroed).
__global__ void __launch_bounds__(256) chol_diag_kernel(double* Gall, long long ldg, long long gstride, double* Xall,
                                                        long long ldx, long long xstride, int kb, int* info,
                                                        int info_base) {
  extern __shared__ double dsm[];
  double (*a)[65] = reinterpret_cast<double (*)[65]>(dsm);             // working copy
  double (*rx)[65] = reinterpret_cast<double (*)[65]>(dsm + 64 * 65);  // R, then X row by row
  double* dinv_sh = dsm + 2 * 64 * 65;  // 1 / R[i][i]
  __shared__ int fail_sh;
  double* G = Gall + (long long)blockIdx.x * gstride;
  double* X = Xall + (long long)blockIdx.x * xstride;
  const int tid = threadIdx.x;
  if (tid == 0) fail_sh = 0;
  for (int e = tid; e < 64 * 64; e += 256) {
    const int i = e >> 6, j = e & 63;
    a[i][j] = (i < kb && j < kb && j >= i) ? G[(long long)i * ldg + j] : 0.0;
    rx[i][j] = 0.0;
  }
  __syncthreads();
  const int q = tid & 63, p0 = tid >> 6;  // column q, rows p0, p0 + 4, ...
  for (int i = 0; i < kb; ++i) {
    const double v = a[i][i];
    const bool ok = v > 0.0;
    if (!ok && tid == 0 && fail_sh == 0) fail_sh = i + 1;
    const double dinv = ok ? rsqrt(v) : 1.0;  // (one reciprocal square root on the pivot chain)
    const double d = ok ? v * dinv : 1.0;
    if (tid == 0) dinv_sh[i] = dinv;
    // row i of R: R[i][j] = a[i][j] / d
    if (tid < kb && tid >= i) rx[i][tid] = (tid == i) ? d : a[i][tid] * dinv;
    // trailing update with the scaled row: a[p][q] -= R[i][p] R[i][q], i < p <= q
    if (q > i && q < kb) {
      const double riq = a[i][q] * dinv;
      // 4 rows per round, loads first (row i is read-only in this step)
      for (int pp = i + 1 + p0; pp <= q; pp += 16) {
        double ri[4], aq[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int r = pp + 4 * u;
          ri[u] = r <= q ? a[i][r] : 0.0;
          aq[u] = r <= q ? a[r][q] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int r = pp + 4 * u;
          if (r <= q) a[r][q] = fma(-(ri[u] * dinv), riq, aq[u]);
        }
      }
    }
    __syncthreads();
  }
  // X = R^{-1} by COLUMNS, each an independent back substitution R x = e_j (no CTA barriers):
  // 4 lanes per column split the dot products, x_i = (delta_ij - sum_{l=i+1..j} R[i][l] x_l) / R[i][i];
  // X is built in `a` (the working copy is no longer needed), R stays in rx.
  {
    const int col = tid >> 2, sub = tid & 3;  // 64 columns x 4 lanes = 256 threads
    const bool live = col < kb;
    for (int i = kb - 1; i >= 0; --i) {
      double acc = 0.0;
      if (live && col > i)
        for (int l = i + 1 + sub; l <= col; l += 4) acc = fma(rx[i][l], a[l][col], acc);
      acc += __shfl_xor_sync(0xffffffffu, acc, 1);
      acc += __shfl_xor_sync(0xffffffffu, acc, 2);
      if (live && sub == 0 && col >= i) a[i][col] = ((col == i) ? 1.0 - acc : -acc) * dinv_sh[i];
      __syncwarp();
    }
  }
  __syncthreads();
  // only X_kk is needed by the blocked driver (R_kk itself is never read again)
  for (int e = tid; e < kb * kb; e += 256) {
    const int i = e / kb, j = e - i * kb;
    X[(long long)i * ldx + j] = (j >= i) ? a[i][j] : 0.0;
  }
  if (tid == 0 && fail_sh) info[blockIdx.x] = info_base + fail_sh;
}

// ------------------------------------------------------------------ adaptive CholeskyQR2
// lam_out[b] ~ lambda_max of (mode 0) the symmetric G[b] or (mode 1) X[b] X[b]^T with X upper:
// power iteration from the all-ones vector (deterministic), `iters` steps; ||A v|| with ||v|| = 1
// is a lower bound of lambda_max.
// (early exit: once lam > stop[b] / other[b] the refinement decision is already made; the power
// estimate of a PSD operator never decreases)
template <int MODE>
__global__ void __launch_bounds__(256) lmax_kernel(const double* Aall, int s, int iters, double* lam_out,
                                                   const double* other, double stop) {
  extern __shared__ double lsm[];
  double* v = lsm;
  double* u = lsm + s;
  double* wv = lsm + 2 * s;
  __shared__ double nrm_sh;
  const double* A = Aall + (long long)blockIdx.x * s * s;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < s; i += 256) v[i] = 1.0 / sqrt((double)s);
  __syncthreads();
  double lam = 0.0;
  for (int itn = 0; itn < iters; ++itn) {
    const double* src = v;
    if (MODE == 1) {
      for (int j = tid; j < s; j += 256) {  // u = X^T v (X upper: rows i <= j)
        double a = 0.0;
        for (int i = 0; i <= j; ++i) a = fma(A[(long long)i * s + j], v[i], a);
        u[j] = a;
      }
      __syncthreads();
      src = u;
    }
    for (int i = warp; i < s; i += 8) {  // w = A src (MODE 0) or X u (MODE 1, columns j >= i)
      double a = 0.0;
      for (int j = (MODE == 1 ? i : 0) + lane; j < s; j += 32) a = fma(A[(long long)i * s + j], src[j], a);
      a = warp_sum_f(a);
      if (lane == 0) wv[i] = a;
    }
    __syncthreads();
    if (warp == 0) {
      double q = 0.0;
      for (int i = lane; i < s; i += 32) q = fma(wv[i], wv[i], q);
      q = warp_sum_f(q);
      if (lane == 0) nrm_sh = sqrt(q);
    }
    __syncthreads();
    lam = nrm_sh;
    if (other && lam * other[blockIdx.x] > stop) break;  // uniform across the CTA
    const double inv = lam > 0.0 ? 1.0 / lam : 0.0;
    for (int i = tid; i < s; i += 256) v[i] = wv[i] * inv;
    __syncthreads();
  }
  if (tid == 0) lam_out[blockIdx.x] = lam;
}

// The same power iteration for s <= 128 with the matrix held in registers: the matrix-based kernel
// above re-reads G (or X) from L2 on every step (12 x 128 KB per block at s = 128: L2-bandwidth bound,
// ~0.5 ms per c2 batch of 2108 blocks).  Persistent (one CTA of 512 threads per SM, blocks strided);
// warp w holds rows w + 16 i (i < 8), lane l columns l + 32 c (c < 4), the tile loaded once per block.
// Row sums by a warp reduce-scatter (complete within the warp), column sums (mode 1: u = X^T v)
// through shared memory in a fixed order; same start vector, steps and early exit as lmax_kernel.
template <int MODE>
__global__ void __launch_bounds__(512, 1) lmax_reg_kernel(const double* Aall, int B, int s, int iters,
                                                          double* lam_out, const double* other, double stop) {
  constexpr int RS = 17;
  __shared__ double v[128], u[128], wv[128], red[128 * RS];
  __shared__ double nrm_sh;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int b = blockIdx.x; b < B; b += gridDim.x) {
    const double* A = Aall + (long long)b * s * s;
    double a[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int r = warp + 16 * i;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int col = lane + 32 * c;
        a[i][c] = (r < s && col < s && (MODE == 0 || col >= r)) ? A[(long long)r * s + col] : 0.0;
      }
    }
    if (tid < 128) v[tid] = tid < s ? 1.0 / sqrt((double)s) : 0.0;
    __syncthreads();
    double lam = 0.0;
    for (int itn = 0; itn < iters; ++itn) {
      const double* src = v;
      if (MODE == 1) {  // u = X^T v: column sums of the tile over this warp's rows, then over warps
        double vr[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) vr[i] = v[warp + 16 * i];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          double t = 0.0;
#pragma unroll
          for (int i = 0; i < 8; ++i) t = fma(a[i][c], vr[i], t);
          red[(lane + 32 * c) * RS + warp] = t;
        }
        __syncthreads();
        if (tid < 128) {
          double t = 0.0;
#pragma unroll
          for (int w = 0; w < 16; ++w) t += red[tid * RS + w];
          u[tid] = t;
        }
        __syncthreads();
        src = u;
      }
      // w = A src: row sums (the warp's 8 rows over all 128 columns)
      double xs[4], q[8];
#pragma unroll
      for (int c = 0; c < 4; ++c) xs[c] = src[lane + 32 * c];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        q[i] = 0.0;
#pragma unroll
        for (int c = 0; c < 4; ++c) q[i] = fma(a[i][c], xs[c], q[i]);
      }
      itk::warp_reduce_scatter<8>(q, lane);
      if ((lane & 3) == 0) wv[warp + 16 * itk::rs_row<8>(lane)] = q[0];
      __syncthreads();
      if (warp == 0) {
        double t = 0.0;
#pragma unroll
        for (int i = 0; i < 4; ++i) t = fma(wv[lane + 32 * i], wv[lane + 32 * i], t);
        t = itk::warp_sum(t);
        if (lane == 0) nrm_sh = sqrt(t);
      }
      __syncthreads();
      lam = nrm_sh;
      if (other && lam * other[b] > stop) break;  // uniform across the CTA
      const double inv = lam > 0.0 ? 1.0 / lam : 0.0;
      if (tid < 128) v[tid] = wv[tid] * inv;
      __syncthreads();
    }
    if (tid == 0) lam_out[b] = lam;
    __syncthreads();  // v / u / wv are reused by the next block
  }
}

// list[0..cnt) = blocks whose estimated u * kappa(A_S)^2 = u * lamG * lamM (x safety) exceeds tau
__global__ void __launch_bounds__(1024) refine_select_kernel(int B, const double* lamG, const double* lamM,
                                                             double thresh, int* list, int* cnt) {
  __shared__ int base_sh;
  if (threadIdx.x == 0) base_sh = 0;
  __syncthreads();
  for (int b0 = 0; b0 < B; b0 += 1024) {
    const int b = b0 + threadIdx.x;
    const bool need = b < B && !(lamG[b] * lamM[b] <= thresh);  // NaN -> refine
    const unsigned bal = __ballot_sync(0xffffffffu, need);
    __shared__ int wcount[32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) wcount[warp] = __popc(bal);
    __syncthreads();
    int off = base_sh;
    for (int w2 = 0; w2 < warp; ++w2) off += wcount[w2];
    if (need) list[off + __popc(bal & ((1u << lane) - 1u))] = b;
    __syncthreads();
    if (threadIdx.x == 0) {
      int tot = 0;
      for (int w2 = 0; w2 < 32; ++w2) tot += wcount[w2];
      base_sh += tot;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) *cnt = base_sh;
}

// dst[i] = src[list[i]] (gather, dir 0) or dst[list[i]] = src[i] (scatter, dir 1); `count` doubles or
// ints (elem 8 or 4 bytes) per matrix
__global__ void batch_move_kernel(const char* src, char* dst, const int* list, long long bytes, int dir) {
  const int i = blockIdx.x;
  const long long so = (dir == 0 ? (long long)list[i] : (long long)i) * bytes;
  const long long d0 = (dir == 0 ? (long long)i : (long long)list[i]) * bytes;
  for (long long e = threadIdx.x * 8LL; e < bytes; e += blockDim.x * 8LL) {
    if (e + 8 <= bytes) *reinterpret_cast<unsigned long long*>(dst + d0 + e) = *reinterpret_cast<const unsigned long long*>(src + so + e);
    else for (long long k = e; k < bytes; ++k) dst[d0 + k] = src[so + k];
  }
}

}  // namespace

static void chol_tile(cudaStream_t st, int batch, double* G, long long ldg, long long gstride, double* X,
                      long long ldx, long long xstride, int s, int* info, int info_base) {
  if (s <= 512) {
    const size_t sm = CholSmem<32>::bytes(s);
    cudaFuncSetAttribute(chol_trtri_blocked_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    chol_trtri_blocked_kernel<32><<<batch, CT, sm, st>>>(G, ldg, gstride, X, ldx, xstride, s, info, info_base);
  } else {
    const size_t sm = CholSmem<16>::bytes(s);
    cudaFuncSetAttribute(chol_trtri_blocked_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    chol_trtri_blocked_kernel<16><<<batch, CT, sm, st>>>(G, ldg, gstride, X, ldx, xstride, s, info, info_base);
  }
  count_launches(1);
}

// Matrices one launch of the diagonal-tile kernel runs in a single wave (SMs x resident CTAs).
int chol_diag_wave() {
  static int wave = [] {
    constexpr size_t kSmem = (2 * 64 * 65 + 64) * sizeof(double);
    cudaFuncSetAttribute(chol_diag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmem);
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, chol_diag_kernel, 256, kSmem);
    return std::max(1, sms * per);
  }();
  return wave;
}

size_t chol_inv_workspace(int s) {
  // the batched (DMMA) route needs the off-diagonal blocks of R and one s x 64 panel per matrix
  return (s >= 128 && (s & 1) == 0) ? ((size_t)s * s + (size_t)s * 64) * sizeof(double) : 0;
}

void launch_chol_trtri(cudaStream_t st, int batch, double* G, double* X, int s, int* info, double* ws) {
  if (batch <= 0) return;
  const long long ss = (long long)s * s;
  if (!ws || chol_inv_workspace(s) == 0) {
    chol_tile(st, batch, G, s, ss, X, s, ss, s, info, 0);  // one CTA per matrix
    return;
  }
  // Blocked, batched over all matrices: per 64-wide step k
  //   diag:     R_kk, X_kk = R_kk^{-1}                    (chol_tile on the diagonal tile, in place)
  //   panel:    R[k, k+1:] = X_kk^T G[k, k+1:]             (DMMA, X_kk^T lower triangular)
  //   trailing: G[k+1:, k+1:] -= R[k, k+1:]^T R[k, k+1:]   (DMMA, upper triangle only)
  // then X = R^{-1} by column blocks: X[0:j, J] = -(X[0:j, 0:j] R[0:j, J]) X_JJ.
  constexpr int NB = 64;  // (128-wide steps measured slower: the diagonal tiles dominate)
  constexpr size_t kDiagSmem = (2 * 64 * 65 + 64) * sizeof(double);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(chol_diag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDiagSmem);
    attr = true;
  }
  static const bool prof = getenv("KPP_P1_PROFILE") != nullptr;
  cudaEvent_t ev[5];
  if (prof) for (auto& e : ev) { cudaEventCreate(&e); }
  if (prof) cudaEventRecord(ev[0], st);
  double* R = ws;                  // [batch][s][s]: off-diagonal blocks of R
  double* T = ws + (long long)batch * ss;  // [batch][s][NB]
  cudaMemsetAsync(X, 0, (size_t)batch * ss * sizeof(double), st);
  for (int k0 = 0; k0 < s; k0 += NB) {
    const int kb = s - k0 < NB ? s - k0 : NB;
    const long long dk = (long long)k0 * (s + 1);
    cudaEvent_t e0, e1, e2, e3;
    if (prof) { cudaEventCreate(&e0); cudaEventCreate(&e1); cudaEventCreate(&e2); cudaEventCreate(&e3); cudaEventRecord(e0, st); }
    chol_diag_kernel<<<batch, 256, kDiagSmem, st>>>(G + dk, s, ss, X + dk, s, ss, kb, info, k0);
    count_launches(1);
    if (prof) cudaEventRecord(e1, st);
    const int c0 = k0 + kb, tr = s - c0;
    if (tr <= 0) {
      if (prof) { cudaEventSynchronize(e1); float a; cudaEventElapsedTime(&a, e0, e1); fprintf(stderr, "  step %d: diag %.3f\n", k0, a); }
      break;
    }
    Operand xkk{X + dk, s, ss, nullptr, 0, 1};                        // logical (i,k) = X[k][i]
    Operand gp{G + (long long)k0 * s + c0, s, ss, nullptr, 0, 0};
    launch_dgemm(st, batch, kb, tr, kb, xkk, gp, R + (long long)k0 * s + c0, s, ss, 1, 0, 1);
    Operand rpt{R + (long long)k0 * s + c0, s, ss, nullptr, 0, 1};    // logical (i,k) = R[k0+k][c0+i]
    Operand rp{R + (long long)k0 * s + c0, s, ss, nullptr, 0, 0};
    if (prof) cudaEventRecord(e2, st);
    // super-steps of two 64-wide steps (s >= 256): the first step updates only the next 64 rows
    // (G[c0:c0+64, c0:] -= R[k0, c0:c0+64]^T R[k0, c0:]), the second applies both steps' panels to
    // the rest in one K = 128 update (G[c0:, c0:] -= R[k0-64:k0+64, c0:]^T R[k0-64:k0+64, c0:]):
    // half the read-modify-write passes over the trailing matrix, twice the K per pass
    static const bool super = !(getenv("KPP_CHOL_SUPER") && atoi(getenv("KPP_CHOL_SUPER")) == 0);
    const bool sup = super && s >= 256 && kb == NB;
    const bool first = sup && ((k0 / NB) & 1) == 0 && tr > NB;
    const bool second = sup && ((k0 / NB) & 1) == 1;
    if (first) {
      launch_dgemm(st, batch, NB, tr, kb, rpt, rp, G + (long long)c0 * (s + 1), s, ss, 1, 1, 0, -1.0, 1);
    } else if (second) {
      Operand r2t{R + (long long)(k0 - NB) * s + c0, s, ss, nullptr, 0, 1};
      Operand r2{R + (long long)(k0 - NB) * s + c0, s, ss, nullptr, 0, 0};
      launch_dgemm(st, batch, tr, tr, 2 * NB, r2t, r2, G + (long long)c0 * (s + 1), s, ss, 1, 1, 0, -1.0, 1);
    } else {
      launch_dgemm(st, batch, tr, tr, kb, rpt, rp, G + (long long)c0 * (s + 1), s, ss, 1, 1, 0, -1.0, 1);
    }
    if (prof) {
      cudaEventRecord(e3, st);
      cudaEventSynchronize(e3);
      float a, b, c;
      cudaEventElapsedTime(&a, e0, e1);
      cudaEventElapsedTime(&b, e1, e2);
      cudaEventElapsedTime(&c, e2, e3);
      fprintf(stderr, "  step %d: diag %.3f panel %.3f trailing %.3f\n", k0, a, b, c);
    }
  }
  if (prof) cudaEventRecord(ev[1], st);
  for (int j0 = NB; j0 < s; j0 += NB) {
    const int kb = s - j0 < NB ? s - j0 : NB;
    Operand xa{X, s, ss, nullptr, 0, 0}, rj{R + j0, s, ss, nullptr, 0, 0};
    launch_dgemm(st, batch, j0, kb, j0, xa, rj, T, NB, (long long)s * NB, 1, 0, 2);      // T = X00 R0J
    Operand ta{T, NB, (long long)s * NB, nullptr, 0, 0}, xjj{X + (long long)j0 * (s + 1), s, ss, nullptr, 0, 0};
    launch_dgemm(st, batch, j0, kb, kb, ta, xjj, X + j0, s, ss, 1, 0, 0, -1.0, 0);       // X0J = -T XJJ
  }
  if (prof) {
    cudaEventRecord(ev[2], st);
    cudaEventSynchronize(ev[2]);
    float a = 0.f, b = 0.f;
    cudaEventElapsedTime(&a, ev[0], ev[1]);
    cudaEventElapsedTime(&b, ev[1], ev[2]);
    fprintf(stderr, "[kpp blocked chol] batch %d s %d: cholesky %.3f ms, inverse %.3f ms\n", batch, s, a, b);
    for (auto& e : ev) cudaEventDestroy(e);
  }
}

void launch_gather_principal(cudaStream_t st, int batch, const double* A, long long lda,
                             const int32_t* S, int s, double lam, long long col_begin,
                             long long col_end, double* G) {
  if (batch <= 0) return;
  if (!getenv("KPP_GATHER_FULL")) {
    const int T = (s + 31) / 32;
    gather_sym_kernel<<<dim3(T * (T + 1) / 2, batch), 256, 0, st>>>(A, lda, S, s, lam, col_begin, col_end, G);
  } else {
    dim3 grid((s + 3) / 4, batch);
    gather_principal_kernel<<<grid, 512, 0, st>>>(A, lda, S, s, lam, col_begin, col_end, G);
  }
  count_launches(1);
}

void launch_mirror_upper(cudaStream_t st, int batch, double* M, int s) {
  if (batch <= 0) return;
  const int T = (s + 31) / 32;
  mirror_upper_kernel<<<dim3(T * (T + 1) / 2, batch), 256, 0, st>>>(M, s);
  count_launches(1);
}

void launch_add_diag(cudaStream_t st, int batch, double* G, int s, double lam) {
  if (batch <= 0) return;
  add_diag_kernel<<<batch, 256, 0, st>>>(G, s, lam);
  count_launches(1);
}

void launch_sumsq(cudaStream_t st, const double* b, long long m, double* out) {
  sumsq_kernel<<<1, 1024, 0, st>>>(b, m, out);
  count_launches(1);
}

}  // namespace kpp

namespace kpp {
void launch_lmax(cudaStream_t st, int batch, const double* A, int s, int mode, int iters, double* lam,
                 const double* other, double stop) {
  if (batch <= 0) return;
  static const bool reg_off = getenv("KPP_LMAX_REG") && atoi(getenv("KPP_LMAX_REG")) == 0;
  if (s <= 128 && !reg_off) {
    static int nsm = 0;
    if (!nsm) {
      int dev = 0;
      cudaGetDevice(&dev);
      if (cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || nsm <= 0) nsm = 148;
    }
    const int grid = batch < nsm ? batch : nsm;
    if (mode == 0) lmax_reg_kernel<0><<<grid, 512, 0, st>>>(A, batch, s, iters, lam, other, stop);
    else lmax_reg_kernel<1><<<grid, 512, 0, st>>>(A, batch, s, iters, lam, other, stop);
    count_launches(1);
    return;
  }
  const size_t sm = 3 * (size_t)s * sizeof(double);
  if (mode == 0) {
    cudaFuncSetAttribute(lmax_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    lmax_kernel<0><<<batch, 256, sm, st>>>(A, s, iters, lam, other, stop);
  } else {
    cudaFuncSetAttribute(lmax_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    lmax_kernel<1><<<batch, 256, sm, st>>>(A, s, iters, lam, other, stop);
  }
  count_launches(1);
}
void launch_refine_select(cudaStream_t st, int batch, const double* lamG, const double* lamM, double thresh,
                          int* list, int* cnt) {
  refine_select_kernel<<<1, 1024, 0, st>>>(batch, lamG, lamM, thresh, list, cnt);
  count_launches(1);
}
void launch_batch_move(cudaStream_t st, int count, const void* src, void* dst, const int* list, long long bytes,
                       int scatter) {
  if (count <= 0) return;
  batch_move_kernel<<<count, 256, 0, st>>>((const char*)src, (char*)dst, list, bytes, scatter);
  count_launches(1);
}
}  // namespace kpp
