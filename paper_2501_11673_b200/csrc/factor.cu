// factor.cu -- small dense factorizations of Phase 1 (SURVEY 8(a) rows 2 and 2').
//
// One CTA per memoized block: Cholesky R^T R = G (G = A_S A_S^T + lam I for K++,
// P:140/P:1319; G = A_SS + lam I for CD++, Alg 3 l.8 P:753) followed by the triangular
// inverse X = R^{-1}, from which the runtime forms M = X X^T = G^{-1} on the tensor cores.
// Memoizing M (rather than R) turns the per-iteration solve into one s x s
// matvec; DESIGN.md records the parity measurement that justifies it.
//
// Up-looking Cholesky: row i of R is R_ij = (G_ij - sum_{k<i} R_ki R_kj) / R_ii, one
// thread per column j, R kept in place in global memory (L1/L2 resident).
// Triangular inverse: column j of X by back substitution, one thread per column.
#include <cstdint>

#include "kpp_internal.h"

namespace kpp {
namespace {

constexpr int CT = 512;

__global__ void __launch_bounds__(CT) chol_trtri_kernel(double* Gall, double* Xall, int s, int* info) {
  double* G = Gall + (long long)blockIdx.x * s * s;
  double* X = Xall + (long long)blockIdx.x * s * s;
  __shared__ double diag_sh;
  __shared__ int fail_sh;
  if (threadIdx.x == 0) fail_sh = 0;
  __syncthreads();
  for (int i = 0; i < s; ++i) {
    // numerators for row i (columns j >= i)
    for (int j = i + threadIdx.x; j < s; j += blockDim.x) {
      double a = 0.0;
      for (int k = 0; k < i; ++k) a = fma(-G[(long long)k * s + i], G[(long long)k * s + j], a);
      const double v = G[(long long)i * s + j] + a;
      if (j == i) {
        if (!(v > 0.0)) {
          fail_sh = i + 1;
          diag_sh = 1.0;
        } else {
          diag_sh = sqrt(v);
        }
      }
      G[(long long)i * s + j] = v;  // numerator, scaled below
    }
    __syncthreads();
    const double d = diag_sh;
    for (int j = i + threadIdx.x; j < s; j += blockDim.x)
      G[(long long)i * s + j] = (j == i) ? d : G[(long long)i * s + j] / d;
    __syncthreads();
  }
  // zero the strictly lower part
  for (long long e = threadIdx.x; e < (long long)s * s; e += blockDim.x) {
    const int i = (int)(e / s), j = (int)(e % s);
    if (i > j) G[e] = 0.0;
  }
  if (threadIdx.x == 0) info[blockIdx.x] = fail_sh;
  __syncthreads();
  // X = R^{-1}: column j, rows i = j, j-1, ..., 0
  for (int j = threadIdx.x; j < s; j += blockDim.x) {
    for (int i = j + 1; i < s; ++i) X[(long long)i * s + j] = 0.0;
    X[(long long)j * s + j] = 1.0 / G[(long long)j * s + j];
    for (int i = j - 1; i >= 0; --i) {
      double a = 0.0;
      for (int k = i + 1; k <= j; ++k) a = fma(G[(long long)i * s + k], X[(long long)k * s + j], a);
      X[(long long)i * s + j] = -a / G[(long long)i * s + i];
    }
  }
}

__global__ void gather_principal_kernel(const double* A, long long lda, const int32_t* Sall, int s,
                                        double lam, long long cb, long long ce, double* Gall) {
  const int32_t* S = Sall + (long long)blockIdx.y * s;
  double* G = Gall + (long long)blockIdx.y * s * s;
  const int k = blockIdx.x;  // row of the block
  const double* row = A + (long long)S[k] * lda;
  for (int l = threadIdx.x; l < s; l += blockDim.x) {
    const long long c = S[l];
    const double v = (c >= cb && c < ce) ? row[c - cb] : 0.0;
    G[(long long)k * s + l] = v + ((k == l) ? lam : 0.0);
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

}  // namespace

void launch_chol_trtri(cudaStream_t st, int batch, double* G, double* X, int s, int* info) {
  if (batch <= 0) return;
  chol_trtri_kernel<<<batch, CT, 0, st>>>(G, X, s, info);
  count_launches(1);
}

void launch_gather_principal(cudaStream_t st, int batch, const double* A, long long lda,
                             const int32_t* S, int s, double lam, long long col_begin,
                             long long col_end, double* G) {
  if (batch <= 0) return;
  dim3 grid(s, batch);
  gather_principal_kernel<<<grid, 128, 0, st>>>(A, lda, S, s, lam, col_begin, col_end, G);
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
