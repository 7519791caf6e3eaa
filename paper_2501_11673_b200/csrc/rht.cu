// rht.cu -- randomized Hadamard preprocessing.
//
// Def 1.1: Q = H D with H the Sylvester-order Hadamard matrix (H^T H = m I) and
// D = diag(d)/sqrt(m), d_i Rademacher.  K++ (Alg 5 l.2-3) solves (Q A) x = Q b; CD++
// (Alg 3 l.2-3) solves (Q A Q^T) x~ = Q b and returns x = Q^T x~ = D H x~ (l.16).
// Non-power-of-2 sizes are padded (zero rows for K++; unit diagonal for CD++, R4).
//
// The transforms are HBM-bound butterflies.  `fht_rows_pass` applies RSTG consecutive butterfly
// stages (half-sizes 2^k .. 2^(k+RSTG-1)) along the ROW index of a row-major matrix: a CTA owns a
// group of 2^RSTG rows (stride 2^k) times a chunk of 128 columns, each thread holds one column of
// the group in registers, so every pass reads and writes the matrix once with coalesced rows.
// log2(m) stages take ceil(log2 m / RSTG) passes; the first pass also applies D (and the padding).
// The two-sided CD++ transform is H (D A D) H = H (H (D A D))^T (D A D and the result are
// symmetric): row pass, tiled transpose, row pass.
// Sign stream (binding convention shared with the oracle's independent implementation, DESIGN.md
// R3): d_i = -1 iff the lowest bit of word (i mod 4) of Philox-4x32-10((lo32(i/4), hi32(i/4), 3, 0),
// (lo32 seed, hi32 seed)) is set.
#include <cstdint>

#include "kpp_internal.h"

namespace kpp {
namespace {

constexpr int RSTG = 5;        // butterfly stages per pass (32 values per thread)
constexpr int RCOLS = 128;     // columns per CTA

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

// dvec[i] = d_i / sqrt(m2) for i < m, 0 for padding (scale applied by the first pass)
__global__ void rht_sign_kernel(uint64_t seed, long long m, long long m2, double* dvec) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= m2) return;
  const unsigned long long c = (unsigned long long)i >> 2;
  uint32_t w[4] = {(uint32_t)(c & 0xffffffffull), (uint32_t)(c >> 32), 3u, 0u};
  philox4(w, (uint32_t)(seed & 0xffffffffull), (uint32_t)(seed >> 32));
  const double sc = 1.0 / sqrt((double)m2);
  dvec[i] = i < m ? (((w[i & 3] & 1u) ? -1.0 : 1.0) * sc) : 0.0;
}

// One pass of stages k .. k+ns-1 along rows.  src (first pass: the user's matrix, rows < m_src,
// ld lds, scaled by rowscale[i] (and colscale[j] when given); rows beyond m_src are zero, or
// unit-diagonal when pad_diag) -> dst (m2 x n, ld ldd).  src == dst for later passes.
__global__ void __launch_bounds__(RCOLS) fht_rows_pass(const double* src, long long lds, long long m_src,
                                                       long long n_src, double* dst, long long ldd, long long n,
                                                       int k, int ns, const double* rowscale,
                                                       const double* colscale, int pad_diag) {
  const long long j = blockIdx.y * (long long)RCOLS + threadIdx.x;
  const long long g = blockIdx.x;  // group: bits k .. k+ns-1 of the row index are zero
  const long long lo = g & ((1LL << k) - 1), hi = g >> k;
  const long long base = (hi << (k + ns)) | lo;
  const int cnt = 1 << ns;
  double v[1 << RSTG];
#pragma unroll
  for (int i = 0; i < (1 << RSTG); ++i) {
    double a = 0.0;
    if (i < cnt && j < n) {
      const long long r = base + ((long long)i << k);
      if (rowscale) {
        if (r < m_src && j < n_src) {
          a = src[r * lds + j] * rowscale[r];
          if (colscale) a *= colscale[j];
        } else if (pad_diag && r == j) {
          a = rowscale[r] * colscale[j];  // A_pad = [[A, 0], [0, I]] scaled by D on both sides
        }
      } else {
        a = src[r * lds + j];
      }
    }
    v[i] = a;
  }
#pragma unroll
  for (int hh = 1; hh < (1 << RSTG); hh <<= 1) {
    if (hh >= cnt) break;
#pragma unroll
    for (int i0 = 0; i0 < (1 << RSTG); i0 += 2 * hh)
#pragma unroll
      for (int i = i0; i < i0 + hh; ++i) {
        const double a = v[i], b = v[i + hh];
        v[i] = a + b;
        v[i + hh] = a - b;
      }
  }
  if (j < n) {
#pragma unroll
    for (int i = 0; i < (1 << RSTG); ++i)
      if (i < cnt) dst[(base + ((long long)i << k)) * ldd + j] = v[i];
  }
}

__global__ void transpose_kernel(const double* src, double* dst, long long n) {
  __shared__ double tile[32][33];
  const long long bx = blockIdx.x * 32LL, by = blockIdx.y * 32LL;
  for (int yy = threadIdx.y; yy < 32; yy += 8) {
    const long long r = by + yy, c = bx + threadIdx.x;
    tile[yy][threadIdx.x] = (r < n && c < n) ? src[r * n + c] : 0.0;
  }
  __syncthreads();
  for (int yy = threadIdx.y; yy < 32; yy += 8) {
    const long long r = bx + yy, c = by + threadIdx.x;
    if (r < n && c < n) dst[r * n + c] = tile[threadIdx.x][yy];
  }
}

// back-rotation helpers: out[i] = dvec[i] * v[i] * m2 ... (see launch_rht_vec)
__global__ void scale_kernel(const double* v, const double* dvec, long long n, double* out) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) out[i] = v[i] * dvec[i];
}

}  // namespace

void launch_rht_signs(cudaStream_t st, uint64_t seed, long long m, long long m2, double* dvec) {
  rht_sign_kernel<<<(unsigned)((m2 + 255) / 256), 256, 0, st>>>(seed, m, m2, dvec);
  count_launches(1);
}

// dst = H (diag(rowscale) src_pad [diag(colscale)]) along rows: m2 = 2^L rows, n columns.
void launch_fht_rows(cudaStream_t st, const double* src, long long lds, long long m_src, long long n_src,
                     double* dst, long long ldd, long long m2, long long n, const double* rowscale,
                     const double* colscale, int pad_diag) {
  int L = 0;
  while ((1LL << L) < m2) ++L;
  bool first = true;
  for (int k = 0; k < L || first; k += RSTG) {
    const int ns = L - k < RSTG ? L - k : RSTG;
    dim3 grid((unsigned)(m2 >> ns), (unsigned)((n + RCOLS - 1) / RCOLS));
    if (first)
      fht_rows_pass<<<grid, RCOLS, 0, st>>>(src, lds, m_src, n_src, dst, ldd, n, k, ns, rowscale, colscale,
                                             pad_diag);
    else
      fht_rows_pass<<<grid, RCOLS, 0, st>>>(dst, ldd, m2, n, dst, ldd, n, k, ns, nullptr, nullptr, 0);
    count_launches(1);
    first = false;
    if (L == 0) break;
  }
}

void launch_transpose(cudaStream_t st, const double* src, double* dst, long long n) {
  dim3 grid((unsigned)((n + 31) / 32), (unsigned)((n + 31) / 32));
  transpose_kernel<<<grid, dim3(32, 8), 0, st>>>(src, dst, n);
  count_launches(1);
}

void launch_scale(cudaStream_t st, const double* v, const double* dvec, long long n, double* out) {
  scale_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(v, dvec, n, out);
  count_launches(1);
}

}  // namespace kpp
