// window.cuh -- replicated scalar window logic of Alg 5 l.13-18 /
// Alg 3 l.14-20, shared by both Phase-2 engines.
#pragma once
#include <cmath>

#include "kpp_internal.h"

namespace kpp {

// Accumulate e = ||r_t||^2 into the window sums; at a checkpoint (t mod 2 zeta == 2 zeta - 1):
// stop test E1 <= tol^2 ||b||^2, else the adaptive rho update of Eq (weighted)
// with omega_i = a_{i-1}/a_i, a_i = (i+1)^{ln(i+1)} (reading Q8), rho = 1 - rhat^{1/zeta}
// clamped to [0, rho_max] (Q9; rho_max = 0.99 unless KPP_OPT_RHO_MAX).  Returns 0 continue, 1 tolerance met, 2 non-finite residual.
// tm = t mod 2 zeta is passed in (the persistent kernel keeps it incrementally: no 64-bit division).
// The checkpoint itself (every 2 zeta iterations: log/exp/pow) is kept out of line so that the
// persistent kernels' loop bodies stay small (instruction-cache footprint).
static __device__ __noinline__ int window_checkpoint_dev(DevState& st, long long zeta, double tol2bb, double bb,
                                                         int adaptive, bool writer, double* hist_res,
                                                         double* hist_rho, long long hist_cap) {
  st.ichk += 1;
  const bool stop = st.E1 <= tol2bb;
  if (!stop && adaptive && st.E0 > 0.0) {
    const double li = log((double)st.ichk), li1 = log((double)(st.ichk + 1));
    const double om = exp(li * li - li1 * li1);
    st.rhat = om * st.rhat + (1.0 - om) * (st.E1 / st.E0);
    double rr = 1.0 - pow(st.rhat, 1.0 / (double)zeta);
    rr = fmin(fmax(rr, 0.0), st.rho_max);
    st.rho = rr;
  }
  if (writer && st.nh < hist_cap) {
    hist_res[st.nh] = sqrt(st.E1 / bb);
    hist_rho[st.nh] = st.rho;
  }
  st.nh += 1;
  st.E0 = 0.0;
  st.E1 = 0.0;
  return stop ? 1 : 0;
}

__device__ __forceinline__ int window_step_dev(DevState& st, long long tm, double e, long long zeta,
                                               double tol2bb, double bb, int adaptive, bool writer,
                                               double* hist_res, double* hist_rho,
                                               long long hist_cap) {
  if (!isfinite(e)) return 2;
  if (tm < zeta) st.E0 += e; else st.E1 += e;
  if (tm != 2 * zeta - 1) return 0;
  return window_checkpoint_dev(st, zeta, tol2bb, bb, adaptive, writer, hist_res, hist_rho, hist_cap);
}

}  // namespace kpp
