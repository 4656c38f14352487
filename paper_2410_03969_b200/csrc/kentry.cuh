#pragma once
// kentry.cuh — one kernel-matrix entry A(p, q) from two point records
// (record layout: [0] global id, [1] ||x||^2, [xoff, xoff+d) coordinates).
// Follows oracle.hpp:71-90 (Gram trick: ((-2 dot) + sqn_p) + sqn_q, clamp at 0,
// same global index pinned to 0), oracle.hpp:103-112 (direct distances, ascending
// coordinate order) and kernels.hpp:60-64 operation by operation, no FMA contraction.
#include "common.cuh"
#include "kernels.h"

namespace rpcb {

__device__ __forceinline__ double kernel_entry(const double* __restrict__ rp,
                                               const double* __restrict__ rq, RecordLayout lay,
                                               int d, int kind, int kfun, double sigma) {
  const double* xp = rp + lay.xoff;
  const double* xq = rq + lay.xoff;
  if (kind == kL1) {
    double s = 0.0;
    for (int j = 0; j < d; ++j) s = __dadd_rn(s, fabs(__dsub_rn(xp[j], xq[j])));
    return exp(__ddiv_rn(-s, sigma));
  }
  double dd;
  if (kind == kGaussDirect) {
    dd = 0.0;
    for (int j = 0; j < d; ++j) {
      const double t = __dsub_rn(xp[j], xq[j]);
      dd = __dadd_rn(dd, __dmul_rn(t, t));
    }
  } else {
    double dot = 0.0;
    for (int j = 0; j < d; ++j) dot = __dadd_rn(dot, __dmul_rn(xp[j], xq[j]));
    dd = __dadd_rn(__dadd_rn(-2.0 * dot, rp[1]), rq[1]);
    if (dd < 0.0) dd = 0.0;
    if (rp[0] == rq[0]) dd = 0.0;  // same global index pinned to 0 (oracle.hpp:80-88)
  }
  // kernel_from_sq_dist (kernels.hpp:60-79)
  if (kfun == kFunMatern32) {
    const double z = __dmul_rn(1.7320508075688772, __ddiv_rn(__dsqrt_rn(dd), sigma));
    return __dmul_rn(__dadd_rn(1.0, z), exp(-z));
  }
  if (kfun == kFunMatern52) {
    const double rho2 = __ddiv_rn(dd, __dmul_rn(sigma, sigma));
    const double z = __dsqrt_rn(__dmul_rn(5.0, rho2));
    return __dmul_rn(__dadd_rn(__dadd_rn(1.0, z), __dmul_rn(5.0 / 3.0, rho2)), exp(-z));
  }
  return exp(__ddiv_rn(__dmul_rn(-0.5, dd), __dmul_rn(sigma, sigma)));
}

}  // namespace rpcb
