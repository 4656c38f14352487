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
                                               int d, int kind, double sigma) {
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
  return exp(__ddiv_rn(__dmul_rn(-0.5, dd), __dmul_rn(sigma, sigma)));
}

}  // namespace rpcb
