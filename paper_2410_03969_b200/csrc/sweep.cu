// sweep.cu — K3 (proposal block H), K4 (rejection-sampling Cholesky sweep in one
// CTA) and the accepted block's inverse L^{-1} used by the fused update (K6).
//
// H (rpcholesky.hpp:366-371) = A(S', S') - F(S', :) F(S', :)^T over the b
// proposals in draw order (duplicates included).  The kernel part follows
// oracle.hpp:71-90 / 103-112 and kernels.hpp:60-64 operation by operation
// without FMA contraction, so given identical inputs it matches the CPU oracle
// up to the last-ulp difference between CUDA's and glibc's exp().
//
// The sweep (rpcholesky.hpp:167-201) replays the reference's exact operation
// order: accept iff u_i * r_i < h_ii (u = diag(H) at entry, one draw per
// proposal, counters draw0 + i), root = sqrt(h_ii), l_j = h_ji / root,
// h_pq -= l_p * l_q with two roundings.  Only the lower triangle of H is ever
// read by the reference sweep, so it is held packed in shared memory.
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

__global__ void __launch_bounds__(256) hblock_kernel(const double* __restrict__ prop,
                                                     RecordLayout lay, int b, int d, int kcur,
                                                     int kind, double sigma,
                                                     double* __restrict__ H) {
  __shared__ double sp[16][33];
  __shared__ double sq[16][33];
  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * 16 + tx;
  const int p = blockIdx.y * 16 + ty, q = blockIdx.x * 16 + tx;
  double acc = 0.0;
  for (int k0 = 0; k0 < kcur; k0 += 32) {
    for (int i = tid; i < 16 * 32; i += 256) {
      const int rr = i >> 5, kk = i & 31;
      const int pp = blockIdx.y * 16 + rr, qq = blockIdx.x * 16 + rr;
      const bool kin = k0 + kk < kcur;
      sp[rr][kk] = (pp < b && kin) ? prop[(int64_t)pp * lay.rec + lay.foff + k0 + kk] : 0.0;
      sq[rr][kk] = (qq < b && kin) ? prop[(int64_t)qq * lay.rec + lay.foff + k0 + kk] : 0.0;
    }
    __syncthreads();
#pragma unroll 8
    for (int kk = 0; kk < 32; ++kk) acc = __dadd_rn(acc, __dmul_rn(sp[ty][kk], sq[tx][kk]));
    __syncthreads();
  }
  if (p < b && q < b) {
    const double a = kernel_entry(prop + (int64_t)p * lay.rec, prop + (int64_t)q * lay.rec, lay,
                                  d, kind, sigma);
    H[(int64_t)p * b + q] = __dsub_rn(a, acc);
  }
}

void launch_hblock(const double* prop, RecordLayout lay, int b, int dpad, int d, int kcur,
                   int kind, double sigma, double* H, cudaStream_t st) {
  (void)dpad;
  const int nb = (b + 15) / 16;
  hblock_kernel<<<dim3(nb, nb), dim3(16, 16), 0, st>>>(prop, lay, b, d, kcur, kind, sigma, H);
}

constexpr int kSweepThreads = 1024;

__device__ __forceinline__ int64_t tri(int p) { return (int64_t)p * (p + 1) / 2; }

__global__ void __launch_bounds__(kSweepThreads) sweep_kernel(
    const double* __restrict__ H, int b, uint64_t seed, uint64_t draw0,
    const double* __restrict__ prop, RecordLayout lay, int* __restrict__ pos,
    int64_t* __restrict__ acc_ids, double* __restrict__ lcol, double* __restrict__ lacc_cm,
    SweepOut* out, double* hp_global) {
  extern __shared__ double sm[];
  __shared__ int s_m;
  __shared__ int s_pos[256];
  double* lcur = sm;
  double* rdraw = sm + b;
  double* udiag = sm + 2 * b;
  double* hp = hp_global ? hp_global : sm + 3 * b;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int nwarps = kSweepThreads / 32;
  for (int p = warp; p < b; p += nwarps)
    for (int q = lane; q <= p; q += 32) hp[tri(p) + q] = H[(int64_t)p * b + q];
  for (int i = tid; i < b; i += kSweepThreads) {
    rdraw[i] = u01(splitmix64_draw(seed, draw0 + (uint64_t)i));
    udiag[i] = H[(int64_t)i * b + i];
  }
  if (tid == 0) s_m = 0;
  __syncthreads();
  for (int i = 0; i < b; ++i) {
    const double hii = hp[tri(i) + i];
    if (!(__dmul_rn(udiag[i], rdraw[i]) < hii)) continue;  // uniform across the CTA
    const double root = __dsqrt_rn(hii);
    const int m = s_m;
    for (int j = i + tid; j < b; j += kSweepThreads) {
      const double lj = __ddiv_rn(hp[tri(j) + i], root);
      lcur[j] = lj;
      lcol[(int64_t)m * b + j] = lj;
    }
    __syncthreads();
    for (int p = i + 1 + warp; p < b; p += nwarps) {
      const double lp = lcur[p];
      const int64_t base = tri(p);
      for (int q = i + 1 + lane; q <= p; q += 32)
        hp[base + q] = __dsub_rn(hp[base + q], __dmul_rn(lp, lcur[q]));
    }
    if (tid == 0) {
      s_pos[m] = i;
      s_m = m + 1;
    }
    __syncthreads();
  }
  const int m = s_m;
  for (int a = tid; a < m; a += kSweepThreads) {
    pos[a] = s_pos[a];
    acc_ids[a] = (int64_t)prop[(int64_t)s_pos[a] * lay.rec];
  }
  // chol_factor(a, c) = l(pos_a, pos_c)  (rpcholesky.hpp:192-199), column-major
  for (int idx = tid; idx < m * m; idx += kSweepThreads) {
    const int c = idx / m, a = idx % m;
    lacc_cm[idx] = (a >= c) ? lcol[(int64_t)c * b + s_pos[a]] : 0.0;
  }
  if (tid == 0) out->m = m;
}

void launch_sweep(const double* H, int b, uint64_t seed, uint64_t draw0, const double* prop,
                  RecordLayout lay, int* pos, int64_t* acc_ids, double* lcol, double* lacc_cm,
                  SweepOut* out, double* scratch_hp, cudaStream_t st) {
  const size_t packed = (size_t)b * (b + 1) / 2;
  size_t smem = (size_t)3 * b * sizeof(double);
  double* hpg = nullptr;
  if (smem + packed * sizeof(double) <= 200 * 1024) {
    smem += packed * sizeof(double);
  } else {
    hpg = scratch_hp;  // global (L2-resident) fallback for large blocks
  }
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(sweep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
    attr = true;
  }
  sweep_kernel<<<1, kSweepThreads, smem, st>>>(H, b, seed, draw0, prop, lay, pos, acc_ids, lcol,
                                                lacc_cm, out, hpg);
}

// One CTA per column c of L^{-1}: forward substitution L x = e_c, axpy form.
__global__ void __launch_bounds__(256) linv_kernel(const double* __restrict__ lacc_cm, int m,
                                                   int nb, int64_t ldl, int koff,
                                                   double* __restrict__ linv_rm) {
  extern __shared__ double rhs[];
  const int c = blockIdx.x, tid = threadIdx.x;
  for (int a = tid; a < m; a += 256) rhs[a] = (a == c) ? 1.0 : 0.0;
  __syncthreads();
  for (int t = c; t < m; ++t) {
    const double xt = __ddiv_rn(rhs[t], lacc_cm[(int64_t)t * m + t]);
    __syncthreads();
    for (int a = t + 1 + tid; a < m; a += 256)
      rhs[a] = fma(-lacc_cm[(int64_t)t * m + a], xt, rhs[a]);
    if (tid == 0) rhs[t] = xt;
    __syncthreads();
  }
  for (int a = tid; a < nb; a += 256)
    linv_rm[(int64_t)perm_row(a) * ldl + c + koff] = (a >= c && a < m) ? rhs[a] : 0.0;
}

void launch_linv(const double* lacc_cm, int m, int nb, int64_t ldl, int koff, double* linv_rm,
                 cudaStream_t st) {
  if (m > 0) linv_kernel<<<m, 256, m * sizeof(double), st>>>(lacc_cm, m, nb, ldl, koff, linv_rm);
}

}  // namespace rpcb
