// update.cu — dispatch of the fused round-update kernel (update_impl.cuh) and the
// per-round operand gather.
#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace rpcb {

int launch_update_wc1(const UpdateParams& p, int nf, cudaStream_t st);
int launch_update_wc2(const UpdateParams& p, int nfw, cudaStream_t st);
int launch_update_cols(const UpdateParams& p, int nf, cudaStream_t st);

// Fragment count nf = ceil(m / 8).  nf <= 16: two ping-pong warp groups per CTA, each
// with 64-row tiles and a single warp column (no padded columns).  16 < nf <= 32: one
// group of 8 warps, two warp columns, 64-row tiles.
int update_tile_rows(int m) {
  const int nf = std::max(1, (m + 7) / 8);
  if (nf <= 32) return 64;
  return -1;
}

int launch_update(const UpdateParams& p, cudaStream_t st) {
  const int nf = std::max(1, (p.m + 7) / 8);
  if (p.columns_only && nf <= 16) return launch_update_cols(p, nf, st);
  // m <= 128: two ping-pong groups, one warp column, A(R,S) L^{-T} from registers
  // (update_regp2: L^{-1} was stored in that path's column order)
  if (update_regp2(p.m)) return launch_update_wc1(p, nf, st);
  if (nf <= 32) return launch_update_wc2(p, (nf + 1) / 2, st);
  return -1;
}

// Accepted-pivot operands for the update: rows stored at perm_row(n) of
// [256][ld] buffers (zero rows beyond m, zero columns [kcur, round16(kcur))).
__global__ void gather_accepted_kernel(const double* __restrict__ prop, RecordLayout lay,
                                       const int* __restrict__ pos, int m_host,
                                       const int* __restrict__ m_dev, int kcur, int kpad,
                                       int dpad, double* __restrict__ xs, double* __restrict__ fs,
                                       int64_t ldfs, double* __restrict__ sqnS,
                                       double* __restrict__ idS, double xscale) {
  const int n = blockIdx.x;
  const int m = m_dev ? *m_dev : m_host;
  const int dst = perm_row(n);
  double* xr = xs + (int64_t)dst * dpad;
  double* fr = fs + (int64_t)dst * ldfs;
  if (n < m) {
    const double* rec = prop + (int64_t)pos[n] * lay.rec;
    for (int i = threadIdx.x; i < dpad; i += blockDim.x) xr[i] = xscale * rec[lay.xoff + i];
    for (int k = threadIdx.x; k < kpad; k += blockDim.x) fr[k] = k < kcur ? rec[lay.foff + k] : 0.0;
    if (threadIdx.x == 0) {
      sqnS[n] = rec[1];
      idS[n] = rec[0];
    }
  } else {
    for (int i = threadIdx.x; i < dpad; i += blockDim.x) xr[i] = 0.0;
    for (int k = threadIdx.x; k < kpad; k += blockDim.x) fr[k] = 0.0;
    if (threadIdx.x == 0) {
      sqnS[n] = 0.0;
      idS[n] = -1.0;
    }
  }
}

void launch_gather_accepted(const double* prop, RecordLayout lay, const int* pos, int m, int nb,
                            int kcur, int dpad, double* xs, double* fs, int64_t ldfs,
                            double* sqnS, double* idS, cudaStream_t st, const int* m_dev,
                            double xscale) {
  const int kpad = std::min<int64_t>(ldfs, ((kcur + 15) / 16) * 16);
  gather_accepted_kernel<<<nb, 256, 0, st>>>(prop, lay, pos, m, m_dev, kcur, kpad, dpad, xs, fs,
                                             ldfs, sqnS, idS, xscale);
}

// B' = -L^{-1} F_S (m x kcur).  One CTA per 8-column slice of F_S: the slice (m x 8, one
// gather of 64-byte row pieces) is staged in shared memory once, L^{-1} rows are read through
// L1 (the 8 threads of a column group share each row), and each thread sums its outputs over
// c ascending (deterministic; the zeros above L^{-1}'s diagonal are skipped, which leaves
// every sum bitwise unchanged).
constexpr int kBpCols = 8;
__global__ void __launch_bounds__(256) bprime_kernel(const double* __restrict__ linv_rm,
                                                     int64_t ldl, int koff,
                                                     const double* __restrict__ prop,
                                                     RecordLayout lay, const int* __restrict__ pos,
                                                     const int* __restrict__ m_dev, int m_host,
                                                     int kcur, double* __restrict__ bp,
                                                     int64_t ldbp, const double* __restrict__ lext,
                                                     int m_full, int g0, int kprop) {
  extern __shared__ double sF[];  // [m][kBpCols]
  const int m = m_dev ? *m_dev : m_host;
  const int k0 = blockIdx.x * kBpCols;
  for (int i = threadIdx.x; i < m * kBpCols; i += blockDim.x) {
    const int c = i / kBpCols, kk = i % kBpCols, k = k0 + kk;
    double v = 0.0;
    if (k < kprop) v = __ldg(prop + (int64_t)pos[c] * lay.rec + lay.foff + k);
    else if (k < kcur) v = __ldg(lext + (int64_t)(k - kprop) * m_full + g0 + c);
    sF[i] = v;
  }
  __syncthreads();
  const int kk = threadIdx.x % kBpCols, a0 = threadIdx.x / kBpCols;
  constexpr int kRowStep = 256 / kBpCols;  // 32
  const int k = k0 + kk;
  for (int ab = 0; ab < m; ab += 4 * kRowStep) {
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    const double* lr[4];
    int amax = -1;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int a = ab + a0 + kRowStep * j;
      lr[j] = linv_rm + (int64_t)perm_row(a < m ? a : 0) * ldl;
      if (a < m) amax = a;
    }
    for (int c = 0; c <= amax; ++c) {
      const double f = sF[c * kBpCols + kk];
      const int col = linv_slot(c, m, koff, 1);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int a = ab + a0 + kRowStep * j;
        if (c <= a && a < m) acc[j] = fma(__ldg(lr[j] + col), f, acc[j]);
      }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int a = ab + a0 + kRowStep * j;
      if (a < m && k < kcur) bp[(int64_t)perm_row(a) * ldbp + k] = -acc[j];
    }
  }
}

void launch_bprime(const double* linv_rm, int64_t ldl, int koff, const double* prop,
                   RecordLayout lay, const int* pos, const int* m_dev, int m_max, int kcur,
                   double* bp, int64_t ldbp, cudaStream_t st, const double* lext, int m_full,
                   int g0, int kprop) {
  if (kcur <= 0 || m_max <= 0) return;
  const unsigned grid = (unsigned)((kcur + kBpCols - 1) / kBpCols);
  bprime_kernel<<<grid, 256, sizeof(double) * kBpCols * m_max, st>>>(
      linv_rm, ldl, koff, prop, lay, pos, m_dev, m_max, kcur, bp, ldbp, lext, m_full, g0,
      lext ? kprop : kcur);
}

}  // namespace rpcb
