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
  // 64 < m <= 96: two warp columns of half the accumulators, two CTAs per SM (measured
  // 9% faster than the ping-pong pair at C4 rounds 1-2; slower for m > 96)
  if (nf > 8 && nf <= 12) return launch_update_wc2(p, (nf + 1) / 2, st);
  if (nf <= 16) return launch_update_wc1(p, nf, st);
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
                                       double* __restrict__ idS) {
  const int n = blockIdx.x;
  const int m = m_dev ? *m_dev : m_host;
  const int dst = perm_row(n);
  double* xr = xs + (int64_t)dst * dpad;
  double* fr = fs + (int64_t)dst * ldfs;
  if (n < m) {
    const double* rec = prop + (int64_t)pos[n] * lay.rec;
    for (int i = threadIdx.x; i < dpad; i += blockDim.x) xr[i] = rec[lay.xoff + i];
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
                            double* sqnS, double* idS, cudaStream_t st, const int* m_dev) {
  const int kpad = std::min<int64_t>(ldfs, ((kcur + 15) / 16) * 16);
  gather_accepted_kernel<<<nb, 256, 0, st>>>(prop, lay, pos, m, m_dev, kcur, kpad, dpad, xs, fs,
                                             ldfs, sqnS, idS);
}

// Tiled C[8 x 128] = L^{-1}[8 rows, :m] * F_S[:m, 128 columns]; each output summed over
// c ascending (deterministic), negated.
__global__ void __launch_bounds__(256) bprime_kernel(const double* __restrict__ linv_rm,
                                                     int64_t ldl, int koff,
                                                     const double* __restrict__ prop,
                                                     RecordLayout lay, const int* __restrict__ pos,
                                                     const int* __restrict__ m_dev, int kcur,
                                                     double* __restrict__ bp, int64_t ldbp) {
  __shared__ double sL[8][257];
  __shared__ double sF[16][129];
  const int m = *m_dev;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int n = blockIdx.y * 8 + ty;
  const int k0 = blockIdx.x * 128;
  for (int i = threadIdx.x; i < 8 * m; i += 256) {
    const int r = i / m, c = i % m;
    sL[r][c] = linv_rm[(int64_t)perm_row(blockIdx.y * 8 + r) * ldl + c + koff];
  }
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int c0 = 0; c0 < m; c0 += 16) {
    __syncthreads();
    for (int i = threadIdx.x; i < 16 * 128; i += 256) {
      const int cc = i >> 7, kk = i & 127;
      const int c = c0 + cc, k = k0 + kk;
      sF[cc][kk] = (c < m && k < kcur) ? prop[(int64_t)pos[c] * lay.rec + lay.foff + k] : 0.0;
    }
    __syncthreads();
    const int cend = min(16, m - c0);
    for (int cc = 0; cc < cend; ++cc) {
      const double l = sL[ty][c0 + cc];
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[j] = fma(l, sF[cc][tx + 32 * j], acc[j]);
    }
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int k = k0 + tx + 32 * j;
    if (k < kcur) bp[(int64_t)perm_row(n) * ldbp + k] = -acc[j];
  }
}

void launch_bprime(const double* linv_rm, int64_t ldl, int koff, const double* prop,
                   RecordLayout lay, const int* pos, const int* m_dev, int m_max, int kcur,
                   double* bp, int64_t ldbp, cudaStream_t st) {
  if (kcur <= 0 || m_max <= 0) return;
  dim3 grid((unsigned)((kcur + 127) / 128), (unsigned)((m_max + 7) / 8));
  bprime_kernel<<<grid, 256, 0, st>>>(linv_rm, ldl, koff, prop, lay, pos, m_dev, kcur, bp, ldbp);
}

}  // namespace rpcb
