// update.cu — dispatch of the fused round-update kernel (update_impl.cuh) and the
// per-round operand gather.
#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace rpcb {

int launch_update_wc1(const UpdateParams& p, int nf, cudaStream_t st);
int launch_update_wc2(const UpdateParams& p, int nfw, cudaStream_t st);

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

}  // namespace rpcb
