// krr_core.cu — the KRR preconditioner's k x k core on the device, hand-written
// (Preconditioner, krr.hpp:30-70):  core = F^T F + mu I,  its Cholesky factor, and
// apply_inverse's solve with it.  No BLAS/LAPACK library is involved.
//
//   core_syrk   F^T F on the FP64 tensor cores (mma.sync m8n8k4 -> DMMA): lower 64 x 64
//               output tiles x a fixed number of row slices (chosen from k only, so the
//               result is bit-reproducible); the slices are summed in slice order.
//   core_potrf  right-looking blocked Cholesky, 64-column panels: one CTA factors the
//               diagonal block in shared memory, the panel below is solved row by row, the
//               trailing lower triangle gets the rank-64 update.
//   core_potrs  L L^T z = t for one vector: one CTA, 64-row blocks; a warp solves the
//               diagonal block with shuffles, the whole CTA applies its update.
//
// Storage: row-major [kc][kc], kc = k rounded up to 64; rows/columns >= k hold the
// identity (so padded entries of every solve stay 0).  Only the lower triangle is read.
#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace rpcb {

namespace {

constexpr int kT = 64;       // tile / panel width
constexpr int kSyrkRows = 32;  // F rows staged per step
constexpr int kSyrkLd = 68;    // padded smem row (68 doubles: conflict-free fragment loads)

__host__ __device__ inline int n_lower_tiles(int nb) { return nb * (nb + 1) / 2; }
__device__ inline void tile_of(int t, int& bi, int& bj) {  // t -> (bi >= bj), row by row
  bi = (int)((sqrtf(8.0f * t + 1.0f) - 1.0f) * 0.5f);
  while (bi * (bi + 1) / 2 > t) --bi;
  while ((bi + 1) * (bi + 2) / 2 <= t) ++bi;
  bj = t - bi * (bi + 1) / 2;
}

// part[s][tile][64][64] = sum over rows of slice s of F(r, I)^T F(r, J).
__global__ void __launch_bounds__(256) syrk_partial_kernel(const double* __restrict__ F,
                                                           int64_t ldf, int64_t n, int k,
                                                           int slices,
                                                           double* __restrict__ part) {
  __shared__ __align__(16) double FI[kSyrkRows][kSyrkLd];
  __shared__ __align__(16) double FJ[kSyrkRows][kSyrkLd];
  const int tile = blockIdx.x, s = blockIdx.y;
  int bi, bj;
  tile_of(tile, bi, bj);
  const int i0 = bi * kT, j0 = bj * kT;
  const int64_t rs = (n + slices - 1) / slices;
  const int64_t r0 = (int64_t)s * rs, r1 = r0 + rs < n ? r0 + rs : n;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;  // warp w: output rows 8w..8w+7
  double acc[8][2];
#pragma unroll
  for (int f = 0; f < 8; ++f) acc[f][0] = acc[f][1] = 0.0;
  for (int64_t rb = r0; rb < r1; rb += kSyrkRows) {
    // stage 32 rows x 64 columns of F for the I and J column blocks (zero beyond n, k)
    for (int e = threadIdx.x; e < kSyrkRows * kT; e += blockDim.x) {
      const int rr = e / kT, c = e % kT;
      const int64_t r = rb + rr;
      const bool rok = r < r1;
      FI[rr][c] = (rok && i0 + c < k) ? F[r * ldf + i0 + c] : 0.0;
      FJ[rr][c] = (rok && j0 + c < k) ? F[r * ldf + j0 + c] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < kSyrkRows; kk += 4) {
      const int r = kk + (lane & 3);
      const double a = FI[r][8 * w + (lane >> 2)];  // A = F(r, I)^T: 8 x 4 row-major
#pragma unroll
      for (int f = 0; f < 8; ++f) {
        const double b = FJ[r][8 * f + (lane >> 2)];  // B = F(r, J): 4 x 8 col-major
        dmma884(acc[f][0], acc[f][1], a, b);
      }
    }
    __syncthreads();
  }
  double* out = part + ((int64_t)s * gridDim.x + tile) * (kT * kT);
  const int row = 8 * w + (lane >> 2);
#pragma unroll
  for (int f = 0; f < 8; ++f) {
    const int col = 8 * f + 2 * (lane & 3);
    out[row * kT + col] = acc[f][0];
    out[row * kT + col + 1] = acc[f][1];
  }
}

// core(i, j) = sum_s part[s] (slice order) + mu [i == j]; identity outside k x k; lower only.
__global__ void syrk_reduce_kernel(const double* __restrict__ part, int slices, int ntiles, int k,
                                   double mu, double* __restrict__ core, int64_t kc) {
  const int tile = blockIdx.x;
  int bi, bj;
  tile_of(tile, bi, bj);
  for (int e = threadIdx.x; e < kT * kT; e += blockDim.x) {
    const int ii = e / kT, jj = e % kT;
    const int i = bi * kT + ii, j = bj * kT + jj;
    if (j > i) continue;
    double v;
    if (i >= k || j >= k) {
      v = i == j ? 1.0 : 0.0;
    } else {
      v = 0.0;
      for (int s = 0; s < slices; ++s) v += part[((int64_t)s * ntiles + tile) * (kT * kT) + e];
      if (i == j) v += mu;
    }
    core[(int64_t)i * kc + j] = v;
  }
}

// Unblocked Cholesky of the 64 x 64 diagonal block at (j0, j0), in shared memory.
__global__ void __launch_bounds__(256) potrf_diag_kernel(double* __restrict__ A, int64_t kc,
                                                         int j0, int* info) {
  __shared__ double a[kT][kT + 1];
  __shared__ int bad;
  for (int e = threadIdx.x; e < kT * kT; e += blockDim.x) {
    const int i = e / kT, j = e % kT;
    a[i][j] = j <= i ? A[(int64_t)(j0 + i) * kc + j0 + j] : 0.0;
  }
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  for (int c = 0; c < kT; ++c) {
    const double dc = a[c][c];
    if (!(dc > 0.0)) {  // not positive definite: report, keep the block finite
      if (threadIdx.x == 0) bad = 1;
      break;
    }
    const double root = sqrt(dc);
    __syncthreads();  // everyone has read a[c][c]
    if (threadIdx.x == 0) a[c][c] = root;
    for (int i = c + 1 + threadIdx.x; i < kT; i += blockDim.x) a[i][c] = a[i][c] / root;
    __syncthreads();
    for (int e = threadIdx.x; e < (kT - c - 1) * (kT - c - 1); e += blockDim.x) {
      const int i = c + 1 + e / (kT - c - 1), j = c + 1 + e % (kT - c - 1);
      if (j <= i) a[i][j] -= a[i][c] * a[j][c];
    }
    __syncthreads();
  }
  __syncthreads();
  if (bad) {
    if (threadIdx.x == 0) *info = j0 + 1;
    return;
  }
  for (int e = threadIdx.x; e < kT * kT; e += blockDim.x) {
    const int i = e / kT, j = e % kT;
    if (j <= i) A[(int64_t)(j0 + i) * kc + j0 + j] = a[i][j];
  }
}

// Panel below the diagonal block: row i <- row i * L_jj^{-T} (forward substitution per row).
__global__ void __launch_bounds__(128) potrf_panel_kernel(double* __restrict__ A, int64_t kc,
                                                          int j0) {
  __shared__ double l[kT][kT + 1];
  for (int e = threadIdx.x; e < kT * kT; e += blockDim.x) {
    const int i = e / kT, j = e % kT;
    l[i][j] = j <= i ? A[(int64_t)(j0 + i) * kc + j0 + j] : 0.0;
  }
  __syncthreads();
  const int64_t i = j0 + kT + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= kc) return;
  double* row = A + i * kc + j0;
  double x[kT];
#pragma unroll
  for (int c = 0; c < kT; ++c) x[c] = row[c];
#pragma unroll
  for (int c = 0; c < kT; ++c) {
    double v = x[c];
#pragma unroll
    for (int t = 0; t < c; ++t) v -= x[t] * l[c][t];
    x[c] = v / l[c][c];
  }
#pragma unroll
  for (int c = 0; c < kT; ++c) row[c] = x[c];
}

// Trailing update of the lower 64 x 64 tiles right of the panel: A(I, J) -= P(I) P(J)^T.
__global__ void __launch_bounds__(256) potrf_update_kernel(double* __restrict__ A, int64_t kc,
                                                           int j0) {
  constexpr int kH = kT / 2;  // panel columns staged per pass (static smem < 48 KB)
  __shared__ double PI[kT][kH + 1], PJ[kT][kH + 1];
  int bi, bj;
  tile_of(blockIdx.x, bi, bj);
  const int b0 = (j0 + kT) / kT;  // first trailing block
  bi += b0;
  bj += b0;
  const int i0 = bi * kT, jj0 = bj * kT;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;  // 4 x 4 outputs per thread
  double acc[4][4] = {};
  for (int h = 0; h < kT; h += kH) {
    __syncthreads();
    for (int e = threadIdx.x; e < kT * kH; e += blockDim.x) {
      const int r = e / kH, c = e % kH;
      PI[r][c] = A[(int64_t)(i0 + r) * kc + j0 + h + c];
      PJ[r][c] = A[(int64_t)(jj0 + r) * kc + j0 + h + c];
    }
    __syncthreads();
    for (int c = 0; c < kH; ++c) {
      double a[4], b[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        a[q] = PI[ty + 16 * q][c];
        b[q] = PJ[tx + 16 * q][c];
      }
#pragma unroll
      for (int p = 0; p < 4; ++p)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[p][q] += a[p] * b[q];
    }
  }
#pragma unroll
  for (int p = 0; p < 4; ++p)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int i = i0 + ty + 16 * p, j = jj0 + tx + 16 * q;
      if (j <= i) A[(int64_t)i * kc + j] -= acc[p][q];
    }
}

// L L^T z = t in place (t: kc doubles).  One CTA of 256 threads.
__global__ void __launch_bounds__(256) potrs_kernel(const double* __restrict__ L, int64_t kc,
                                                    double* __restrict__ t) {
  extern __shared__ double v[];  // [kc]
  __shared__ double blk[kT];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < kc; i += blockDim.x) v[i] = t[i];
  __syncthreads();
  const int nb = (int)(kc / kT);
  // forward: L y = t
  for (int b = 0; b < nb; ++b) {
    const int j0 = b * kT;
    if (w == 0) {
      double y0 = v[j0 + lane], y1 = v[j0 + 32 + lane];  // rows lane, lane + 32 of the block
      for (int c = 0; c < kT; ++c) {
        const double mine = c < 32 ? y0 : y1;
        double yc = __shfl_sync(0xffffffffu, mine, c & 31);
        yc = yc / L[(int64_t)(j0 + c) * kc + j0 + c];
        if (lane == (c & 31)) {
          if (c < 32) y0 = yc; else y1 = yc;
        }
        if (lane > c) y0 -= L[(int64_t)(j0 + lane) * kc + j0 + c] * yc;
        if (lane + 32 > c) y1 -= L[(int64_t)(j0 + lane + 32) * kc + j0 + c] * yc;
      }
      blk[lane] = y0;
      blk[lane + 32] = y1;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < kT; i += blockDim.x) v[j0 + i] = blk[i];
    for (int64_t i = j0 + kT + threadIdx.x; i < kc; i += blockDim.x) {
      const double* row = L + i * kc + j0;
      double s = v[i];
      for (int c = 0; c < kT; ++c) s -= row[c] * blk[c];
      v[i] = s;
    }
    __syncthreads();
  }
  // backward: L^T z = y
  for (int b = nb - 1; b >= 0; --b) {
    const int j0 = b * kT;
    if (w == 0) {
      double z0 = v[j0 + lane], z1 = v[j0 + 32 + lane];
      for (int c = kT - 1; c >= 0; --c) {
        const double mine = c < 32 ? z0 : z1;
        double zc = __shfl_sync(0xffffffffu, mine, c & 31);
        zc = zc / L[(int64_t)(j0 + c) * kc + j0 + c];
        if (lane == (c & 31)) {
          if (c < 32) z0 = zc; else z1 = zc;
        }
        // rows r < c of the block: z_r -= L(c, r) z_c
        if (lane < c) z0 -= L[(int64_t)(j0 + c) * kc + j0 + lane] * zc;
        if (lane + 32 < c) z1 -= L[(int64_t)(j0 + c) * kc + j0 + lane + 32] * zc;
      }
      blk[lane] = z0;
      blk[lane + 32] = z1;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < kT; i += blockDim.x) v[j0 + i] = blk[i];
    for (int i = threadIdx.x; i < j0; i += blockDim.x) {
      double s = v[i];
      for (int c = 0; c < kT; ++c) s -= L[(int64_t)(j0 + c) * kc + i] * blk[c];
      v[i] = s;
    }
    __syncthreads();
  }
  for (int i = threadIdx.x; i < kc; i += blockDim.x) t[i] = v[i];
}

int syrk_slices(int k) {
  const int ntiles = n_lower_tiles((k + kT - 1) / kT);
  const int want = (2 * 148 + ntiles - 1) / ntiles;  // >= ~2 CTAs per SM; depends on k only
  return want < 1 ? 1 : (want > 64 ? 64 : want);
}

}  // namespace

int64_t core_dim(int k) { return (int64_t)((k + kT - 1) / kT) * kT; }

size_t core_syrk_scratch_doubles(int k) {
  return (size_t)syrk_slices(k) * n_lower_tiles((k + kT - 1) / kT) * kT * kT;
}

void launch_core_syrk(const double* F, int64_t ldf, int64_t n, int k, double mu, double* core,
                      double* scratch, cudaStream_t st) {
  const int64_t kc = core_dim(k);
  const int nb = (int)(kc / kT), ntiles = n_lower_tiles(nb), slices = syrk_slices(k);
  syrk_partial_kernel<<<dim3(ntiles, slices), 256, 0, st>>>(F, ldf, n, k, slices, scratch);
  syrk_reduce_kernel<<<ntiles, 256, 0, st>>>(scratch, slices, ntiles, k, mu, core, kc);
}

void launch_core_potrf(double* core, int64_t kc, int* info, cudaStream_t st) {
  const int nb = (int)(kc / kT);
  for (int b = 0; b < nb; ++b) {
    const int j0 = b * kT;
    potrf_diag_kernel<<<1, 256, 0, st>>>(core, kc, j0, info);
    const int rest = (int)(kc - j0 - kT);
    if (rest <= 0) break;
    potrf_panel_kernel<<<(rest + 127) / 128, 128, 0, st>>>(core, kc, j0);
    potrf_update_kernel<<<n_lower_tiles(rest / kT), 256, 0, st>>>(core, kc, j0);
  }
}

void launch_core_potrs(const double* L, int64_t kc, double* t, cudaStream_t st) {
  const size_t smem = sizeof(double) * (size_t)kc;
  ensure_smem_attr((const void*)potrs_kernel, (int)std::max<size_t>(smem, 1));
  potrs_kernel<<<1, 256, smem, st>>>(L, kc, t);
}

}  // namespace rpcb
