// lowmem.cu — low-memory variant (accelerated_rpcholesky_lowmem, rpcholesky.hpp:408-485):
// update dispatch and the small replicated per-round kernels.
//
// Per round, on the b proposals S' and the kold pivots S (all replicated):
//   F(S', :) = A(S', S) L^{-T}            kprop + gemm   (the reference's W_prop^T,
//                                                          rpcholesky.hpp:441-444)
//   H = A(S', S') - F(S', :) F(S', :)^T    hblock (sweep.cu), then the rejection sweep
//   L_new = [[L, 0], [F_S, L_sel]]          append (rpcholesky.hpp:470-475)
//   Linv_new rows [kold, kold+m) = [-L_sel^{-1} F_S L^{-1} | L_sel^{-1}]   gemm x2
#include <algorithm>

#include "common.cuh"
#include "kentry.cuh"
#include "kernels.h"

namespace rpcb {

int launch_lowmem_wc1(const LowmemParams& p, int nf, cudaStream_t st);
int launch_lowmem_wc2(const LowmemParams& p, int nfw, cudaStream_t st);

int launch_lowmem(const LowmemParams& p, cudaStream_t st) {
  const int nf = std::max(1, (p.m + 7) / 8);
  if (nf <= 16) {
    const int r = launch_lowmem_wc1(p, nf, st);
    if (r != -1) return r;
    // -1: two groups' resident X tiles exceed shared memory (large d): one group of 8 warps
  }
  if (nf <= 32) return launch_lowmem_wc2(p, (nf + 1) / 2, st);
  return -1;
}

// C = alpha op(A) op(B) (+ beta C) for the low-memory path's small products (b x k x k,
// m x k x k).  32 x 32 output tiles (enough CTAs for M ~ 120 rows), 32-wide k chunks staged
// in shared memory with the next chunk prefetched into registers.  Each output is one
// ascending-k FMA chain, the same operation order as before the retiling (bitwise equal).
__global__ void __launch_bounds__(256) gemm_kernel(int M, int N, int K, double alpha,
                                                   const double* __restrict__ A, int64_t lda, int ta,
                                                   const double* __restrict__ B, int64_t ldb, int tb,
                                                   double beta, double* __restrict__ Cm, int64_t ldc) {
  constexpr int T = 32, KC = 32;
  __shared__ double As[KC][T + 1];  // [k][i]
  __shared__ double Bs[KC][T + 1];  // [k][j]
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int i0 = blockIdx.y * T, j0 = blockIdx.x * T;
  double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
  double ra[4], rb[4];
  auto fetch = [&](int k0) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int e = threadIdx.x + 256 * r;
      int kk, ii;
      if (ta) { ii = e & 31; kk = e >> 5; } else { kk = e & 31; ii = e >> 5; }
      const int i = i0 + ii, k = k0 + kk;
      ra[r] = (i < M && k < K) ? (ta ? A[(int64_t)k * lda + i] : A[(int64_t)i * lda + k]) : 0.0;
      int jj;
      if (tb) { kk = e & 31; jj = e >> 5; } else { jj = e & 31; kk = e >> 5; }
      const int j = j0 + jj, k2 = k0 + kk;
      rb[r] = (j < N && k2 < K) ? (tb ? B[(int64_t)j * ldb + k2] : B[(int64_t)k2 * ldb + j]) : 0.0;
    }
  };
  auto stash = [&]() {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int e = threadIdx.x + 256 * r;
      int kk, ii;
      if (ta) { ii = e & 31; kk = e >> 5; } else { kk = e & 31; ii = e >> 5; }
      As[kk][ii] = ra[r];
      int jj;
      if (tb) { kk = e & 31; jj = e >> 5; } else { jj = e & 31; kk = e >> 5; }
      Bs[kk][jj] = rb[r];
    }
  };
  fetch(0);
  for (int k0 = 0; k0 < K; k0 += KC) {
    stash();
    __syncthreads();
    if (k0 + KC < K) fetch(k0 + KC);  // in flight during this chunk's FMAs
#pragma unroll
    for (int kk = 0; kk < KC; ++kk) {
      const double a0 = As[kk][ty], a1 = As[kk][ty + 16];
      const double b0 = Bs[kk][tx], b1 = Bs[kk][tx + 16];
      acc[0][0] = fma(a0, b0, acc[0][0]);
      acc[0][1] = fma(a0, b1, acc[0][1]);
      acc[1][0] = fma(a1, b0, acc[1][0]);
      acc[1][1] = fma(a1, b1, acc[1][1]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int i = i0 + ty + 16 * r;
    if (i >= M) continue;
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const int j = j0 + tx + 16 * c;
      if (j >= N) continue;
      double* o = Cm + (int64_t)i * ldc + j;
      *o = beta == 0.0 ? alpha * acc[r][c] : fma(beta, *o, alpha * acc[r][c]);
    }
  }
}

void launch_gemm(int M, int N, int K, double alpha, const double* A, int64_t lda, int ta,
                 const double* B, int64_t ldb, int tb, double beta, double* C, int64_t ldc,
                 cudaStream_t st) {
  if (M <= 0 || N <= 0) return;
  dim3 grid((unsigned)((N + 31) / 32), (unsigned)((M + 31) / 32));
  gemm_kernel<<<grid, 256, 0, st>>>(M, N, K, alpha, A, lda, ta, B, ldb, tb, beta, C, ldc);
}

__global__ void kprop_kernel(const double* __restrict__ prop, RecordLayout lay,
                             const double* __restrict__ piv, RecordLayout play, int k, int d,
                             int kind, int kfun, double sigma, double* __restrict__ K,
                             int64_t ldk) {
  const int j = blockIdx.y;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= k) return;
  K[(int64_t)j * ldk + i] =
      kernel_entry(prop + (int64_t)j * lay.rec, piv + (int64_t)i * play.rec, lay, d, kind, kfun,
                   sigma);
}

void launch_kprop(const double* prop, RecordLayout lay, int b, const double* piv, int64_t prec,
                  int k, int d, int kind, int kfun, double sigma, double* K, int64_t ldk,
                  cudaStream_t st) {
  if (k <= 0 || b <= 0) return;
  RecordLayout play;
  play.rec = prec;
  play.xoff = 2;
  play.foff = prec;
  kprop_kernel<<<dim3((unsigned)((k + 127) / 128), (unsigned)b), 128, 0, st>>>(
      prop, lay, piv, play, k, d, kind, kfun, sigma, K, ldk);
}

__global__ void lowmem_append_kernel(const double* __restrict__ prop, RecordLayout lay,
                                     const int* __restrict__ pos, int m, int kold, int64_t prec,
                                     const double* __restrict__ lacc_cm,
                                     const double* __restrict__ linv_rm, int64_t ldl,
                                     double* __restrict__ piv, double* __restrict__ fs,
                                     int64_t ldk, double* __restrict__ Lrm,
                                     double* __restrict__ Linv, int64_t ldw) {
  const int a = blockIdx.x;
  const double* rec = prop + (int64_t)pos[a] * lay.rec;
  double* prow = piv + (int64_t)(kold + a) * prec;
  for (int w = threadIdx.x; w < prec; w += blockDim.x) prow[w] = rec[w];
  double* lrow = Lrm + (int64_t)(kold + a) * ldw;
  double* irow = Linv + (int64_t)(kold + a) * ldw;
  for (int c = threadIdx.x; c < kold; c += blockDim.x) {
    const double f = rec[lay.foff + c];
    fs[(int64_t)a * ldk + c] = f;
    lrow[c] = f;
  }
  for (int c = threadIdx.x; c < m; c += blockDim.x) {
    lrow[kold + c] = c <= a ? lacc_cm[(int64_t)c * m + a] : 0.0;
    irow[kold + c] = c <= a ? linv_rm[(int64_t)perm_row(a) * ldl + c] : 0.0;
  }
}

void launch_lowmem_append(const double* prop, RecordLayout lay, const int* pos, int m, int kold,
                          int64_t prec, const double* lacc_cm, const double* linv_rm, int64_t ldl,
                          double* piv, double* fs, int64_t ldk, double* Lrm, double* Linv,
                          int64_t ldw, cudaStream_t st) {
  if (m <= 0) return;
  lowmem_append_kernel<<<m, 128, 0, st>>>(prop, lay, pos, m, kold, prec, lacc_cm, linv_rm, ldl,
                                          piv, fs, ldk, Lrm, Linv, ldw);
}

__global__ void lowmem_chol_kernel(const double* __restrict__ Lrm, int64_t ldw, int k,
                                   double* __restrict__ chol) {
  const int c = blockIdx.x;
  for (int a = threadIdx.x; a < k; a += blockDim.x)
    chol[(int64_t)c * k + a] = a >= c ? Lrm[(int64_t)a * ldw + c] : 0.0;
}

void launch_lowmem_chol(const double* Lrm, int64_t ldw, int k, double* chol, cudaStream_t st) {
  if (k <= 0) return;
  lowmem_chol_kernel<<<k, 256, 0, st>>>(Lrm, ldw, k, chol);
}

}  // namespace rpcb
