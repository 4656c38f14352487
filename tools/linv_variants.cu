// Debug aid: L^{-1} kernel variants on a random well-conditioned L (m x m, column-major),
// timed with CUDA events and checked bitwise against V0 (the library's column substitution).
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <cuda_runtime.h>

__host__ __device__ __forceinline__ int perm8(int r) { return ((r & 3) << 1) | (r >> 2); }
__host__ __device__ __forceinline__ int perm_row(int n) { return (n & ~7) + perm8(n & 7); }

constexpr int kW = 8;
template <int MODE>  // 0: full, 1: staging only
__global__ void __launch_bounds__(32 * kW) v0(const double* __restrict__ lacc_cm, int m, int nb, int64_t ldl,
                                             double* __restrict__ linv_rm) {
  extern __shared__ double smem_l[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int c = blockIdx.x * kW + warp;
  const int n2 = (m * m) >> 1;
  const double2* src2 = reinterpret_cast<const double2*>(lacc_cm);
  double2* dst2 = reinterpret_cast<double2*>(smem_l);
#pragma unroll 8
  for (int i = tid; i < n2; i += blockDim.x) dst2[i] = __ldg(src2 + i);
  if (tid == 0 && ((m * m) & 1)) smem_l[m * m - 1] = lacc_cm[m * m - 1];
  __syncthreads();
  if (MODE == 1) { if (c < m && lane == 0) linv_rm[c] = smem_l[c]; return; }
  const double* sL = smem_l;
  if (c >= m) return;
  double x[8], rd[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int a = lane + 32 * q;
    x[q] = (a == c) ? 1.0 : 0.0;
    rd[q] = a < m ? 1.0 / sL[(int64_t)a * m + a] : 0.0;
  }
  for (int t = c; t < m; ++t) {
    const int ql = t >> 5, ll = t & 31;
    double xt_own = 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (q == ql) xt_own = x[q] * rd[q];
    const double xt = __shfl_sync(0xffffffffu, xt_own, ll);
    const double* Lt = sL + (int64_t)t * m;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int a = lane + 32 * q;
      if (a == t) x[q] = xt;
      else if (a > t && a < m) x[q] = fma(-Lt[a], xt, x[q]);
    }
  }
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int a = lane + 32 * q;
    if (a < nb) linv_rm[(int64_t)perm_row(a) * ldl + c] = (a >= c && a < m) ? x[q] : 0.0;
  }
}

// V2: one warp per column, no staging: L columns read straight from global (L2/L1), the
// next column's values prefetched one step ahead.  NQ = ceil(m / 32) compile-time.
template <int NQ>
__global__ void __launch_bounds__(32 * kW) v2(const double* __restrict__ L, int m, int nb, int64_t ldl,
                                             double* __restrict__ linv_rm) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c = blockIdx.x * kW + warp;
  if (c >= m) return;
  double x[NQ], rd[NQ], ln[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    const int a = lane + 32 * q;
    x[q] = (a == c) ? 1.0 : 0.0;
    rd[q] = a < m ? 1.0 / __ldg(L + (int64_t)a * m + a) : 0.0;
    ln[q] = (a < m) ? __ldg(L + (int64_t)c * m + a) : 0.0;
  }
  for (int t = c; t < m; ++t) {
    double lc[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) lc[q] = ln[q];
    if (t + 1 < m) {
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        const int a = lane + 32 * q;
        ln[q] = (a < m) ? __ldg(L + (int64_t)(t + 1) * m + a) : 0.0;
      }
    }
    const int ql = t >> 5, ll = t & 31;
    double xt_own = 0.0;
#pragma unroll
    for (int q = 0; q < NQ; ++q)
      if (q == ql) xt_own = x[q] * rd[q];
    const double xt = __shfl_sync(0xffffffffu, xt_own, ll);
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int a = lane + 32 * q;
      if (a == t) x[q] = xt;
      else if (a > t) x[q] = fma(-lc[q], xt, x[q]);
    }
  }
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    const int a = lane + 32 * q;
    if (a < nb) linv_rm[(int64_t)perm_row(a) * ldl + c] = (a >= c && a < m) ? x[q] : 0.0;
  }
}


// V3: v0 with branch-free steps: the column's L values are loaded unconditionally (clamped
// row) one step ahead of use, the update is a select, NQ = ceil(m / 32) compile-time.
template <int NQ>
__global__ void __launch_bounds__(32 * kW) v3(const double* __restrict__ lacc_cm, int m, int nb, int64_t ldl,
                                             double* __restrict__ linv_rm) {
  extern __shared__ double smem_l[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int c = blockIdx.x * kW + warp;
  const int n2 = (m * m) >> 1;
  const double2* src2 = reinterpret_cast<const double2*>(lacc_cm);
  double2* dst2 = reinterpret_cast<double2*>(smem_l);
  {
    double2 buf[8];
    for (int i0 = tid; i0 < n2; i0 += 8 * blockDim.x) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = i0 + u * blockDim.x;
        if (i < n2) buf[u] = __ldg(src2 + i);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = i0 + u * blockDim.x;
        if (i < n2) dst2[i] = buf[u];
      }
    }
  }
  if (tid == 0 && ((m * m) & 1)) smem_l[m * m - 1] = lacc_cm[m * m - 1];
  __syncthreads();
  if (c >= m) return;
  double x[NQ], rd[NQ], ln[NQ];
  int ar[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    const int a = lane + 32 * q;
    ar[q] = a < m ? a : m - 1;
    x[q] = (a == c) ? 1.0 : 0.0;
    rd[q] = 1.0 / smem_l[ar[q] * m + ar[q]];
    ln[q] = smem_l[c * m + ar[q]];
  }
  for (int t = c; t < m; ++t) {
    double lc[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) lc[q] = ln[q];
    const int tn = t + 1 < m ? t + 1 : t;
#pragma unroll
    for (int q = 0; q < NQ; ++q) ln[q] = smem_l[tn * m + ar[q]];
    const int ql = t >> 5, ll = t & 31;
    double xt_own = x[0] * rd[0];
#pragma unroll
    for (int q = 1; q < NQ; ++q) xt_own = (q == ql) ? x[q] * rd[q] : xt_own;
    const double xt = __shfl_sync(0xffffffffu, xt_own, ll);
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int a = lane + 32 * q;
      const double nx = fma(-lc[q], xt, x[q]);
      x[q] = (a == t) ? xt : ((a > t) ? nx : x[q]);
    }
  }
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    const int a = lane + 32 * q;
    if (a < nb) linv_rm[(int64_t)perm_row(a) * ldl + c] = (a >= c && a < m) ? x[q] : 0.0;
  }
}

int main(int argc, char** argv) {
  int m = argc > 1 ? atoi(argv[1]) : 116;
  std::vector<double> L((size_t)m * m, 0.0);
  srand(1);
  for (int c = 0; c < m; ++c)
    for (int a = c; a < m; ++a) L[(size_t)c * m + a] = a == c ? 1.0 + rand() / (double)RAND_MAX : 0.1 * (rand() / (double)RAND_MAX - 0.5);
  double *dL, *dI, *dJ;
  const int nb = 256, ldl = 272;
  cudaMalloc(&dL, sizeof(double) * m * m);
  cudaMalloc(&dI, sizeof(double) * nb * ldl);
  cudaMalloc(&dJ, sizeof(double) * nb * ldl);
  cudaMemcpy(dL, L.data(), sizeof(double) * m * m, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(v0<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(v0<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int grid = (m + kW - 1) / kW;
  const size_t sm = sizeof(double) * m * m;
  auto time = [&](const char* name, auto fn) {
    for (int it = 0; it < 3; ++it) fn();
    cudaEventRecord(e0);
    for (int it = 0; it < 20; ++it) fn();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("m=%d %-28s %8.2f us  (%s)\n", m, name, ms * 1000 / 20, cudaGetErrorString(cudaGetLastError()));
  };
  cudaMemset(dI, 0, sizeof(double) * nb * ldl);
  time("v0 column subst (library)", [&] { v0<0><<<grid, 32 * kW, sm>>>(dL, m, nb, ldl, dI); });
  time("v0 staging only", [&] { v0<1><<<grid, 32 * kW, sm>>>(dL, m, nb, ldl, dJ); });
  std::vector<double> a((size_t)nb * ldl), b((size_t)nb * ldl);
  cudaMemcpy(a.data(), dI, sizeof(double) * nb * ldl, cudaMemcpyDeviceToHost);
  auto check = [&](const char* name) {
    cudaMemcpy(b.data(), dJ, sizeof(double) * nb * ldl, cudaMemcpyDeviceToHost);
    size_t bad = 0;
    for (int r = 0; r < m; ++r) for (int c = 0; c <= r; ++c) {
      const size_t i = (size_t)perm_row(r) * ldl + c;
      if (memcmp(&a[i], &b[i], 8)) ++bad;
    }
    printf("   %s: %zu entries differ bitwise\n", name, bad);
  };
  cudaMemset(dJ, 0, sizeof(double) * nb * ldl);
  if (m <= 128) time("v2 global+prefetch NQ4", [&] { v2<4><<<grid, 32 * kW>>>(dL, m, nb, ldl, dJ); });
  else time("v2 global+prefetch NQ8", [&] { v2<8><<<grid, 32 * kW>>>(dL, m, nb, ldl, dJ); });
  check("v2");
  cudaFuncSetAttribute(v3<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(v3<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(v3<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaMemset(dJ, 0, sizeof(double) * nb * ldl);
  if (m <= 64) time("v3 branch-free NQ2", [&] { v3<2><<<grid, 32 * kW, sm>>>(dL, m, nb, ldl, dJ); });
  else if (m <= 128) time("v3 branch-free NQ4", [&] { v3<4><<<grid, 32 * kW, sm>>>(dL, m, nb, ldl, dJ); });
  else time("v3 branch-free NQ8", [&] { v3<8><<<grid, 32 * kW, sm>>>(dL, m, nb, ldl, dJ); });
  check("v3");
  cudaMemset(dJ, 0, sizeof(double) * nb * ldl);
  if (m <= 128) time("v2 1 warp/CTA NQ4", [&] { v2<4><<<grid, 32 * kW>>>(dL, m, nb, ldl, dJ); });
  return 0;
}
