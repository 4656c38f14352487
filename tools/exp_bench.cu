// Microbenchmark: cost of the kernel-column transform (60 exp per thread) in isolation.
#include <cstdio>
#include <cuda_runtime.h>
__constant__ double kExpC[8] = {92.332482616893656, -1.0830424696249145e-02, -3.6235106466348430e-19,
                                8.3333333333333333e-03, 4.1666666666666667e-02, 1.6666666666666667e-01, 0.5, -745.5};
__device__ __forceinline__ double exp_tab(double x, const double* __restrict__ tab) {
  constexpr double kShift = 6755399441055744.0;
  x = fmax(x, kExpC[7]);
  const double ks = fma(x, kExpC[0], kShift);
  const int k = __double2loint(ks);
  const double kd = ks - kShift;
  double r = fma(kd, kExpC[1], x);
  r = fma(kd, kExpC[2], r);
  double q = fma(r, kExpC[3], kExpC[4]);
  q = fma(q, r, kExpC[5]);
  q = fma(q, r, kExpC[6]);
  q = fma(q * r, r, r);
  const double t = tab[k & 63];
  const int n = k >> 6;
  const int n1 = n >> 1, n2 = n - n1;
  const double s1 = __hiloint2double((n1 + 1023) << 20, 0);
  const double s2 = __hiloint2double((n2 + 1023) << 20, 0);
  return fma(t, q, t) * s1 * s2;
}
template <int NE>
__global__ void k_exp(double* out, int reps, unsigned long long* cyc) {
  __shared__ double tab[64];
  if (threadIdx.x < 64) tab[threadIdx.x] = exp2(threadIdx.x / 64.0);
  __syncthreads();
  double a[NE];
#pragma unroll
  for (int i = 0; i < NE; ++i) a[i] = -(threadIdx.x * 0.01 + i * 0.37);
  unsigned long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int i = 0; i < NE; ++i) a[i] = -exp_tab(a[i] - 1.0, tab) * 3.0;
  }
  unsigned long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int i = 0; i < NE; ++i) s += a[i];
  if (s == 1.2345) out[0] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  double* out; unsigned long long* cyc; cudaMalloc(&out, 8); cudaMalloc(&cyc, 8 * 1024);
  for (int blocks : {148, 296}) {
    k_exp<60><<<blocks, 256>>>(out, 10, cyc);
    cudaDeviceSynchronize();
    unsigned long long h[1024]; cudaMemcpy(h, cyc, 8 * blocks, cudaMemcpyDeviceToHost);
    double avg = 0; for (int i = 0; i < blocks; ++i) avg += h[i]; avg /= blocks;
    printf("blocks %d: %.0f cycles per 60-exp pass per CTA (256 thr)\n", blocks, avg / 10);
  }
  cudaError_t e = cudaGetLastError(); if (e) printf("%s\n", cudaGetErrorString(e));
}
