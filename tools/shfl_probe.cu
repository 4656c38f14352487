// Debug aid: SHFL throughput of warp 0 while the CTA's other warps wait at a barrier.
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(double* out, long long* cyc, int n) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double v[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) v[q] = lane + q;
  long long t0 = 0, t1 = 0;
  if (warp == 0) {
    t0 = clock64();
    for (int it = 0; it < n; ++it) {
      double s = v[it & 15];
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const double w = __shfl_sync(0xffffffffu, s, q);
        v[q] = MODE == 2 ? __dsub_rn(v[q], __dmul_rn(s, w)) : v[q] + w;
      }
    }
    t1 = clock64();
  }
  __syncthreads();
  double a = 0;
#pragma unroll
  for (int q = 0; q < 16; ++q) a += v[q];
  out[threadIdx.x] = a;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 1024 * 8); cudaMalloc(&cyc, 8);
  const int n = 1000;
  auto run = [&](auto kern, int threads, const char* name) {
    for (int w = 0; w < 2; ++w) kern<<<1, threads>>>(out, cyc, n);
    long long c; cudaDeviceSynchronize(); cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%-40s %7.1f cycles per 16-shfl step (%s)\n", name, (double)c / n, cudaGetErrorString(cudaGetLastError()));
  };
  run(k<1>, 32, "1 warp, shfl+add");
  run(k<1>, 512, "512 thr (15 warps at barrier), shfl+add");
  run(k<2>, 32, "1 warp, shfl+dmul+dsub");
  run(k<2>, 512, "512 thr, shfl+dmul+dsub");
  return 0;
}
