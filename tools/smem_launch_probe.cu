// Debug aid: launch cost of an almost-empty kernel vs its dynamic shared memory size.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_touch(double* out, int n) {
  extern __shared__ double sm[];
  sm[threadIdx.x] = threadIdx.x;
  __syncthreads();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = sm[n % blockDim.x];
}
int main() {
  double* out;
  cudaMalloc(&out, 8);
  cudaFuncSetAttribute(k_touch, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int kb : {4, 32, 48, 64, 100, 128, 160, 200, 227}) {
    for (int grid : {1, 148}) {
      for (int i = 0; i < 5; ++i) k_touch<<<grid, 512, kb * 1024>>>(out, i);
      cudaEventRecord(e0);
      for (int i = 0; i < 50; ++i) k_touch<<<grid, 512, kb * 1024>>>(out, i);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      printf("smem %3d KB grid %3d: %.2f us per launch\n", kb, grid, ms * 1000 / 50);
    }
  }
  // alternating small / large smem kernels
  cudaEventRecord(e0);
  for (int i = 0; i < 50; ++i) {
    k_touch<<<1, 512, 4 * 1024>>>(out, i);
    k_touch<<<1, 512, 200 * 1024>>>(out, i);
  }
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("alternating 4KB / 200KB: %.2f us per pair (%s)\n", ms * 1000 / 50, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
