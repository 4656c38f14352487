// Debug aid: host-side cost of a kernel launch with ~1 KB of parameters (six CUtensorMaps,
// like the update kernel) against a small-parameter launch, on an idle stream and behind a
// running cooperative kernel.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/launch_probe tools/launch_probe.cu -lcuda
#include <chrono>
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>

struct Big { char pad[256]; };
__global__ void k_big(Big p, const __grid_constant__ CUtensorMap a, const __grid_constant__ CUtensorMap b,
                      const __grid_constant__ CUtensorMap c, const __grid_constant__ CUtensorMap d,
                      const __grid_constant__ CUtensorMap e, const __grid_constant__ CUtensorMap f, int* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = p.pad[3];
}
__global__ void k_small(int* out) { if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = 1; }
__global__ void k_spin(long long cycles) {
  long long t0 = clock64();
  while (clock64() - t0 < cycles) {}
}

int main() {
  int* out; cudaMalloc(&out, 64);
  cudaStream_t st; cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  Big p{}; CUtensorMap m{};
  auto us = [](auto a, auto b) { return std::chrono::duration<double, std::micro>(b - a).count(); };
  for (int busy = 0; busy < 2; ++busy) {
    double tb = 0, ts = 0; int n = 50;
    for (int i = 0; i < n; ++i) {
      if (busy) k_spin<<<148, 512, 0, st>>>(200000);
      auto t0 = std::chrono::steady_clock::now();
      k_big<<<148, 256, 0, st>>>(p, m, m, m, m, m, m, out);
      auto t1 = std::chrono::steady_clock::now();
      k_small<<<148, 256, 0, st>>>(out);
      auto t2 = std::chrono::steady_clock::now();
      tb += us(t0, t1); ts += us(t1, t2);
      cudaStreamSynchronize(st);
    }
    printf("%s stream: big-param launch %.2f us, small launch %.2f us (%s)\n", busy ? "busy" : "idle",
           tb / n, ts / n, cudaGetErrorString(cudaGetLastError()));
  }
  // launch right after a host spin on a flag written by the running kernel (mapped memory)
  return 0;
}
