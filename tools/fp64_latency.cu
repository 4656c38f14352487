// Debug aid: dependent-chain latency (cycles per op) of FP64 and related ops, one warp.
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void chain(double* out, double a, double b, long long* cyc, int n) {
  double x = a + threadIdx.x * 1e-9;
  __syncwarp();
  const long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    if (OP == 0) x = fma(x, a, b);
    if (OP == 1) x = __dadd_rn(x, b);
    if (OP == 2) x = __dmul_rn(x, a);
    if (OP == 3) x = __dsqrt_rn(x) + 1.0;
    if (OP == 4) x = __ddiv_rn(b, x) + 1.0;
    if (OP == 5) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31) * a;
    if (OP == 6) x = __fmaf_rn((float)x, (float)a, (float)b);
    if (OP == 7) x = 1.0 / x + 0.5;
  }
  const long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 1024 * 8); cudaMalloc(&cyc, 8);
  const char* names[] = {"DFMA", "DADD", "DMUL", "dsqrt_rn+add", "ddiv_rn+add", "SHFL+DMUL", "FFMA(f32 chain)", "1/x + add"};
  const int n = 4096;
  auto run = [&](auto kern, int op) {
    for (int w = 0; w < 2; ++w) kern<<<1, 32>>>(out, 1.0000001, 1e-7, cyc, n);
    long long c; cudaDeviceSynchronize(); cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%-18s %7.1f cycles/op (%s)\n", names[op], (double)c / n, cudaGetErrorString(cudaGetLastError()));
  };
  run(chain<0>, 0); run(chain<1>, 1); run(chain<2>, 2); run(chain<3>, 3);
  run(chain<4>, 4); run(chain<5>, 5); run(chain<6>, 6); run(chain<7>, 7);
  return 0;
}
