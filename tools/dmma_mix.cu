// Debug aid: can one warp per SM sub-partition keep the FP64 DMMA pipe busy, and does
// FP64 CUDA-core work (DFMA) issued by a second warp on the same sub-partition steal
// DMMA throughput?  (Decides whether ping-pong warp groups can hide the exp transform.)
#include <cstdio>
#include <cuda_runtime.h>

template <int ACC>
__device__ __forceinline__ void dmma_body(double (&c)[ACC][2], double a, double b) {
#pragma unroll
  for (int i = 0; i < ACC; ++i)
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
}

// MODE 0: every warp DMMA.  MODE 1: warps with (warp / 4) odd run DFMA chains instead.
// MODE 2: odd-half warps idle (exit).  MODE 3: odd-half warps run integer/LDS-heavy work.
template <int ACC, int MODE>
__global__ void mix(double* out, int iters, int fiters, unsigned long long* cyc) {
  const int warp = threadIdx.x >> 5;
  const bool other = (warp / 4) & 1;
  __shared__ double tab[64];
  if (threadIdx.x < 64) tab[threadIdx.x] = 1.0 + threadIdx.x;
  __syncthreads();
  const unsigned long long t0 = clock64();
  if (MODE == 0 || !other) {
    double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
    double c[ACC][2];
#pragma unroll
    for (int i = 0; i < ACC; ++i) c[i][0] = c[i][1] = 0.0;
    for (int it = 0; it < iters; ++it) dmma_body<ACC>(c, a, b);
    double s = 0;
#pragma unroll
    for (int i = 0; i < ACC; ++i) s += c[i][0] + c[i][1];
    if (s == 12345.678) out[0] = s;
    if ((threadIdx.x & 31) == 0) cyc[blockIdx.x * 32 + warp] = clock64() - t0;
  } else if (MODE == 1) {
    double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-12;
    double c[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i] = i;
    for (int it = 0; it < fiters; ++it)
#pragma unroll
      for (int i = 0; i < 8; ++i) c[i] = fma(c[i], a, b);
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += c[i];
    if (s == 12345.678) out[0] = s;
    if ((threadIdx.x & 31) == 0) cyc[blockIdx.x * 32 + warp] = clock64() - t0;
  } else if (MODE == 3) {
    int k = threadIdx.x;
    double s = 0;
    for (int it = 0; it < fiters; ++it) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        k = (k * 1664525 + 1013904223);
        s += tab[(k >> 8) & 63];
      }
    }
    if (s == 12345.678) out[0] = s;
    if ((threadIdx.x & 31) == 0) cyc[blockIdx.x * 32 + warp] = clock64() - t0;
  }
}

int main() {
  double* out;
  unsigned long long* cyc;
  cudaMalloc(&out, 8);
  cudaMalloc(&cyc, 8 * 32 * 148 * 4);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](auto kern, const char* name, int warps, int dmma_warps, int iters, int fiters,
                 int acc) {
    kern<<<sms, 32 * warps>>>(out, 10, 10, cyc);
    cudaEventRecord(e0);
    kern<<<sms, 32 * warps>>>(out, iters, fiters, cyc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 2.0 * 256 * acc * (double)iters * sms * dmma_warps;
    printf("%-44s warps=%2d dmma_warps=%2d  %.3f ms  DMMA %.2f TFLOP/s  (%s)\n", name, warps,
           dmma_warps, ms, flops / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
  };
  const int it = 20000;
  run(mix<30, 0>, "all DMMA, ACC=30", 4, 4, it, 0, 30);
  run(mix<30, 0>, "all DMMA, ACC=30", 8, 8, it, 0, 30);
  run(mix<30, 0>, "all DMMA, ACC=30", 16, 16, it / 2, 0, 30);
  run(mix<8, 0>, "all DMMA, ACC=8", 4, 4, it, 0, 8);
  run(mix<8, 0>, "all DMMA, ACC=8", 8, 8, it, 0, 8);
  run(mix<30, 2>, "DMMA 4 warps + 4 idle", 8, 4, it, 0, 30);
  // DFMA warps sized to run about as long as the DMMA warps alone
  for (int f : {it * 30 / 8 / 4, it * 30 / 8 / 2, it * 30 / 8})
  {
    char nm[96];
    snprintf(nm, sizeof nm, "DMMA 4 warps + 4 DFMA warps (fiters=%d)", f);
    run(mix<30, 1>, nm, 8, 4, it, f, 30);
  }
  run(mix<30, 3>, "DMMA 4 warps + 4 int/LDS warps", 8, 4, it, it * 4, 30);
  return 0;
}
