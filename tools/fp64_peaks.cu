// FP64 peak microbenchmarks for B200 (sm_100a): DMMA (mma.sync f64) and DFMA.
// Writes one JSON line with measured TFLOP/s; used as the FP64 roofline peak.
#include <cstdio>
#include <cuda_runtime.h>

template <int ACC>
__global__ void dmma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[ACC][2];
#pragma unroll
  for (int i = 0; i < ACC; ++i) { c[i][0] = 0.0; c[i][1] = 0.0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ACC; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ACC; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

template <int ACC>
__global__ void dfma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-12;
  double c[ACC];
#pragma unroll
  for (int i = 0; i < ACC; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ACC; ++i) c[i] = fma(c[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ACC; ++i) s += c[i];
  if (s == 12345.678) out[0] = s;
}

__global__ void copy_kernel(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += stride) b[i] = a[i];
}

int main() {
  double* out; cudaMalloc(&out, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  double best_dmma = 0, best_dfma = 0;
  for (int wpb : {4, 8, 16}) {
    for (int cps : {1, 2, 4}) {
      int iters = 4000;
      dim3 grid(sms * cps), block(32 * wpb);
      dmma_loop<8><<<grid, block>>>(out, 10);
      cudaEventRecord(e0);
      dmma_loop<8><<<grid, block>>>(out, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * 256 * 8 * (double)iters * grid.x * wpb;
      double tf = flops / (ms * 1e-3) / 1e12;
      if (tf > best_dmma) best_dmma = tf;
      fprintf(stderr, "dmma wpb=%d cps=%d: %.2f TFLOP/s\n", wpb, cps, tf);
      dfma_loop<8><<<grid, block>>>(out, 10);
      cudaEventRecord(e0);
      dfma_loop<8><<<grid, block>>>(out, iters * 4);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      flops = 2.0 * 8 * (double)iters * 4 * grid.x * 32 * wpb;
      tf = flops / (ms * 1e-3) / 1e12;
      if (tf > best_dfma) best_dfma = tf;
      fprintf(stderr, "dfma wpb=%d cps=%d: %.2f TFLOP/s\n", wpb, cps, tf);
    }
  }
  size_t n = (size_t)1 << 28;  // 2^28 double2 = 4 GiB each
  double2 *a, *b; cudaMalloc(&a, n * 16); cudaMalloc(&b, n * 16);
  cudaMemset(a, 0, n * 16);
  double best_bw = 0;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    copy_kernel<<<sms * 8, 512>>>(a, b, n);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double gbs = 2.0 * n * 16 / (ms * 1e-3) / 1e9;
    if (gbs > best_bw) best_bw = gbs;
  }
  printf("{\"fp64_dmma_tflops\": %.3f, \"fp64_dfma_tflops\": %.3f, \"hbm_copy_gbs\": %.1f, \"sms\": %d}\n",
         best_dmma, best_dfma, best_bw, sms);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) { fprintf(stderr, "%s\n", cudaGetErrorString(err)); return 1; }
  return 0;
}
