// Debug aid: DMMA issue rate of the update kernel's inner loop shapes with operands
// from shared memory (128B-swizzled [rows][16] fp64 tiles, as the TMA ring holds them).
// One block per SM; 4 warps (one per SM sub-partition) or 8 warps.
//   V1  per k-step: 2 A loads, then per fragment q: 1 B load + 2 DMMA   (current kernel)
//   V2  B-stationary: the chunk's 4x2 A values first, then per fragment q: 4 B loads + 8 DMMA
//   V3  V2 with 16-byte loads: k order permuted inside the chunk so a lane's two k values of
//       a fragment are adjacent (k = 2t, 2t+1 and 8+2t, 9+2t): 2 LDS.128 per fragment
//   V4  V3, next fragment's B values loaded before this fragment's DMMAs (register prefetch)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t swz_off(int row, int k) {
  const int chunk = (k >> 1) ^ (row & 7);
  return (uint32_t)(row * 128 + chunk * 16 + (k & 1) * 8);
}
__device__ __forceinline__ int perm8(int n8) { return n8 < 4 ? 2 * n8 : 2 * (n8 - 4) + 1; }
__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

constexpr int NFW = 15;
constexpr int BM = 64;

template <int V>
__global__ void __launch_bounds__(256, 1) kern(double* out, int iters) {
  extern __shared__ __align__(1024) unsigned char sm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < (BM + 8 * NFW) * 16; i += blockDim.x)
    reinterpret_cast<double*>(sm)[i] = 1.0 + 1e-3 * (i & 63);
  __syncthreads();
  const int g = lane >> 2, t = lane & 3, pg = perm8(g);
  const int wr = warp & 3;
  const unsigned char* Aw = sm + wr * 16 * 128;
  const unsigned char* Bw = sm + BM * 128;
  uint32_t foff[4];
#pragma unroll
  for (int s = 0; s < 4; ++s) foff[s] = swz_off(pg, 4 * s + t);
  const uint32_t p0 = swz_off(pg, 2 * t), p1 = swz_off(pg, 8 + 2 * t);
  double acc[2][NFW][2];
#pragma unroll
  for (int fr = 0; fr < 2; ++fr)
#pragma unroll
    for (int q = 0; q < NFW; ++q) acc[fr][q][0] = acc[fr][q][1] = 0.0;
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
    if (V == 1) {
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        double a[2];
#pragma unroll
        for (int fr = 0; fr < 2; ++fr) a[fr] = *reinterpret_cast<const double*>(Aw + fr * 1024 + foff[s]);
#pragma unroll
        for (int q = 0; q < NFW; ++q) {
          const double bv = *reinterpret_cast<const double*>(Bw + q * 1024 + foff[s]);
#pragma unroll
          for (int fr = 0; fr < 2; ++fr) dmma884(acc[fr][q][0], acc[fr][q][1], a[fr], bv);
        }
      }
    } else if (V == 5) {
      // fr-outer: consecutive DMMAs share the A register (operand reuse), all 15 B values live
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        double a[2], bq[NFW];
#pragma unroll
        for (int fr = 0; fr < 2; ++fr) a[fr] = *reinterpret_cast<const double*>(Aw + fr * 1024 + foff[s]);
#pragma unroll
        for (int q = 0; q < NFW; ++q) bq[q] = *reinterpret_cast<const double*>(Bw + q * 1024 + foff[s]);
#pragma unroll
        for (int fr = 0; fr < 2; ++fr)
#pragma unroll
          for (int q = 0; q < NFW; ++q) dmma884(acc[fr][q][0], acc[fr][q][1], a[fr], bq[q]);
      }
    } else if (V == 2) {
      double a[4][2];
#pragma unroll
      for (int s = 0; s < 4; ++s)
#pragma unroll
        for (int fr = 0; fr < 2; ++fr) a[s][fr] = *reinterpret_cast<const double*>(Aw + fr * 1024 + foff[s]);
#pragma unroll
      for (int q = 0; q < NFW; ++q)
#pragma unroll
        for (int s = 0; s < 4; ++s) {
          const double bv = *reinterpret_cast<const double*>(Bw + q * 1024 + foff[s]);
#pragma unroll
          for (int fr = 0; fr < 2; ++fr) dmma884(acc[fr][q][0], acc[fr][q][1], a[s][fr], bv);
        }
    } else {
      double2 a[2][2];  // [pair][fr]
#pragma unroll
      for (int fr = 0; fr < 2; ++fr) {
        a[0][fr] = *reinterpret_cast<const double2*>(Aw + fr * 1024 + p0);
        a[1][fr] = *reinterpret_cast<const double2*>(Aw + fr * 1024 + p1);
      }
      double2 b0 = *reinterpret_cast<const double2*>(Bw + p0);
      double2 b1 = *reinterpret_cast<const double2*>(Bw + p1);
#pragma unroll
      for (int q = 0; q < NFW; ++q) {
        double2 c0 = b0, c1 = b1;
        if (V == 4 && q + 1 < NFW) {
          b0 = *reinterpret_cast<const double2*>(Bw + (q + 1) * 1024 + p0);
          b1 = *reinterpret_cast<const double2*>(Bw + (q + 1) * 1024 + p1);
        } else if (V == 3) {
          c0 = *reinterpret_cast<const double2*>(Bw + q * 1024 + p0);
          c1 = *reinterpret_cast<const double2*>(Bw + q * 1024 + p1);
        }
#pragma unroll
        for (int fr = 0; fr < 2; ++fr) {
          dmma884(acc[fr][q][0], acc[fr][q][1], a[0][fr].x, c0.x);
          dmma884(acc[fr][q][0], acc[fr][q][1], a[0][fr].y, c0.y);
          dmma884(acc[fr][q][0], acc[fr][q][1], a[1][fr].x, c1.x);
          dmma884(acc[fr][q][0], acc[fr][q][1], a[1][fr].y, c1.y);
        }
      }
    }
    __syncwarp();
  }
  double s = 0;
#pragma unroll
  for (int fr = 0; fr < 2; ++fr)
#pragma unroll
    for (int q = 0; q < NFW; ++q) s += acc[fr][q][0] + acc[fr][q][1];
  if (s == 1.2345) out[0] = s;
}

int main() {
  double* out;
  cudaMalloc(&out, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int smem = (BM + 8 * NFW) * 128;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](auto k, const char* nm, int warps) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int iters = 4000;
    k<<<sms, 32 * warps, smem>>>(out, 10);
    cudaEventRecord(e0);
    k<<<sms, 32 * warps, smem>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double fl = 2.0 * 256 * 4 * 2 * NFW * (double)iters * warps * sms;
    printf("%-4s warps=%d  %.3f ms  %.2f TFLOP/s (%s)\n", nm, warps, ms, fl / (ms * 1e-3) / 1e12,
           cudaGetErrorString(cudaGetLastError()));
  };
  for (int w : {4, 8}) {
    run(kern<1>, "V1", w);
    run(kern<5>, "V5", w);
    run(kern<2>, "V2", w);
    run(kern<3>, "V3", w);
    run(kern<4>, "V4", w);
  }
  return 0;
}
