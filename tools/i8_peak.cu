// i8_peak.cu — measured tcgen05.mma issue-bound throughput per SM for kind::i8 and kind::f16
// (bf16) at M = 128, K = 32 bytes, N = 64 / 128 / 256: one CTA per SM, operands resident in
// shared memory (no TMA traffic), one thread issues NITER products round-robin over the
// accumulators, then commits and waits.  Prints cycles per product and chip-level TOP/s.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o i8_peak tools/i8_peak.cu && ./i8_peak
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint64_t desc_sw64(uint32_t saddr) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(512 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)4 << 61;
  return d;
}

__device__ __forceinline__ bool elect_one() {
  uint32_t p;
  asm volatile("{\n.reg .pred P;\nelect.sync _|P, 0xffffffff;\nselp.u32 %0, 1, 0, P;\n}\n" : "=r"(p));
  return p != 0;
}

// MODE 0: issue from an `if (threadIdx.x == 0)` region; 1: from `if (warp 0 && elect.sync)`;
// 2: the whole warp runs the loop, each product under its own elect.sync
template <int KIND, int MODE>  // KIND 0: i8, 1: bf16
__global__ void __launch_bounds__(128, 1) peak_kernel(int n, int niter, long long* cyc) {
  extern __shared__ __align__(1024) unsigned char smraw[];
  unsigned char* sm = smraw + ((1024u - (smem_u32(smraw) & 1023u)) & 1023u);
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase_s;
  for (int i = threadIdx.x; i < (128 + 256) * 64 / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(sm)[i] = KIND == 0 ? 0x01010101u : 0u;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(
        smem_u32(&tbase_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tbase = tbase_s;
  bool me = false;
  if (MODE == 0) me = threadIdx.x == 0;
  else if (MODE == 1) me = threadIdx.x < 32 && elect_one();
  else me = threadIdx.x < 32;
  if (MODE == 3) {
    // descriptors change with every product (7 A planes x 7 B planes of 8 KB, the residual
    // GEMM's diagonal order), issued from an elect.sync region
    if (threadIdx.x < 32 && elect_one()) {
      const uint32_t idesc = ((2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | (8u << 24));
      const uint32_t ba = smem_u32(sm), bb = ba + 7 * 8192;
      const long long t0 = clock64();
      int cnt = 0;
      for (int i = 0; cnt < niter; ++i) {
#pragma unroll
        for (int d = 0; d < 7; ++d) {
#pragma unroll
          for (int t = 0; t <= d; ++t) {
#pragma unroll
            for (int ks = 0; ks < 2; ++ks) {
              const uint64_t da = desc_sw64(ba + t * 8192 + ks * 32);
              const uint64_t db = desc_sw64(bb + (d - t) * 8192 + ks * 32);
              const uint32_t acc = tbase + (uint32_t)((d & 3) * 128);
              asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                           "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(acc),
                           "l"(da), "l"(db), "r"(idesc), "r"((uint32_t)(i | t | ks)));
              ++cnt;
            }
          }
        }
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
          smem_u32(&bar)));
      uint32_t ok = 0;
      while (!ok)
        asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n"
                     "selp.u32 %0, 1, 0, p;\n}\n" : "=r"(ok) : "r"(smem_u32(&bar)) : "memory");
      cyc[blockIdx.x] = (clock64() - t0) * niter / cnt;
    }
  } else if (me) {
    const uint32_t idesc = KIND == 0 ? ((2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | (8u << 24))
                                     : ((1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | (8u << 24));
    const uint64_t da = desc_sw64(smem_u32(sm)), db = desc_sw64(smem_u32(sm) + 128 * 64);
    const int nacc = 512 / n;
    const long long t0 = clock64();
    for (int i = 0; i < niter; i += 4) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t acc = tbase + (uint32_t)(((i + j) & (nacc - 1)) * n);
        if (MODE == 2 && !elect_one()) continue;
        if (KIND == 0)
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                       "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(acc),
                       "l"(da), "l"(db), "r"(idesc), "r"(1u));
        else
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                       "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(acc),
                       "l"(da), "l"(db), "r"(idesc), "r"(1u));
      }
    }
    if (MODE != 2 || elect_one()) {
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
          smem_u32(&bar)));
    }
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n"
                   "selp.u32 %0, 1, 0, p;\n}\n" : "=r"(ok) : "r"(smem_u32(&bar)) : "memory");
    if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tbase));
}

template <int KIND, int MODE>
static void run(const char* name, int n, int sms) {
  const int niter = 8192;
  long long* cyc;
  cudaMalloc(&cyc, sizeof(long long) * sms);
  const size_t smem = (MODE == 3 ? 14 * 8192 : (128 + 256) * 64) + 1024;
  cudaFuncSetAttribute(peak_kernel<KIND, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  peak_kernel<KIND, MODE><<<sms, 128, smem>>>(n, niter, cyc);
  cudaEventRecord(e0);
  peak_kernel<KIND, MODE><<<sms, 128, smem>>>(n, niter, cyc);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  long long h = 0;
  cudaMemcpy(&h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  const double kel = KIND == 0 ? 32.0 : 16.0;  // K elements per product
  const double ops = 2.0 * 128 * n * kel * niter * sms;
  printf("{\"kind\": \"%s\", \"mode\": %d, \"n\": %d, \"cycles_per_mma\": %.1f, \"ms\": %.4f, \"tops\": %.1f, \"err\": \"%s\"}\n",
         name, MODE, n, (double)h / niter, ms, ops / (ms * 1e-3) / 1e12, cudaGetErrorString(err));
  cudaFree(cyc);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int n : {64, 128, 256}) run<0, 0>("i8", n, sms);
  for (int n : {64, 128, 256}) run<0, 1>("i8", n, sms);
  for (int n : {64, 128, 256}) run<0, 2>("i8", n, sms);
  for (int n : {64, 96, 112, 128}) run<0, 3>("i8-varying", n, sms);
  for (int n : {64, 128, 256}) run<1, 1>("bf16", n, sms);
  return 0;
}
