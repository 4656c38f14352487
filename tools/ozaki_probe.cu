// Exploratory probe (SURVEY/VERDICT "past the DMMA roof"): the residual GEMM C = F B'^T of an
// update round computed from int8 slices on the 5th-generation tensor cores (tcgen05.mma
// kind::i8, int32 accumulators in TMEM), Ozaki scheme I, against an FP64 reference.
//   F (|F_ij| <= 1 for a unit-diagonal kernel): 7 signed digits in base 2^7 (first 2^6) with a
//   fixed scale; B': per row scaled by 2^e_c, 7 digits.  C = 2^(e_c - 12) sum_d 2^(-7 d) A_d,
//   A_d = sum_{t + u = d} F_t B'_u^T (exact int32), d < 7: 28 int8 GEMMs.
// One CTA per 128 F rows x 64 columns: 7 diagonal accumulators x 64 TMEM columns = 448 of
// 512; warp 0 issues TMA (7 + 7 planes per 64-byte K block, 64B swizzle), warp 1 the MMAs,
// warps 2-5 the epilogue (tcgen05.ld, FP64 Horner over the diagonals, scale, store).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2410_03969_b200/csrc
//      -o tools/ozaki_probe tools/ozaki_probe.cu -lcuda
//   ./tools/ozaki_probe [N] [K] [m]
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "common.cuh"

using namespace rpcb;

constexpr int kPl = 7;             // slices per operand
constexpr int kBM = 128;           // F rows per tile (MMA M)
constexpr int kBN = 64;            // output columns per tile (MMA N)
constexpr int kKB = 64;            // K bytes per stage
constexpr int kNst = 2;            // stages
constexpr int kApl = kBM * kKB;    // 8 KB per A plane
constexpr int kBpl = kBN * kKB;    // 4 KB per B plane
constexpr int kStage = kPl * (kApl + kBpl);

__device__ __forceinline__ uint64_t desc_sw64(uint32_t saddr) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1 << 16;              // LBO (unused, swizzled K-major)
  d |= (uint64_t)(512 >> 4) << 32;     // SBO: 8 rows x 64 B
  d |= (uint64_t)1 << 46;              // descriptor version (sm_100)
  d |= (uint64_t)4 << 61;              // SWIZZLE_64B
  return d;
}

__global__ void __launch_bounds__(192, 1) i8gemm_kernel(const __grid_constant__ CUtensorMap tmA,
                                                       const __grid_constant__ CUtensorMap tmB,
                                                       int N, int mpad, int mreal, int nkb,
                                                       const double* __restrict__ cscale,
                                                       double* __restrict__ C, int64_t ldc) {
  extern __shared__ __align__(1024) unsigned char smraw[];
  unsigned char* sm = smraw + ((1024u - (smem_u32(smraw) & 1023u)) & 1023u);
  __shared__ uint64_t full[kNst], empty[kNst], done;
  __shared__ uint32_t tmem_base_s;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row0 = blockIdx.x * kBM, col0 = blockIdx.y * kBN;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kNst; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&done, 1);
    mbar_fence_init();
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(
        smem_u32(&tmem_base_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tbase = tmem_base_s;
  if (warp == 0) {
    if (lane == 0) {
      for (int kb = 0; kb < nkb; ++kb) {
        const int s = kb % kNst;
        if (kb >= kNst) mbar_wait(&empty[s], ((kb / kNst) - 1) & 1);
        mbar_arrive_expect_tx(&full[s], kStage);
        unsigned char* st = sm + s * kStage;
        for (int t = 0; t < kPl; ++t) tma_load_2d(st + t * kApl, &tmA, kb * kKB, t * N + row0, &full[s]);
        for (int u = 0; u < kPl; ++u)
          tma_load_2d(st + kPl * kApl + u * kBpl, &tmB, kb * kKB, u * mpad + col0, &full[s]);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(kBN >> 3) << 17) |
                             ((uint32_t)(kBM >> 4) << 24);
      for (int kb = 0; kb < nkb; ++kb) {
        const int s = kb % kNst;
        mbar_wait(&full[s], (kb / kNst) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        const uint32_t ba = smem_u32(sm + s * kStage), bb = ba + kPl * kApl;
#pragma unroll
        for (int t = 0; t < kPl; ++t)
#pragma unroll
          for (int u = 0; u < kPl - t; ++u)
#pragma unroll
            for (int ks = 0; ks < 2; ++ks) {
              const uint64_t da = desc_sw64(ba + t * kApl + ks * 32);
              const uint64_t db = desc_sw64(bb + u * kBpl + ks * 32);
              const uint32_t accum = (kb | ks | t) != 0;
              asm volatile(
                  "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                  "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(
                      tbase + (uint32_t)((t + u) * kBN)),
                  "l"(da), "l"(db), "r"(idesc), "r"(accum));
            }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
            smem_u32(&empty[s])));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
          smem_u32(&done)));
    }
  } else {
    mbar_wait(&done, 0);
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const int q = warp & 3;
    const int r = row0 + q * 32 + lane;
#pragma unroll 1
    for (int cc = 0; cc < kBN / 16; ++cc) {
      double acc[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) acc[j] = 0.0;
#pragma unroll
      for (int d = kPl - 1; d >= 0; --d) {
        uint32_t v[16];
        const uint32_t ta = tbase + ((uint32_t)(q * 32) << 16) + (uint32_t)(d * kBN + cc * 16);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, "
            "%10, %11, %12, %13, %14, %15}, [%16];\n"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
              "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]),
              "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
            : "r"(ta));
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
        for (int j = 0; j < 16; ++j) acc[j] = fma(acc[j], 0.0078125, (double)(int)v[j]);
      }
      if (r < N) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int c = col0 + cc * 16 + j;
          if (c < mreal) C[(int64_t)r * ldc + c] = acc[j] * cscale[c];
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tbase));
}

// 7 base-2^7 digits of v * 2^6 (|v| <= 1), rounded to nearest (magic-number rint)
__device__ __forceinline__ void slice7(double v, int8_t* out, int64_t pstride) {
  constexpr double kM = 6755399441055744.0;  // 1.5 * 2^52
  double r = v * 64.0;
#pragma unroll
  for (int t = 0; t < kPl; ++t) {
    const double ar = (r + kM) - kM;
    out[t * pstride] = (int8_t)__double2loint(r + kM);
    r = (r - ar) * 128.0;
  }
}
__global__ void slice_rows(const double* __restrict__ X, int64_t ldx, int rows, int K, int kpad,
                           const double* __restrict__ rscale, int8_t* __restrict__ planes,
                           int64_t pstride) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= (int64_t)rows * kpad) return;
  const int r = (int)(i / kpad), k = (int)(i % kpad);
  const double v = k < K ? X[(int64_t)r * ldx + k] * (rscale ? rscale[r] : 1.0) : 0.0;
  slice7(v, planes + (int64_t)r * kpad + k, pstride);
}
// FP64 reference, one output per thread, FMA in k order
__global__ void ref_gemm(const double* __restrict__ F, const double* __restrict__ B, int N, int m,
                         int K, double* __restrict__ C, double* __restrict__ Cabs) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= (int64_t)N * m) return;
  const int r = (int)(i / m), c = (int)(i % m);
  double s = 0.0, a = 0.0;
  for (int k = 0; k < K; ++k) {
    const double f = F[(int64_t)r * K + k], b = B[(int64_t)c * K + k];
    s = fma(f, b, s);
    a = fma(fabs(f), fabs(b), a);
  }
  C[i] = s;
  Cabs[i] = a;
}
__global__ void gen_f(double* F, int N, int K, unsigned long long seed) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= (int64_t)N * K) return;
  const int k = (int)(i % K);
  unsigned long long z = seed + (unsigned long long)i * 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  z ^= z >> 31;
  const double u = ((double)(z >> 11) * 0x1p-53) * 2.0 - 1.0;
  // Cholesky-factor-like columns: magnitudes decaying with the column index
  F[i] = u * 0.9 * exp(-3.0 * k / K) / sqrt(0.25 * K);
}

static PFN_cuTensorMapEncodeTiled_v12000 encode() {
  void* f = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
  return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
}
static bool map_i8(CUtensorMap* mp, const void* base, int kpad, int64_t rows, int box_rows) {
  cuuint64_t dims[2] = {(cuuint64_t)kpad, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)kpad};
  cuuint32_t box[2] = {(cuuint32_t)kKB, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  return encode()(mp, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides,
                  box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
}

int main(int argc, char** argv) {
  const int N = argc > 1 ? atoi(argv[1]) : 1000000;
  const int K = argc > 2 ? atoi(argv[2]) : 836;
  const int m = argc > 3 ? atoi(argv[3]) : 116;
  const int kpad = (K + kKB - 1) / kKB * kKB, mpad = (m + kBN - 1) / kBN * kBN;
  const int Np = (N + kBM - 1) / kBM * kBM;
  printf("N=%d K=%d m=%d (kpad %d, mpad %d)\n", N, K, m, kpad, mpad);
  double *F, *B, *C, *Cr, *Ca, *bs, *cs;
  int8_t *Fp, *Bp;
  cudaMalloc(&F, sizeof(double) * (size_t)N * K);
  cudaMalloc(&B, sizeof(double) * (size_t)m * K);
  cudaMalloc(&C, sizeof(double) * (size_t)N * m);
  cudaMalloc(&Cr, sizeof(double) * (size_t)N * m);
  cudaMalloc(&Ca, sizeof(double) * (size_t)N * m);
  cudaMalloc(&bs, sizeof(double) * m);
  cudaMalloc(&cs, sizeof(double) * mpad);
  cudaMalloc(&Fp, (size_t)kPl * Np * kpad);
  cudaMalloc(&Bp, (size_t)kPl * mpad * kpad);
  cudaMemset(Fp, 0, (size_t)kPl * Np * kpad);
  cudaMemset(Bp, 0, (size_t)kPl * mpad * kpad);
  gen_f<<<(unsigned)(((int64_t)N * K + 255) / 256), 256>>>(F, N, K, 1);
  // B' rows: random with per-row magnitudes 2^-8 .. 2^8
  std::vector<double> hb((size_t)m * K), hscale(m), hcs(mpad, 0.0);
  srand(3);
  for (int c = 0; c < m; ++c) {
    const double mag = std::ldexp(1.0, (rand() % 17) - 8);
    double mx = 0.0;
    for (int k = 0; k < K; ++k) {
      const double v = mag * ((rand() / (double)RAND_MAX) * 2.0 - 1.0);
      hb[(size_t)c * K + k] = v;
      mx = std::fmax(mx, std::fabs(v));
    }
    int e;
    std::frexp(mx, &e);  // mx = f 2^e, f in [0.5, 1)
    hscale[c] = std::ldexp(1.0, -e);
    hcs[c] = std::ldexp(1.0, e - 12);
  }
  cudaMemcpy(B, hb.data(), sizeof(double) * hb.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(bs, hscale.data(), sizeof(double) * m, cudaMemcpyHostToDevice);
  cudaMemcpy(cs, hcs.data(), sizeof(double) * mpad, cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  // slices
  cudaEventRecord(e0);
  slice_rows<<<(unsigned)(((int64_t)N * kpad + 255) / 256), 256>>>(F, K, N, K, kpad, nullptr, Fp,
                                                                    (int64_t)Np * kpad);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  printf("slice F: %.3f ms\n", ms);
  slice_rows<<<(unsigned)(((int64_t)m * kpad + 255) / 256), 256>>>(B, K, m, K, kpad, bs, Bp,
                                                                    (int64_t)mpad * kpad);
  CUtensorMap mA, mB;
  if (!map_i8(&mA, Fp, kpad, (int64_t)kPl * Np, kBM) || !map_i8(&mB, Bp, kpad, (int64_t)kPl * mpad, kBN)) {
    printf("tensor map encode failed\n");
    return 2;
  }
  const size_t smem = (size_t)kNst * kStage + 1024;
  cudaFuncSetAttribute(i8gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  dim3 grid(Np / kBM, mpad / kBN);
  auto run = [&] {
    i8gemm_kernel<<<grid, 192, smem>>>(mA, mB, Np, mpad, m, kpad / kKB, cs, C, m);
  };
  run();
  cudaError_t err = cudaDeviceSynchronize();
  printf("i8gemm first launch: %s\n", cudaGetErrorString(err));
  if (err != cudaSuccess) return 3;
  cudaEventRecord(e0);
  for (int i = 0; i < 5; ++i) run();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  const double tms = ms / 5;
  const double ops = 2.0 * 28 * (double)Np * mpad * kpad;
  printf("i8gemm: %.3f ms per GEMM (%.0f int8 TOPS on the 28 slice products; FP64-equivalent "
         "%.1f TF/s for 2 N m K = %.3g flop)\n",
         tms, ops / (tms * 1e-3) / 1e12, 2.0 * N * m * (double)K / (tms * 1e-3) / 1e12,
         2.0 * N * m * (double)K);
  ref_gemm<<<(unsigned)(((int64_t)N * m + 255) / 256), 256>>>(F, B, N, m, K, Cr, Ca);
  cudaDeviceSynchronize();
  std::vector<double> hc((size_t)N * m), hr((size_t)N * m), ha((size_t)N * m);
  cudaMemcpy(hc.data(), C, sizeof(double) * hc.size(), cudaMemcpyDeviceToHost);
  cudaMemcpy(hr.data(), Cr, sizeof(double) * hr.size(), cudaMemcpyDeviceToHost);
  cudaMemcpy(ha.data(), Ca, sizeof(double) * ha.size(), cudaMemcpyDeviceToHost);
  double maxrel = 0.0, num = 0.0, den = 0.0, maxabs = 0.0;
  for (size_t i = 0; i < hc.size(); ++i) {
    const double dd = std::fabs(hc[i] - hr[i]);
    maxabs = std::fmax(maxabs, dd);
    if (ha[i] > 0) maxrel = std::fmax(maxrel, dd / ha[i]);
    num += dd * dd;
    den += hr[i] * hr[i];
  }
  printf("error vs FP64: max |dC| %.3e, max |dC| / sum|F||B'| %.3e, ||dC||_F / ||C||_F %.3e (%s)\n",
         maxabs, maxrel, std::sqrt(num / den), cudaGetErrorString(cudaGetLastError()));
  return 0;
}
