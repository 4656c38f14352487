// i8cols.cu — standalone kernel columns A(:, S) (K5, Gaussian Gram mode, d <= 32, m <= 128)
// with the Gram products X X(S,:)^T on the 5th-generation tensor cores through int8 digit
// planes (Ozaki scheme I), leaving the shared FP64 pipe to the distance / exp epilogue.
//
// Why.  The FP64 K5 (update kernel, columns-only instantiation) spends ~32 FP64-pipe slots
// per output on the DMMA Gram (K = d padded to 32) and ~12 on the transform; the pipe is
// shared, so the Gram caps it at ~0.5 of what the epilogue alone could do
// (profiles/r02_cols_kernel_ncu_b120.txt).  Here the Gram runs on tcgen05 int8 and the
// FP64 pipe only combines the digit diagonals (7 ops) and evaluates the kernel (~13 ops).
//
// Representation (the residual GEMM's balanced base-2^7 digits, i8gemm.cu, one digit more):
// each point row x_i is scaled by 2^-e_i (max_k |x_ik| < 2^e_i) and held as 8 digits of
// x_i 2^(6 - e_i): x_ik = 2^(e_i - 6) sum_t f_t 2^(-7 t) + O(2^(e_i - 56)), |f_t| <= 64.  Then
//   x_i . x_j = 2^(e_i + e_j - 12) sum_{d < 8} 2^(-7 d) A_d(i, j),  A_d = sum_{t+u=d} f_t g_u^T
// (36 products; exact int32 diagonals in tensor memory, |A_d| < (d + 1) 2^17); the dropped
// products t + u >= 8 and the truncation bound the dot at ~2^-53 of
// 2^(e_i + e_j) sum_k 1, the FP64 DMMA Gram's own rounding level (7 digits measured 1.1e-13
// off the reference on unit-scale points: not kept).  D = ((-2 dot) + ||x_i||^2) + ||x_j||^2 follows the
// reference's Gram-trick order (oracle.hpp:71-90), then clamp, same-index pin and the kernel
// function exactly as the fused update kernel's epilogue (update_impl.cuh kfun_eval).
//
// Kernel: persistent, one CTA per SM, row tiles of 128 points; the column block (m <= 128,
// two halves of 64) stays resident in shared memory.  Warp 0 issues TMA (8 A planes per row
// tile, 32-byte rows, 32-byte swizzle, 4 stages), warp 1 the MMAs (M = 128, N = 64, K = 32,
// 36 products into 8 diagonal accumulators = 512 TMEM columns), warps 2-17 the epilogue
// (4 warps per TMEM lane quadrant, 16 columns each): each diagonal is read, folded into int32
// pairs and released to the next half's products at once, so the FP64 epilogue of one half
// overlaps the next half's MMAs.  Output column-major, out[c ld + r] (coalesced per column).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <mutex>

#include "common.cuh"
#include "kernels.h"
#include "update_impl.cuh"

namespace rpcb {

namespace {
constexpr int kCS = kI8ColsSlices;             // digits per operand (8 x 64 = 512 TMEM columns)
constexpr int kCBM = 128, kCBN = 64, kCKB = 32;  // rows per tile, MMA N, K bytes (d <= 32)
constexpr int kCNst = 4;                       // A stages
constexpr int kCApl = kCBM * kCKB;             // 4 KB per A plane
constexpr int kCAst = kCS * kCApl;             // 28 KB per stage
constexpr int kCBpl = 128 * kCKB;              // B plane (128 columns max)
constexpr int kCEpiWarps = 16;
constexpr int kCThreads = 64 + 32 * kCEpiWarps;
constexpr size_t kCSmem = (size_t)kCNst * kCAst + (size_t)kCS * kCBpl + 1024;
}  // namespace

// K-major operand tile of 32-byte rows with the 32-byte swizzle (one MMA K step per row)
__device__ __forceinline__ uint64_t umma_desc_sw32(uint32_t saddr) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1 << 16;           // leading byte offset (unused: swizzled K-major)
  d |= (uint64_t)(256 >> 4) << 32;  // stride byte offset: 8 rows x 32 B
  d |= (uint64_t)1 << 46;           // descriptor version (sm_100)
  d |= (uint64_t)6 << 61;           // SWIZZLE_32B
  return d;
}

// Single-thread roles (TMA, MMA issue) wait with a suspend hint instead of spinning, so they
// do not take issue slots from the epilogue warps on their schedulers.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile(
        "{\n.reg .pred p;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n"
        "selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity), "r"(1000000u)
        : "memory");
}

// Point digit planes: planes[t][row][32] (rows_pad rows, zero rows beyond n), xexp[row] = e.
// A thread per row; X packed [n][dpad] with zeros beyond d (pack_points).
__global__ void __launch_bounds__(256) xplanes_kernel(const double* __restrict__ X, int64_t dpad,
                                                      int d, int64_t n, int64_t rows_pad,
                                                      int8_t* __restrict__ planes,
                                                      int* __restrict__ xexp) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= rows_pad) return;
  uint32_t w[kCS][8];
#pragma unroll
  for (int t = 0; t < kCS; ++t)
#pragma unroll
    for (int q = 0; q < 8; ++q) w[t][q] = 0u;
  int e = 0;
  if (r < n) {
    const double* xr = X + r * dpad;
    double mx = 0.0;
    for (int k = 0; k < d; ++k) mx = fmax(mx, fabs(xr[k]));
    if (mx > 0.0) frexp(mx, &e);  // mx = f 2^e, f in [0.5, 1)
    const double sc = ldexp(64.0, -e);
    constexpr double kM = 6755399441055744.0;  // 1.5 * 2^52
#pragma unroll
    for (int k = 0; k < kCKB; ++k) {
      double rr = k < d ? xr[k] * sc : 0.0;  // |rr| < 64, exact power-of-two scaling
#pragma unroll
      for (int t = 0; t < kCS; ++t) {
        const double q = rr + kM;
        const uint32_t dg = (uint32_t)__double2loint(q) & 0xffu;
        w[t][k >> 2] |= dg << (8 * (k & 3));
        rr = (rr - (q - kM)) * 128.0;
      }
    }
    xexp[r] = e;
  }
#pragma unroll
  for (int t = 0; t < kCS; ++t) {
    uint4* dst = reinterpret_cast<uint4*>(planes + ((int64_t)t * rows_pad + r) * kCKB);
    dst[0] = make_uint4(w[t][0], w[t][1], w[t][2], w[t][3]);
    dst[1] = make_uint4(w[t][4], w[t][5], w[t][6], w[t][7]);
  }
}

// Column block: B planes [t][j][32] = the point planes of column point j (id in the proposal
// record), zero rows for m <= j < 128; per-column exponent, squared norm and id.
__global__ void __launch_bounds__(64) cplanes_kernel(const int8_t* __restrict__ planes,
                                                     int64_t rows_pad, const int* __restrict__ xexp,
                                                     const double* __restrict__ sqn,
                                                     const double* __restrict__ prop, int64_t rec,
                                                     int m, int8_t* __restrict__ bplanes,
                                                     double* __restrict__ cinfo) {
  const int j = blockIdx.x;
  const bool live = j < m;
  const int64_t id = live ? (int64_t)prop[(int64_t)j * rec] : 0;
  for (int i = threadIdx.x; i < kCS * 2; i += blockDim.x) {
    const int t = i >> 1, h = i & 1;
    uint4 v = make_uint4(0u, 0u, 0u, 0u);
    if (live) v = reinterpret_cast<const uint4*>(planes + ((int64_t)t * rows_pad + id) * kCKB)[h];
    reinterpret_cast<uint4*>(bplanes + ((int64_t)t * 128 + j) * kCKB)[h] = v;
  }
  if (threadIdx.x == 0) {
    cinfo[j] = live ? sqn[id] : 0.0;
    cinfo[128 + j] = live ? (double)id : -1.0;
    cinfo[256 + j] = live ? (double)xexp[id] : 0.0;
  }
}

template <int KF>
__global__ void __launch_bounds__(kCThreads, 1)
    i8cols_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                  int64_t rows_pad, int64_t n, int m, int ncolt, int64_t ntiles,
                  const int* __restrict__ xexp, const double* __restrict__ sqn,
                  const double* __restrict__ cinfo, double escale,
                  double* __restrict__ out, int64_t ld_out) {
  extern __shared__ __align__(1024) unsigned char smraw[];
  unsigned char* sm = smraw + ((1024u - (smem_u32(smraw) & 1023u)) & 1023u);
  unsigned char* sb = sm + kCNst * kCAst;  // resident B planes
  __shared__ uint64_t afull[kCNst], aempty[kCNst], bfull, done, drained[kCS];
  __shared__ uint32_t tmem_base_s;
  // per column: {||x_j||^2, bits (lo: high word of -2^(e_j - 60), hi: pinned row or -1)}
  __shared__ double2 s_col[128];
  __shared__ double s_exp2[64];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kCNst; ++s) {
      mbar_init(&afull[s], 1);
      mbar_init(&aempty[s], 1);
    }
    mbar_init(&bfull, 1);
    mbar_init(&done, 1);
    for (int d = 0; d < kCS; ++d) mbar_init(&drained[d], kCEpiWarps);
    mbar_fence_init();
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
  }
  for (int i = threadIdx.x; i < 128; i += blockDim.x) {
    // pinned row of column i (-1: none; ids < 2^31 here, n <= rows of one device buffer);
    // high word of -2^(e_j - 60): the row adds e_i << 20
    const int id = (int)cinfo[128 + i];
    const int ce = (int)(0x80000000u | (uint32_t)(((int)cinfo[256 + i] - 60 + 1023) << 20));
    s_col[i] = make_double2(cinfo[i], __hiloint2double(id, ce));
  }
  if (threadIdx.x < 64) s_exp2[threadIdx.x] = exp2((double)threadIdx.x / 64.0);
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
    if (elect_one()) {
      mbar_arrive_expect_tx(&bfull, kCS * ncolt * kCBN * kCKB);
      for (int u = 0; u < kCS; ++u)
        for (int h = 0; h < ncolt; ++h)
          tma_load_2d(sb + u * kCBpl + h * kCBN * kCKB, &tmB, 0, u * 128 + h * kCBN, &bfull);
      int it = 0;
      for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
        const int s = it % kCNst;
        if (it >= kCNst) mbar_wait_sleep(&aempty[s], ((it / kCNst) - 1) & 1);
        mbar_arrive_expect_tx(&afull[s], kCAst);
        unsigned char* st = sm + s * kCAst;
        for (int t = 0; t < kCS; ++t)
          tma_load_2d(st + t * kCApl, &tmA, 0, (int)(t * rows_pad + tile * kCBM), &afull[s]);
      }
    }
  } else if (warp == 1) {
    if (elect_one()) {
      // kind::i8: D s32, A and B signed int8, both K-major, M = 128, N = 64 (a partial last
      // column half: N = its live columns rounded up to 16)
      const uint32_t idesc0 = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(kCBM >> 4) << 24);
      mbar_wait_sleep(&bfull, 0);
      const uint32_t bb = smem_u32(sb);
      int it = 0, job = 0;
      for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
        const int s = it % kCNst;
        mbar_wait_sleep(&afull[s], (it / kCNst) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        const uint32_t ba = smem_u32(sm + s * kCAst);
        for (int h = 0; h < ncolt; ++h, ++job) {
          const int nmma = min(kCBN, (m - h * kCBN + 15) & ~15);
          const uint32_t idesc = idesc0 | ((uint32_t)(nmma >> 3) << 17);
#pragma unroll
          for (int d = 0; d < kCS; ++d) {
            if (job > 0) {
              mbar_wait_sleep(&drained[d], (job - 1) & 1);
              asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
            }
#pragma unroll
            for (int t = 0; t <= d; ++t) {
              const uint64_t da = umma_desc_sw32(ba + t * kCApl);
              const uint64_t db = umma_desc_sw32(bb + (d - t) * kCBpl + h * kCBN * kCKB);
              const uint32_t accum = t != 0;
              asm volatile(
                  "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                  "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(
                      tbase + (uint32_t)(d * kCBN)),
                  "l"(da), "l"(db), "r"(idesc), "r"(accum));
            }
          }
          asm volatile(
              "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                  smem_u32(&done)));
        }
        asm volatile(
            "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                smem_u32(&aempty[s])));
      }
    }
  } else {
    const int q = warp & 3;           // TMEM lane quadrant this warp may read
    const int cs = (warp - 2) >> 2;   // 16-column slice of the 64-column half
    int job = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      const int64_t r = tile * kCBM + q * 32 + lane;
      const bool rin = r < n;
      const double sqr = rin ? __ldg(sqn + r) : 0.0;
      const int ri = (int)r;
      const int er = (rin ? __ldg(xexp + r) : 0) << 20;
      double* orow = out + r;
      for (int h = 0; h < ncolt; ++h, ++job) {
        mbar_wait(&done, job & 1);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        const int c0 = h * kCBN + cs * 16;
        if (c0 >= m) {  // no live column in this warp's slice (warp-uniform): release only
          __syncwarp();
          if (lane == 0)
            for (int d = 0; d < kCS; ++d) mbar_arrive(&drained[d]);
          continue;
        }
        // Diagonals read two at a time and released at once; folded as they arrive:
        // P_p = A_{2p} 2^7 + A_{2p+1} (exact int32, |A_d| < (d + 1) 2^17), then
        // sum_d 2^(-7 d) A_d = 2^-49 S,  S = H 2^28 + L,  H = P0 2^14 + P1,  L = P2 2^14 + P3
        // (|H|, |L| < 2^40: int64, to double through the 1.5 2^52 bit pattern; one rounding).
        int P[2][16];
        double S[16];
#pragma unroll
        for (int p = 0; p < kCS / 2; ++p) {
          uint32_t v[2][16];
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const uint32_t ta =
                tbase + ((uint32_t)(q * 32) << 16) + (uint32_t)((2 * p + e) * kCBN + cs * 16);
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, "
                "%10, %11, %12, %13, %14, %15}, [%16];\n"
                : "=r"(v[e][0]), "=r"(v[e][1]), "=r"(v[e][2]), "=r"(v[e][3]), "=r"(v[e][4]),
                  "=r"(v[e][5]), "=r"(v[e][6]), "=r"(v[e][7]), "=r"(v[e][8]), "=r"(v[e][9]),
                  "=r"(v[e][10]), "=r"(v[e][11]), "=r"(v[e][12]), "=r"(v[e][13]), "=r"(v[e][14]),
                  "=r"(v[e][15])
                : "r"(ta));
          }
          asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
          asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
          __syncwarp();
          if (lane == 0) {
            mbar_arrive(&drained[2 * p]);
            mbar_arrive(&drained[2 * p + 1]);
          }
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int pv = (int)v[0][j] * 128 + (int)v[1][j];
            if ((p & 1) == 0) {
              P[p >> 1][j] = pv;
            } else {
              const long long w = (long long)P[p >> 1][j] * 16384 + (long long)pv +
                                  0x4338000000000000LL;
              const double x = __longlong_as_double(w) - 6755399441055744.0;
              S[j] = p == 1 ? x : fma(S[j], 268435456.0, x);
            }
          }
        }
        // warp-uniform: every lane's row and all 16 columns live -> stores without predicates
        const bool full = (c0 + 16 <= m) && (tile * kCBM + q * 32 + 32 <= n);
        double* op = orow + (int64_t)c0 * ld_out;  // advanced by one column per element
#pragma unroll
        for (int j = 0; j < 16; ++j, op += ld_out) {
          const int c = c0 + j;
          const double2 cinf = s_col[c];
          // -2 dot = -2 * 2^(e_i + e_j - 12) * 2^-49 * S = S * (-2^(e_i + e_j - 60)), exact, so
          // fma(S, sc, |x_i|^2) is the reference's ((-2 dot) + |x_i|^2) rounding
          const double sc = __hiloint2double(__double2loint(cinf.y) + er, 0);
          double dd = __dadd_rn(fma(S[j], sc, sqr), cinf.x);
          // clamp at 0 and the same-index pin (oracle.hpp:84-88), integer tests
          if ((__double2hiint(dd) < 0) | (ri == __double2hiint(cinf.y))) dd = 0.0;
          double val;
          if constexpr (KF == kFunExp) {
            // exp_tab (update_impl.cuh) inline, the -708 clamp as one FP64 max (same values)
            constexpr double kShift = 6755399441055744.0;  // 1.5 * 2^52
            const double x = fmax(dd * escale, -708.0);
            const double ks = fma(x, kExpC[0], kShift);
            const int k = __double2loint(ks);
            const double kd = ks - kShift;
            double r = fma(kd, kExpC[1], x);
            r = fma(kd, kExpC[2], r);
            double qq = fma(r, kExpC[3], kExpC[4]);
            qq = fma(qq, r, kExpC[5]);
            qq = fma(qq, r, kExpC[6]);
            qq = fma(qq * r, r, r);
            const double t = s_exp2[k & 63];
            const double y = fma(t, qq, t);
            val = __hiloint2double(__double2hiint(y) + ((k >> 6) << 20), __double2loint(y));
          } else {
            val = kfun_eval(dd, KF, escale, s_exp2);
          }
          if (full || (rin && c < m)) __stcs(op, val);
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tbase));
}

static bool i8c_map(CUtensorMap* mp, const void* base, int64_t rows, int box_rows) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)kCKB, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)kCKB};
  cuuint32_t box[2] = {(cuuint32_t)kCKB, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  return fn(mp, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_32B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int64_t i8cols_plane_bytes(int64_t n) { return (int64_t)kCS * ((n + kCBM - 1) / kCBM * kCBM) * kCKB; }

void launch_i8cols_prep(const double* X, int64_t dpad, int d, int64_t n, int8_t* planes,
                        int* xexp, cudaStream_t st) {
  const int64_t rows_pad = (n + kCBM - 1) / kCBM * kCBM;
  xplanes_kernel<<<(unsigned)((rows_pad + 255) / 256), 256, 0, st>>>(X, dpad, d, n, rows_pad,
                                                                     planes, xexp);
}

int launch_i8cols(const int8_t* planes, const int* xexp, const double* sqn, int64_t n,
                  const double* prop, int64_t rec, int m, int kfun, double escale,
                  int8_t* bplanes, double* cinfo, double* out, int64_t ld_out, cudaStream_t st) {
  if (m < 1 || m > 128 || n <= 0 || n >= ((int64_t)1 << 31)) return -1;
  const int64_t rows_pad = (n + kCBM - 1) / kCBM * kCBM;
  cplanes_kernel<<<128, 64, 0, st>>>(planes, rows_pad, xexp, sqn, prop, rec, m, bplanes, cinfo);
  CUtensorMap mA, mB;
  if (!i8c_map(&mA, planes, (int64_t)kCS * rows_pad, kCBM) ||
      !i8c_map(&mB, bplanes, (int64_t)kCS * 128, kCBN))
    return -3;
  const int ncolt = (m + kCBN - 1) / kCBN;
  const int64_t ntiles = rows_pad / kCBM;
  const unsigned grid = (unsigned)std::min<int64_t>(ntiles, num_sms());
  auto go = [&](auto kern) {
    if (ensure_smem_attr((const void*)kern, (int)kCSmem) != cudaSuccess) return -2;
    kern<<<grid, kCThreads, kCSmem, st>>>(mA, mB, rows_pad, n, m, ncolt, ntiles, xexp, sqn, cinfo,
                                          escale, out, ld_out);
    return 0;
  };
  if (kfun == kFunMatern32) return go(i8cols_kernel<kFunMatern32>);
  if (kfun == kFunMatern52) return go(i8cols_kernel<kFunMatern52>);
  return go(i8cols_kernel<kFunExp>);
}

}  // namespace rpcb
