#pragma once
// update_impl.cuh — K5+K6: the fused round update, one CTA per BM-row tile of the shard.
//
// For the accepted pivots S (m columns) of a round it computes, without ever
// materialising the N x m kernel panel in HBM:
//   phase 1  acc  = -A(R, S)                      (K5: kernel columns, fused)
//            acc += F(R, :kcur) F(S, :kcur)^T     (K6: FP64 DMMA GEMM)
//            G    = -acc = A(R,S) - F F_S^T       (rpcholesky.hpp:378-383)
//            G is parked in its final place F(R, kcur:kcur+m) (L2-resident)
//   phase 2  G   <- G L^{-T}: DMMA GEMM whose A operand is G streamed back by TMA
//            (right_solve_lower_transposed, rpcholesky.hpp:147-151, 384)
//   epilogue F(R, kcur:kcur+m) = G ; u(R) = max(u - rowwise||G||^2, 0) ;
//            per-tile ||G||_F^2 partial                  (rpcholesky.hpp:385-388)
// Kernel columns (oracle.hpp:71-90, kernels.hpp:60-64): the Gaussian Gram term
// X(R,:) X(S,:)^T runs on the same DMMA pipeline as the residual GEMM (K = dpad),
// followed by the clamp / same-index pin / exp epilogue in registers; Gaussian-direct
// and l1 distances run on the FP64 CUDA cores from the same staged X tiles in
// ascending coordinate order (bit-identical distances to the reference's sums).
//
// Execution: persistent CTAs (one per SM) of 8 warps walk row tiles; thread 0
// streams [rows][16] fp64 tiles with 2D TMA (cp.async.bulk.tensor, 128B swizzle)
// into an S-stage ring guarded by full/empty mbarriers, running ahead across tile
// boundaries (the next tile's first tiles load during this tile's epilogue); all
// warps run mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4).  Operand rows are permuted inside 8-row
// groups (perm8, common.cuh) so every fragment load is bank-conflict free.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <mutex>

#include "common.cuh"
#include "kernels.h"

namespace rpcb {

template <int WC, int NFW>
struct UCfg {
  static constexpr int NCW = 8;             // warps (all consumers; thread 0 also issues TMA)
  static constexpr int NT = 32 * NCW;
  static constexpr int WR = NCW / WC;
  static constexpr int BM = 16 * WR;        // tile rows
  static constexpr int NF = WC * NFW;       // 8-column fragments
  static constexpr int NB = 8 * NF;         // tile columns (m padded)
  static constexpr int S = 4;               // pipeline stages
  static constexpr int A_BYTES = BM * 128;
  static constexpr int B_BYTES = NB * 128;
  static constexpr int STAGE = A_BYTES + B_BYTES;
  static constexpr int MISC = NB * 16 + WC * BM * 8 + BM * 8 + (2 * S) * 8;
  static constexpr int SMEM = S * STAGE + MISC + 1024;
};

// Compact exp for the kernel-column epilogue (arguments are <= 0 here):
// Cody-Waite reduction x = n ln2 + r, |r| <= ln2/2, degree-13 Taylor polynomial
// (truncation < 5e-18 relative), exact power-of-two scaling in two steps so
// results down to the subnormal range stay correct.  ~1 ulp, branch-free.
__device__ __forceinline__ double exp_compact(double x) {
  x = fmax(x, -745.5);
  const double n = rint(x * 1.4426950408889634);
  double r = fma(n, -6.93147180369123816490e-01, x);
  r = fma(n, -1.90821492927058770002e-10, r);
  double q = 1.6059043836821613e-10;          // 1/13!
  q = fma(q, r, 2.0876756987868100e-09);      // 1/12!
  q = fma(q, r, 2.5052108385441720e-08);      // 1/11!
  q = fma(q, r, 2.7557319223985893e-07);      // 1/10!
  q = fma(q, r, 2.7557319223985888e-06);      // 1/9!
  q = fma(q, r, 2.4801587301587302e-05);      // 1/8!
  q = fma(q, r, 1.9841269841269841e-04);      // 1/7!
  q = fma(q, r, 1.3888888888888889e-03);      // 1/6!
  q = fma(q, r, 8.3333333333333332e-03);      // 1/5!
  q = fma(q, r, 4.1666666666666664e-02);      // 1/4!
  q = fma(q, r, 1.6666666666666666e-01);      // 1/3!
  q = fma(q, r, 0.5);
  q = fma(q, r, 1.0);
  q = fma(q, r, 1.0);
  const int ni = (int)n;
  const int k1 = ni >> 1, k2 = ni - k1;
  const double s1 = __longlong_as_double((long long)(k1 + 1023) << 52);
  const double s2 = __longlong_as_double((long long)(k2 + 1023) << 52);
  return q * s1 * s2;
}

template <int WC, int NFW, bool GRAM, int MINB>
__global__ void __launch_bounds__(UCfg<WC, NFW>::NT, MINB)
    update_kernel(UpdateParams p, const __grid_constant__ CUtensorMap tmX,
                  const __grid_constant__ CUtensorMap tmXS, const __grid_constant__ CUtensorMap tmF,
                  const __grid_constant__ CUtensorMap tmFS, const __grid_constant__ CUtensorMap tmG,
                  const __grid_constant__ CUtensorMap tmL) {
  using C = UCfg<WC, NFW>;
  constexpr int BM = C::BM, S = C::S, NCW = C::NCW;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  // 1024-byte aligned ring (128B-swizzle atoms).  Offsets stay relative to the
  // __shared__ array so every fragment load is an LDS with an immediate offset.
  const uint32_t align = (1024u - (smem_u32(smem_raw) & 1023u)) & 1023u;
  unsigned char* stages = smem_raw + align;
  double* s_sqnS = reinterpret_cast<double*>(stages + S * C::STAGE);
  double* s_idS = s_sqnS + C::NB;
  double* s_rown = s_idS + C::NB;  // [WC][BM]
  double* s_rowg2 = s_rown + WC * BM;
  uint64_t* full = reinterpret_cast<uint64_t*>(s_rowg2 + BM);
  uint64_t* empty = full + S;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int m = p.m, kcur = p.kcur;
  const int nX = p.dchunks;
  const int nFk = (kcur + 15) >> 4;
  // Phase-2 A tiles start at F column kcur - koff: TMA box starts must be 16-byte
  // aligned in the inner dimension, so for odd kcur one extra leading column is
  // loaded and multiplied by the zero column 0 of the shifted L^{-1} (koff = 1).
  const int koff = kcur & 1;
  const int nL = p.columns_only ? 0 : (m + koff + 15) >> 4;
  const int T = nX + nFk + nL;               // chunks per tile
  const int ntiles = (int)((p.n_loc + BM - 1) / BM);
  const int my_tiles = blockIdx.x < ntiles ? (ntiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  const int total = my_tiles * T;            // chunks this CTA consumes (persistent)

  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCW);
    }
    mbar_fence_init();
    tma_prefetch_desc(&tmX);
    tma_prefetch_desc(&tmXS);
    tma_prefetch_desc(&tmF);
    tma_prefetch_desc(&tmFS);
    tma_prefetch_desc(&tmG);
    tma_prefetch_desc(&tmL);
  }
  for (int n = tid; n < C::NB; n += C::NT) {
    s_sqnS[n] = p.sqnS[n];
    s_idS[n] = p.idS[n];
  }
  __syncthreads();

  // ---- producer (thread 0): issue chunk `issued` when its stage is free and, for
  // phase-2 chunks of tile k, once that tile's G is parked (parked > k).
  int issued = 0;      // meaningful in thread 0 only
  int parked = 0;      // tiles whose G has been parked (CTA-uniform)
  auto pump = [&](int done_w0) {
    if (tid != 0) return;
    while (issued < total && issued < done_w0 + S) {
      const int k = issued / T, c = issued - k * T;
      if (c >= nX + nFk && parked <= k) break;
      const int s = issued % S;
      if (issued >= S) mbar_wait(&empty[s], ((issued / S) & 1) ^ 1);
      unsigned char* As = stages + s * C::STAGE;
      unsigned char* Bs = As + C::A_BYTES;
      const int r0 = (int)((blockIdx.x + (int64_t)k * gridDim.x) * BM);
      mbar_arrive_expect_tx(&full[s], C::STAGE);
      if (c < nX) {
        tma_load_2d(As, &tmX, 16 * c, r0, &full[s]);
        tma_load_2d(Bs, &tmXS, 16 * c, 0, &full[s]);
      } else if (c < nX + nFk) {
        tma_load_2d(As, &tmF, 16 * (c - nX), r0, &full[s]);
        tma_load_2d(Bs, &tmFS, 16 * (c - nX), 0, &full[s]);
      } else {
        tma_load_2d(As, &tmG, kcur - koff + 16 * (c - nX - nFk), r0, &full[s]);
        tma_load_2d(Bs, &tmL, 16 * (c - nX - nFk), 0, &full[s]);
      }
      ++issued;
    }
  };
  pump(0);

  const int g = lane >> 2, t = lane & 3;
  const int wr = warp / WC, wc = warp % WC;
  const int pg = perm8(g);
  int arow[2];  // tile rows of this lane's A-fragment rows
#pragma unroll
  for (int fr = 0; fr < 2; ++fr) arow[fr] = wr * 16 + 8 * fr + pg;

  // Swizzled byte offsets of this lane's fragment element (row & 7 == pg, k = 4s + t)
  // inside any 8-row group: identical for the A and B operands, so every fragment
  // load below is base + compile-time immediate + one of these four registers.
  uint32_t foff[4];
#pragma unroll
  for (int s = 0; s < 4; ++s) foff[s] = swz_off(pg, 4 * s + t);
  const uint32_t a_base = (uint32_t)(wr * 16) * 128u;
  const uint32_t b_base = (uint32_t)(wc * NFW) * 1024u;

  double acc[2][NFW][2];

  // q_lo: first fragment that can be non-zero (phase 2 skips the zero upper triangle
  // of L^{-T}; phase 1 passes 0).
  auto mma_stage = [&](uint32_t st_off, int q_lo) {
    const unsigned char* Aw = stages + st_off + a_base;
    const unsigned char* Bw = stages + st_off + C::A_BYTES + b_base;
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      double a[2];
#pragma unroll
      for (int fr = 0; fr < 2; ++fr) a[fr] = *reinterpret_cast<const double*>(Aw + fr * 1024 + foff[s]);
#pragma unroll
      for (int q = 0; q < NFW; ++q) {
        if (q < q_lo) continue;
        const double bv = *reinterpret_cast<const double*>(Bw + q * 1024 + foff[s]);
#pragma unroll
        for (int fr = 0; fr < 2; ++fr) dmma884(acc[fr][q][0], acc[fr][q][1], a[fr], bv);
      }
    }
  };

  // Phase-2 variant: the four k-steps' A fragments are loaded once, then each B
  // fragment column block is either skipped whole (upper triangle of L^{-T}) or
  // accumulated over all four k-steps — one uniform branch per fragment per chunk.
  auto mma_stage_tri = [&](uint32_t st_off, int q_lo) {
    const unsigned char* Aw = stages + st_off + a_base;
    const unsigned char* Bw = stages + st_off + C::A_BYTES + b_base;
    double a[4][2];
#pragma unroll
    for (int s = 0; s < 4; ++s)
#pragma unroll
      for (int fr = 0; fr < 2; ++fr) a[s][fr] = *reinterpret_cast<const double*>(Aw + fr * 1024 + foff[s]);
#pragma unroll
    for (int q = 0; q < NFW; ++q) {
      if (q < q_lo) continue;
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        const double bv = *reinterpret_cast<const double*>(Bw + q * 1024 + foff[s]);
#pragma unroll
        for (int fr = 0; fr < 2; ++fr) dmma884(acc[fr][q][0], acc[fr][q][1], a[s][fr], bv);
      }
    }
  };

  auto dist_stage = [&](uint32_t st_off) {
    const unsigned char* As = stages + st_off;
    const unsigned char* Bs = As + C::A_BYTES;
    const bool l1 = p.kind == kL1;
#pragma unroll 1
    for (int j = 0; j < 16; ++j) {
      double xr[2];
#pragma unroll
      for (int fr = 0; fr < 2; ++fr) xr[fr] = *reinterpret_cast<const double*>(As + swz_off(arow[fr], j));
#pragma unroll
      for (int q = 0; q < NFW; ++q) {
        const int Q = wc * NFW + q;
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          const double xs = *reinterpret_cast<const double*>(Bs + swz_off(8 * Q + perm8(2 * t + v), j));
#pragma unroll
          for (int fr = 0; fr < 2; ++fr) {
            const double df = __dsub_rn(xr[fr], xs);
            acc[fr][q][v] = l1 ? __dadd_rn(acc[fr][q][v], fabs(df))
                               : __dadd_rn(acc[fr][q][v], __dmul_rn(df, df));
          }
        }
      }
    }
  };

  int cons = 0;  // chunks consumed by this warp so far (CTA-uniform in practice)
  auto consume = [&](auto&& body) {
    const int s = cons % S;
    mbar_wait(&full[s], (cons / S) & 1);
    __syncwarp();
    body((uint32_t)(s * C::STAGE));
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    ++cons;
    if (warp == 0) pump(cons);
  };

#pragma unroll 1
  for (int k = 0; k < my_tiles; ++k) {
    const int tile = (int)blockIdx.x + k * (int)gridDim.x;
    const int64_t tile_row0 = (int64_t)tile * BM;
#pragma unroll
    for (int fr = 0; fr < 2; ++fr)
#pragma unroll
      for (int q = 0; q < NFW; ++q) acc[fr][q][0] = acc[fr][q][1] = 0.0;

    // ---- phase 1a: kernel-column distances / Gram products (X tiles) -------------
#pragma unroll 1
    for (int c = 0; c < nX; ++c) {
      if constexpr (GRAM) consume([&](uint32_t so) { mma_stage(so, 0); });
      else consume([&](uint32_t so) { dist_stage(so); });
    }
    // ---- acc (Gram dot / distance) -> -A(R, S) ------------------------------------
    {
      // exponent = D * (-0.5 / sigma^2) (Gaussian) or D * (-1 / sigma) (l1): one multiply
      // instead of the reference's division, <= 1 ulp apart (kernel values agree to 1e-15).
      const double escale = (!GRAM && p.kind == kL1) ? -1.0 / p.sigma : -0.5 / (p.sigma * p.sigma);
#pragma unroll
      for (int fr = 0; fr < 2; ++fr) {
        const int64_t grow = tile_row0 + arow[fr];
        const bool rin = grow < p.n_loc;
        const double sqr = rin ? p.sqn[grow] : 0.0;
        const double gid = (double)(p.row0 + grow);
#pragma unroll
        for (int q = 0; q < NFW; ++q) {
#pragma unroll
          for (int v = 0; v < 2; ++v) {
            const int col = 8 * (wc * NFW + q) + 2 * t + v;
            double val = 0.0;
            if (col < m && rin) {
              double dd = acc[fr][q][v];
              if (GRAM) {
                dd = __dadd_rn(__dadd_rn(-2.0 * dd, sqr), s_sqnS[col]);
                if (dd < 0.0) dd = 0.0;
                if (gid == s_idS[col]) dd = 0.0;
              }
              val = exp_compact(dd * escale);
            }
            acc[fr][q][v] = -val;
          }
        }
      }
    }
    // ---- phase 1b: residual GEMM F(R,:) F(S,:)^T (F tiles) ---------------------------
#pragma unroll 1
    for (int c = 0; c < nFk; ++c) consume([&](uint32_t so) { mma_stage(so, 0); });

    if (p.columns_only) {  // standalone K5: A(R, S) -> column-major output
#pragma unroll
      for (int fr = 0; fr < 2; ++fr) {
        const int64_t grow = tile_row0 + arow[fr];
        if (grow >= p.n_loc) continue;
#pragma unroll
        for (int q = 0; q < NFW; ++q)
#pragma unroll
          for (int v = 0; v < 2; ++v) {
            const int col = 8 * (wc * NFW + q) + 2 * t + v;
            if (col < m) p.cols_out[(int64_t)col * p.ld_out + grow] = -acc[fr][q][v];
          }
      }
      continue;
    }

    // ---- park G = -acc in F(R, kcur:kcur+m) for phase 2 --------------------------
#pragma unroll
    for (int fr = 0; fr < 2; ++fr) {
      const int64_t grow = tile_row0 + arow[fr];
      double* frow = p.F + grow * p.ldf + kcur;
#pragma unroll
      for (int q = 0; q < NFW; ++q)
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          const int col = 8 * (wc * NFW + q) + 2 * t + v;
          if (col < m && grow < p.n_loc) frow[col] = -acc[fr][q][v];
          acc[fr][q][v] = 0.0;
        }
    }
    fence_proxy_async_global();
    __syncthreads();
    parked = k + 1;
    if (warp == 0) pump(cons);

    // ---- phase 2: G L^{-T} ------------------------------------------------------------
#pragma unroll 1
    for (int j = 0; j < nL; ++j) {
      // chunk j covers G columns [16j - koff, 16j + 16 - koff); L^{-T}[k][n] = 0 for n < k,
      // so fragments whose 8 columns all lie below 16j - koff contribute nothing.
      const int q_lo = max(0, (16 * j - koff) / 8 - wc * NFW);
      consume([&](uint32_t so) { mma_stage_tri(so, q_lo); });
    }

    // ---- epilogue ------------------------------------------------------------------
    double rs[2] = {0.0, 0.0};
#pragma unroll
    for (int fr = 0; fr < 2; ++fr) {
      const int64_t grow = tile_row0 + arow[fr];
      const bool rin = grow < p.n_loc;
      double* frow = p.F + grow * p.ldf + kcur;
#pragma unroll
      for (int q = 0; q < NFW; ++q)
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          const int col = 8 * (wc * NFW + q) + 2 * t + v;
          if (col < m && rin) {
            const double val = acc[fr][q][v];
            frow[col] = val;
            rs[fr] = fma(val, val, rs[fr]);
          }
        }
      rs[fr] += __shfl_xor_sync(0xffffffffu, rs[fr], 1);
      rs[fr] += __shfl_xor_sync(0xffffffffu, rs[fr], 2);
      if (t == 0) s_rown[wc * BM + arow[fr]] = rs[fr];
    }
    __syncthreads();
    if (tid < BM) {
      const int64_t grow = tile_row0 + tid;
      double s2 = 0.0;
#pragma unroll
      for (int w = 0; w < WC; ++w) s2 = __dadd_rn(s2, s_rown[w * BM + tid]);
      if (grow < p.n_loc) {
        const double un = __dsub_rn(p.u[grow], s2);
        p.u[grow] = un < 0.0 ? 0.0 : un;
      } else {
        s2 = 0.0;
      }
      s_rowg2[tid] = s2;
    }
    __syncthreads();
    if (tid == 0) {
      double s2 = 0.0;
      for (int r = 0; r < BM; ++r) s2 = __dadd_rn(s2, s_rowg2[r]);
      p.tile_g2[tile] = s2;
    }
  }
}

// ---------------------------------------------------------------------------
// host side: tensor maps + dispatch
// ---------------------------------------------------------------------------
inline PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  });
  return fn;
}

// [rows][ld] row-major fp64, inner extent `inner` elements, box {16, box_rows}, 128B swizzle
inline bool make_map(CUtensorMap* m, const double* base, uint64_t inner, uint64_t rows,
                     uint64_t ld, uint32_t box_rows) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {std::max<uint64_t>(inner, 1), std::max<uint64_t>(rows, 1)};
  cuuint64_t strides[1] = {ld * sizeof(double)};
  cuuint32_t box[2] = {16, box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides,
                  box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

inline int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

template <int WC, int NFW, bool GRAM, int MINB>
int launch_t(const UpdateParams& p, cudaStream_t st) {
  using C = UCfg<WC, NFW>;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(update_kernel<WC, NFW, GRAM, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             C::SMEM) != cudaSuccess)
      return -2;
    attr = true;
  }
  CUtensorMap mX, mXS, mF, mFS, mG, mL;
  bool ok = make_map(&mX, p.X, p.dpad, p.n_loc, p.dpad, C::BM) &&
            make_map(&mXS, p.xs, p.dpad, C::NB, p.dpad, C::NB) &&
            make_map(&mF, p.F, p.kcur, p.n_loc, p.ldf, C::BM) &&
            make_map(&mFS, p.fs, p.kcur, C::NB, p.ldfs, C::NB) &&
            make_map(&mG, p.F, p.kcur + p.m, p.n_loc, p.ldf, C::BM) &&
            make_map(&mL, p.linv, p.ldl, C::NB, p.ldl, C::NB);
  if (!ok) return -3;
  // persistent: one CTA per SM, tiles strided by the grid (p.tile_g2 is per tile)
  const int64_t ntiles = (p.n_loc + C::BM - 1) / C::BM;
  const unsigned grid = (unsigned)std::min<int64_t>(ntiles, (int64_t)MINB * num_sms());
  if (grid)
    update_kernel<WC, NFW, GRAM, MINB><<<grid, C::NT, C::SMEM, st>>>(p, mX, mXS, mF, mFS, mG, mL);
  return C::BM;
}

}  // namespace rpcb
