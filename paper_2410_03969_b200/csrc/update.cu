// update.cu — K5+K6: the fused round update, one CTA per BM-row tile of the shard.
//
// For the accepted pivots S (m columns) of a round it computes, without ever
// writing the N x m kernel panel to HBM:
//   phase 1  acc  = -A(R, S)                      (K5: kernel columns, fused)
//            acc += F(R, :kcur) F(S, :kcur)^T     (K6: FP64 DMMA GEMM)
//            G    = -acc  = A(R,S) - F F_S^T      (rpcholesky.hpp:378-383)
//   phase 2  G   <- G L^{-T}  as a DMMA GEMM with the precomputed L^{-1}
//            (right_solve_lower_transposed, rpcholesky.hpp:147-151, 384)
//   epilogue F(R, kcur:kcur+m) = G ; u(R) = max(u - rowwise||G||^2, 0) ;
//            per-tile ||G||_F^2 partial                  (rpcholesky.hpp:385-388)
// Kernel columns (oracle.hpp:71-90, kernels.hpp:60-64): the Gaussian Gram term
// X(R,:) X(S,:)^T runs on the same DMMA pipeline as the residual GEMM (K = dpad),
// followed by the clamp / same-index pin / exp epilogue in registers; the
// Gaussian-direct and l1 distances run on the FP64 CUDA cores from the same
// staged X tiles, accumulating coordinates in ascending order (bit-identical
// distances to the reference's sequential sums).
//
// Data movement: cp.async (LDGSTS) multi-stage pipeline of [rows][16] fp64 tiles
// with the 128-byte swizzle; DMMA fragments use the stride-2 row map so every
// fragment load is bank-conflict free (common.cuh).
#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace rpcb {

template <int WC, int NFW>
struct UCfg {
  static constexpr int NF = WC * NFW;  // 8-column fragments
  static constexpr int NB = 8 * NF;    // tile columns (padded m)
  static constexpr int NBK = 16 * ((NF + 1) / 2);
  static constexpr int WR = 8 / WC;
  static constexpr int BM = 16 * WR;   // tile rows
  static constexpr int S1 = (WC == 1) ? 4 : 3;
  static constexpr int S2 = (WC == 1) ? 3 : 2;
  static constexpr int A_BYTES = BM * 128;
  static constexpr int B_BYTES = NB * 128;
  static constexpr int STAGE = A_BYTES + B_BYTES;
  static constexpr int GT_BYTES = BM * NBK * 8;
  static constexpr int FIN_LD = NB + 1;
  static constexpr int FIN_BYTES = BM * FIN_LD * 8;
  static constexpr int R1a = S1 * STAGE > GT_BYTES ? S1 * STAGE : GT_BYTES;
  static constexpr int R1 = ((R1a > FIN_BYTES ? R1a : FIN_BYTES) + 1023) / 1024 * 1024;
  static constexpr int R2 = S2 * B_BYTES;
  static constexpr int MISC = NB * (4 + 8 + 8) + BM * 8;
  static constexpr int SMEM = R1 + R2 + MISC + 1024;
};

__device__ __forceinline__ int colmap(int Q, int n8, int NF) {
  return ((Q | 1) < NF) ? (16 * (Q >> 1) + 2 * n8 + (Q & 1)) : (16 * (Q >> 1) + n8);
}

__device__ __forceinline__ double lds64(const unsigned char* base, uint32_t off) {
  return *reinterpret_cast<const double*>(base + off);
}

template <int WC, int NFW>
__global__ void __launch_bounds__(256, 1) update_kernel(UpdateParams p) {
  using C = UCfg<WC, NFW>;
  constexpr int NF = C::NF, NB = C::NB, BM = C::BM;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem =
      (unsigned char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  unsigned char* r1 = smem;
  unsigned char* r2 = smem + C::R1;
  int* s_pos = reinterpret_cast<int*>(r2 + C::R2);
  double* s_sqnS = reinterpret_cast<double*>(s_pos + NB);
  double* s_idS = s_sqnS + NB;
  double* s_rowg2 = s_idS + NB;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wr = warp / WC, wc = warp % WC;
  const int64_t tile_row0 = (int64_t)blockIdx.x * BM;
  const int m = p.m;
  const int kcur = p.kcur;
  const int nX = p.dchunks;
  const int nFk = (kcur + 15) >> 4;
  const int total1 = nX + nFk;

  for (int n = tid; n < NB; n += 256) {
    if (n < m) {
      const int ps = p.pos[n];
      s_pos[n] = ps;
      const double* rec = p.prop + (int64_t)ps * p.lay.rec;
      s_idS[n] = rec[0];
      s_sqnS[n] = rec[1];
    } else {
      s_pos[n] = -1;
      s_idS[n] = -1.0;
      s_sqnS[n] = 0.0;
    }
  }
  __syncthreads();

  // ---- tile loaders ------------------------------------------------------
  auto load_stage1 = [&](int stage, int kc) {
    unsigned char* As = r1 + stage * C::STAGE;
    unsigned char* Bs = As + C::A_BYTES;
    const bool isx = kc < nX;
    const int k0 = isx ? kc * 16 : (kc - nX) * 16;
    for (int i = tid; i < BM * 8; i += 256) {
      const int r = i >> 3, c16 = i & 7;
      const int64_t grow = tile_row0 + r;
      const void* src = p.X;
      int bytes = 0;
      if (grow < p.n_loc) {
        if (isx) {
          src = p.X + grow * p.ldx + k0 + 2 * c16;
          bytes = 16;
        } else {
          const int kk = k0 + 2 * c16;
          bytes = max(0, min(16, (kcur - kk) * 8));
          if (bytes) src = p.F + grow * p.ldf + kk;
        }
      }
      cp_async16(As + r * 128 + ((c16 ^ (r & 7)) << 4), src, bytes);
    }
    for (int i = tid; i < NB * 8; i += 256) {
      const int n = i >> 3, c16 = i & 7;
      const void* src = p.X;
      int bytes = 0;
      if (n < m) {
        const double* rec = p.prop + (int64_t)s_pos[n] * p.lay.rec;
        if (isx) {
          src = rec + p.lay.xoff + k0 + 2 * c16;
          bytes = 16;
        } else {
          const int kk = k0 + 2 * c16;
          bytes = max(0, min(16, (kcur - kk) * 8));
          if (bytes) src = rec + p.lay.foff + kk;
        }
      }
      cp_async16(Bs + n * 128 + ((c16 ^ (n & 7)) << 4), src, bytes);
    }
  };
  auto load_stage2 = [&](int stage, int kc) {
    unsigned char* Bs = r2 + stage * C::B_BYTES;
    for (int i = tid; i < NB * 8; i += 256) {
      const int n = i >> 3, c16 = i & 7;
      cp_async16(Bs + n * 128 + ((c16 ^ (n & 7)) << 4), p.linv + (int64_t)n * p.ldl + kc * 16 + 2 * c16,
                 16);
    }
  };

  double acc[2][NFW][2];
#pragma unroll
  for (int fr = 0; fr < 2; ++fr)
#pragma unroll
    for (int q = 0; q < NFW; ++q) acc[fr][q][0] = acc[fr][q][1] = 0.0;

  const int ra0 = wr * 16 + 2 * g;  // rows of A fragments: ra0 + fr

  auto mma_tile = [&](const unsigned char* As, uint32_t a_block_off, const unsigned char* Bs) {
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      double a[2];
#pragma unroll
      for (int fr = 0; fr < 2; ++fr) a[fr] = lds64(As, a_block_off + swz_off(ra0 + fr, 4 * s + t));
#pragma unroll
      for (int q = 0; q < NFW; ++q) {
        const int Q = wc * NFW + q;
        const double bv = lds64(Bs, swz_off(colmap(Q, g, NF), 4 * s + t));
#pragma unroll
        for (int fr = 0; fr < 2; ++fr) dmma884(acc[fr][q][0], acc[fr][q][1], a[fr], bv);
      }
    }
  };

  auto dist_tile = [&](const unsigned char* As, const unsigned char* Bs) {
    const bool l1 = p.kind == kL1;
#pragma unroll 2
    for (int j = 0; j < 16; ++j) {
      double xr[2];
#pragma unroll
      for (int fr = 0; fr < 2; ++fr) xr[fr] = lds64(As, swz_off(ra0 + fr, j));
#pragma unroll
      for (int q = 0; q < NFW; ++q) {
        const int Q = wc * NFW + q;
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          const double xs = lds64(Bs, swz_off(colmap(Q, 2 * t + v, NF), j));
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

  auto transform = [&]() {
    const double sig2 = __dmul_rn(p.sigma, p.sigma);
#pragma unroll
    for (int fr = 0; fr < 2; ++fr) {
      const int64_t grow = tile_row0 + ra0 + fr;
      const bool rin = grow < p.n_loc;
      const double sqr = rin ? p.sqn[grow] : 0.0;
      const double gid = (double)(p.row0 + grow);
#pragma unroll
      for (int q = 0; q < NFW; ++q) {
        const int Q = wc * NFW + q;
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          const int col = colmap(Q, 2 * t + v, NF);
          double val = 0.0;
          if (col < m && rin) {
            const double a = acc[fr][q][v];
            if (p.kind == kL1) {
              val = exp(__ddiv_rn(-a, p.sigma));
            } else {
              double dd = a;
              if (p.kind == kGaussGram) {
                dd = __dadd_rn(__dadd_rn(-2.0 * a, sqr), s_sqnS[col]);
                if (dd < 0.0) dd = 0.0;
                if (gid == s_idS[col]) dd = 0.0;
              }
              val = exp(__ddiv_rn(__dmul_rn(-0.5, dd), sig2));
            }
          }
          acc[fr][q][v] = -val;
        }
      }
    }
  };

  // ---- phase 1: kernel columns + residual GEMM ------------------------------
#pragma unroll 1
  for (int s = 0; s < C::S1 - 1; ++s) {
    if (s < total1) load_stage1(s, s);
    cp_async_commit();
  }
#pragma unroll 1
  for (int c = 0; c < total1; ++c) {
    cp_async_wait<C::S1 - 2>();
    __syncthreads();
    const int nxt = c + C::S1 - 1;
    if (nxt < total1) load_stage1(nxt % C::S1, nxt);
    cp_async_commit();
    const unsigned char* As = r1 + (c % C::S1) * C::STAGE;
    const unsigned char* Bs = As + C::A_BYTES;
    if (c >= nX || p.kind == kGaussGram) {
      mma_tile(As, 0u, Bs);
    } else {
      dist_tile(As, Bs);
    }
    if (c == nX - 1) transform();
  }
  cp_async_wait<0>();
  __syncthreads();

  double* fin = reinterpret_cast<double*>(r1);
  if (p.columns_only) {
    // standalone K5: A(R, S) = -acc, column-major output (KernelOracle::columns)
#pragma unroll
    for (int fr = 0; fr < 2; ++fr)
#pragma unroll
      for (int q = 0; q < NFW; ++q)
#pragma unroll
        for (int v = 0; v < 2; ++v)
          fin[(ra0 + fr) * C::FIN_LD + colmap(wc * NFW + q, 2 * t + v, NF)] = -acc[fr][q][v];
    __syncthreads();
    for (int idx = tid; idx < BM * m; idx += 256) {
      const int col = idx / BM, r = idx % BM;
      const int64_t grow = tile_row0 + r;
      if (grow < p.n_loc) p.cols_out[(int64_t)col * p.ld_out + grow] = fin[r * C::FIN_LD + col];
    }
    return;
  }

  // ---- phase 2: G <- G L^{-T} ------------------------------------------------
  unsigned char* gt = r1;  // NBK/16 swizzled [BM][16] blocks holding G = -acc
#pragma unroll
  for (int fr = 0; fr < 2; ++fr)
#pragma unroll
    for (int q = 0; q < NFW; ++q)
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const int col = colmap(wc * NFW + q, 2 * t + v, NF);
        *reinterpret_cast<double*>(gt + (col >> 4) * C::A_BYTES + swz_off(ra0 + fr, col & 15)) =
            -acc[fr][q][v];
        acc[fr][q][v] = 0.0;
      }
  if (NB != C::NBK) {  // zero the unused half of the last 16-column block
    for (int i = tid; i < BM * 8; i += 256) {
      const int r = i >> 3, k = 8 + (i & 7);
      *reinterpret_cast<double*>(gt + (NB >> 4) * C::A_BYTES + swz_off(r, k)) = 0.0;
    }
  }
  __syncthreads();
  const int nL = (m + 15) >> 4;
#pragma unroll 1
  for (int s = 0; s < C::S2 - 1; ++s) {
    if (s < nL) load_stage2(s, s);
    cp_async_commit();
  }
#pragma unroll 1
  for (int c = 0; c < nL; ++c) {
    cp_async_wait<C::S2 - 2>();
    __syncthreads();
    const int nxt = c + C::S2 - 1;
    if (nxt < nL) load_stage2(nxt % C::S2, nxt);
    cp_async_commit();
    mma_tile(gt, (uint32_t)(c * C::A_BYTES), r2 + (c % C::S2) * C::B_BYTES);
  }
  cp_async_wait<0>();
  __syncthreads();

  // ---- epilogue: append columns to F, update the residual diagonal ----------
#pragma unroll
  for (int fr = 0; fr < 2; ++fr)
#pragma unroll
    for (int q = 0; q < NFW; ++q)
#pragma unroll
      for (int v = 0; v < 2; ++v)
        fin[(ra0 + fr) * C::FIN_LD + colmap(wc * NFW + q, 2 * t + v, NF)] = acc[fr][q][v];
  __syncthreads();
  for (int r = warp; r < BM; r += 8) {
    const int64_t grow = tile_row0 + r;
    double s2 = 0.0;
    if (grow < p.n_loc) {
      double* frow = p.F + grow * p.ldf + kcur;
      for (int col = lane; col < m; col += 32) {
        const double v = fin[r * C::FIN_LD + col];
        frow[col] = v;
        s2 = fma(v, v, s2);
      }
      s2 = warp_sum_xor(s2);
      if (lane == 0) {
        const double un = __dsub_rn(p.u[grow], s2);
        p.u[grow] = un < 0.0 ? 0.0 : un;
      }
    }
    if (lane == 0) s_rowg2[r] = grow < p.n_loc ? s2 : 0.0;
  }
  __syncthreads();
  if (tid == 0) {
    double s = 0.0;
    for (int r = 0; r < BM; ++r) s = __dadd_rn(s, s_rowg2[r]);
    p.tile_g2[blockIdx.x] = s;
  }
}

template <int WC, int NFW>
static int launch_t(const UpdateParams& p, cudaStream_t st) {
  using C = UCfg<WC, NFW>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(update_kernel<WC, NFW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         C::SMEM);
    attr = true;
  }
  const unsigned grid = (unsigned)((p.n_loc + C::BM - 1) / C::BM);
  if (grid) update_kernel<WC, NFW><<<grid, 256, C::SMEM, st>>>(p);
  return C::BM;
}

int update_tile_rows(int m) {
  const int nf = (m + 7) / 8;
  if (nf <= 16) return 128;
  if (nf <= 32) return 64;
  return -1;
}

int launch_update(const UpdateParams& p, cudaStream_t st) {
  const int nf = std::max(1, (p.m + 7) / 8);
#define RPCB_CASE1(N) \
  case N:             \
    return launch_t<1, N>(p, st);
#define RPCB_CASE2(N) \
  case N:             \
    return launch_t<2, N>(p, st);
  if (nf <= 16) {
    switch (nf) {
      RPCB_CASE1(1) RPCB_CASE1(2) RPCB_CASE1(3) RPCB_CASE1(4) RPCB_CASE1(5) RPCB_CASE1(6)
      RPCB_CASE1(7) RPCB_CASE1(8) RPCB_CASE1(9) RPCB_CASE1(10) RPCB_CASE1(11) RPCB_CASE1(12)
      RPCB_CASE1(13) RPCB_CASE1(14) RPCB_CASE1(15) RPCB_CASE1(16)
    }
  } else if (nf <= 32) {
    switch ((nf + 1) / 2) {
      RPCB_CASE2(9) RPCB_CASE2(10) RPCB_CASE2(11) RPCB_CASE2(12) RPCB_CASE2(13)
      RPCB_CASE2(14) RPCB_CASE2(15) RPCB_CASE2(16)
    }
  }
#undef RPCB_CASE1
#undef RPCB_CASE2
  return -1;
}

}  // namespace rpcb
