#pragma once
#include <chrono>
#include <cstdio>
#include <cstdlib>
// update_impl.cuh — K5+K6: the fused round update, one CTA per BM-row tile of the shard.
//
// For the accepted pivots S (m columns) of a round it computes, without ever
// materialising the N x m kernel panel in HBM:
//   phase 0  A(R, S) kernel columns in registers (K5, fused), parked in its final
//            place F(R, kcur:kcur+m) (L2-resident)
//   phase 1  acc  = F(R, :kcur) B'^T,  B' = -L^{-1} F(S, :kcur)   (K6: FP64 DMMA GEMM)
//   phase 2  acc += A(R, S) L^{-T}: DMMA GEMM whose A operand is streamed back by TMA
//            so acc = A L^{-T} - F (L^{-1} F_S)^T = (A - F F_S^T) L^{-T}
//            (rpcholesky.hpp:378-384: residual GEMM + right_solve_lower_transposed)
//   epilogue F(R, kcur:kcur+m) = G ; u(R) = max(u - rowwise||G||^2, 0) ;
//            per-tile ||G||_F^2 partial                  (rpcholesky.hpp:385-388)
// Kernel columns (oracle.hpp:71-90, kernels.hpp:60-64): the Gaussian Gram term
// X(R,:) X(S,:)^T runs on the same DMMA pipeline as the residual GEMM (K = dpad),
// followed by the clamp / same-index pin / exp epilogue in registers; Gaussian-direct
// and l1 distances run on the FP64 CUDA cores from the same staged X tiles in
// ascending coordinate order (bit-identical distances to the reference's sums).
//
// Execution: persistent CTAs of 8 warps (two ping-pong groups of 4 for m <= 128) walk row
// tiles; [rows][16] fp64 tiles are streamed with 2D TMA (cp.async.bulk.tensor, 128B
// swizzle) into an S-stage ring per group guarded by full/empty mbarriers, issued round
// robin by lane 0 of the group's warps and running ahead across tile boundaries; all
// warps run mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4).  Operand rows are permuted inside 8-row
// groups (perm8, common.cuh) so every fragment load is bank-conflict free.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <mutex>
#include <type_traits>

#include "common.cuh"
#include "kernels.h"

namespace rpcb {

// G independent warp groups per CTA ("ping-pong"): each group of 8/G warps owns its
// own stage ring, barriers and tile sequence, so one group's non-DMMA work (exp
// transform, park, epilogue) overlaps the other group's DMMA main loop, while the
// CTA keeps the 255-register budget of 256 threads.
template <int WC, int NFW, int G>
struct UCfg {
  static constexpr int NT = 256;            // threads per CTA
  static constexpr int NCW = 8 / G;         // warps per group (thread 0 of a group issues TMA)
  static constexpr int GT = 32 * NCW;       // threads per group
  static constexpr int WR = NCW / WC;
  static constexpr int BM = 16 * WR;        // tile rows (per group tile)
  static constexpr int NF = WC * NFW;       // 8-column fragments
  static constexpr int NB = 8 * NF;         // tile columns (m padded)
  static constexpr int S = 4;               // pipeline stages
  static constexpr int A_BYTES = BM * 128;
  static constexpr int B_BYTES = NB * 128;
  static constexpr int STAGE = A_BYTES + B_BYTES;
  static constexpr int GMISC = WC * BM * 8 + BM * 8 + (2 * S) * 8;  // per group
  static constexpr int MISC = NB * 16 + 64 * 8 + G * GMISC;
  static constexpr int SMEM = G * S * STAGE + MISC + 1024;
};

// exp for the kernel-column epilogue: x = (64 n + j) ln2/64 + r with |r| <= ln2/128,
// exp(x) = 2^n * T[j] * (1 + expm1(r)), T[j] = 2^(j/64) from a shared-memory table,
// expm1 by a degree-5 polynomial (truncation < 4e-17 relative).  ~1 ulp; about half
// the FP64 work and dependency depth of a plain Cody-Waite + degree-13 Taylor.
__constant__ double kExpC[8] = {92.332482616893656,        // 64 / ln 2
                                -1.0830424696249145e-02,   // -ln2/64 (high)
                                -3.6235106466348430e-19,   // -ln2/64 (low)
                                8.3333333333333333e-03, 4.1666666666666667e-02,
                                1.6666666666666667e-01, 0.5, 0.0};

// No FP64<->int conversion instructions (slow paths on this part): k = rint(x 64/ln2)
// comes out of the low mantissa bits of x * 64/ln2 + 1.5 * 2^52 (one rounding, ties
// to even, exact for |k| < 2^51).
// The argument is clamped at -708 so every result is normal and 2^n is an exact integer
// add to the exponent field (no FP64 multiplies: the FP64 pipe is the one the DMMA main
// loop issues to).  Below -708 the value returned is exp(-708) = 3.3e-308 instead of a
// subnormal or zero, an absolute difference below 3.3e-308.
__device__ __forceinline__ double exp_tab(double x, const double* __restrict__ tab) {
  constexpr double kShift = 6755399441055744.0;  // 1.5 * 2^52
  // x <= 0 here: the clamp is an unsigned compare of the bit patterns (integer pipe)
  if ((unsigned long long)__double_as_longlong(x) > 0xC086200000000000ull) x = -708.0;
  const double ks = fma(x, kExpC[0], kShift);
  const int k = __double2loint(ks);
  const double kd = ks - kShift;
  double r = fma(kd, kExpC[1], x);
  r = fma(kd, kExpC[2], r);
  double q = fma(r, kExpC[3], kExpC[4]);
  q = fma(q, r, kExpC[5]);
  q = fma(q, r, kExpC[6]);
  q = fma(q * r, r, r);                                      // expm1(r)
  const double t = tab[k & 63];
  const double y = fma(t, q, t);
  return __hiloint2double(__double2hiint(y) + ((k >> 6) << 20), __double2loint(y));
}

// D := 0 where D < 0 (clamp) or where the row and column are the same point (pin),
// oracle.hpp:84-88; integer tests on the bit patterns (ids are non-negative integers held
// exactly in doubles; -0.0 maps to 0.0, which yields the same kernel value 1).
__device__ __forceinline__ double clamp_pin(double dd, double gid, double idc) {
  const bool neg = __double2hiint(dd) < 0;
  const bool pin = __double_as_longlong(gid) == __double_as_longlong(idc);
  return (neg || pin) ? 0.0 : dd;
}

// Kernel value from the distance term (KernelFun, kernels.hpp:60-79); s = host-computed scale.
__device__ __forceinline__ double kfun_eval(double dd, int f, double s, const double* tab) {
  if (f == kFunMatern32) {
    const double z = 1.7320508075688772 * (sqrt(dd) * s);
    return (1.0 + z) * exp_tab(-z, tab);
  }
  if (f == kFunMatern52) {
    const double rho2 = dd * s;
    const double z = sqrt(5.0 * rho2);
    return (1.0 + z + (5.0 / 3.0) * rho2) * exp_tab(-z, tab);
  }
  return exp_tab(dd * s, tab);
}

// f(integral_constant<J>) for J = 0 .. N-1 (compile-time indices into register arrays).
template <int N, int J = 0, class F>
__device__ __forceinline__ void static_for_asc(F&& f) {
  if constexpr (J < N) {
    f(std::integral_constant<int, J>{});
    static_for_asc<N, J + 1>(f);
  }
}

// f(integral_constant<J>) for J = N-1 down to 0 (compile-time indices into register arrays).
template <int J, class F>
__device__ __forceinline__ void static_for_desc(F&& f) {
  if constexpr (J >= 0) {
    f(std::integral_constant<int, J>{});
    static_for_desc<J - 1>(f);
  }
}

// COLS: compiled for the standalone K5 only (p.columns_only): phases 1-2, the park and the
// epilogue are compiled out, so registers go to more resident CTAs instead.
template <int WC, int NFW, bool GRAM, int MINB, int G, bool COLS = false>
__global__ void __launch_bounds__(UCfg<WC, NFW, G>::NT, MINB)
    update_kernel(UpdateParams p, const __grid_constant__ CUtensorMap tmX,
                  const __grid_constant__ CUtensorMap tmXS, const __grid_constant__ CUtensorMap tmF,
                  const __grid_constant__ CUtensorMap tmFS, const __grid_constant__ CUtensorMap tmG,
                  const __grid_constant__ CUtensorMap tmL) {
  using C = UCfg<WC, NFW, G>;
  constexpr int BM = C::BM, S = C::S, NCW = C::NCW, GT = C::GT;
  // REGP2 (one warp column, m <= 128): A(R,S) L^{-T} is formed in place from the registers
  // that hold A(R,S) after the transform (no park in F, no phase-2 reload): chunk J of the
  // triangular product only feeds output columns >= 16 J, so walking J downwards lets every
  // chunk read its operand columns before they are overwritten by output columns.
  constexpr bool REGP2 = (WC == 1) && !COLS;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  // 1024-byte aligned ring (128B-swizzle atoms).  Offsets stay relative to the
  // __shared__ array so every fragment load is an LDS with an immediate offset.
  const uint32_t align = (1024u - (smem_u32(smem_raw) & 1023u)) & 1023u;
  const int tid = threadIdx.x, lane = tid & 31;
  const int grp = (tid >> 5) / NCW;          // warp group
  const int warp = (tid >> 5) % NCW;         // warp within the group
  const int gtid = tid % GT;                 // thread within the group
  unsigned char* stages = smem_raw + align + grp * S * C::STAGE;
  double* s_sqnS = reinterpret_cast<double*>(smem_raw + align + G * S * C::STAGE);
  double* s_idS = s_sqnS + C::NB;
  double* s_exp2 = s_idS + C::NB;  // 2^(j/64), j = 0..63
  unsigned char* gmisc = reinterpret_cast<unsigned char*>(s_exp2 + 64) + grp * C::GMISC;
  double* s_rown = reinterpret_cast<double*>(gmisc);  // [WC][BM]
  double* s_rowg2 = s_rown + WC * BM;
  uint64_t* full = reinterpret_cast<uint64_t*>(s_rowg2 + BM);
  uint64_t* empty = full + S;
  auto gsync = [&]() { named_bar_sync(1 + grp, GT); };
  __shared__ volatile int s_go;  // ping-pong stagger: group 1 starts once group 0 passed its first exp

  const int m = p.m, kcur = p.kcur;
  const int nX = p.dchunks;
  const int nFk = (COLS || (REGP2 && p.cext)) ? 0 : (kcur + 15) >> 4;
  // Phase-2 A tiles start at F column kcur - koff: TMA box starts must be 16-byte
  // aligned in the inner dimension, so for odd kcur one extra leading column is
  // loaded and multiplied by the zero column 0 of the shifted L^{-1} (koff = 1).
  const int koff = kcur & 1;
  const int nL = (COLS || p.columns_only) ? 0 : REGP2 ? (m + 15) >> 4 : (m + koff + 15) >> 4;
  // REGP2 with a tensor-core residual (p.cext): C's 16-column chunks stream through the ring's
  // A slots in place of the F chunks (TMA, tmG re-pointed at C), so the add is prefetched
  const int nCk = (REGP2 && p.cext) ? (m + 15) >> 4 : 0;
  const int T = nX + nFk + nL + nCk;         // chunks per tile
  const int ntiles = (int)((p.n_loc + BM - 1) / BM);
  const int vb = (int)blockIdx.x * G + grp, vgrid = (int)gridDim.x * G;  // virtual block per group
  const int my_tiles = vb < ntiles ? (ntiles - 1 - vb) / vgrid + 1 : 0;
  const int total = my_tiles * T;            // chunks this group consumes (persistent)

  if (gtid == 0) {
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
  if (tid < 64) s_exp2[tid] = exp2((double)tid / 64.0);
  if (tid == 0) s_go = (G == 1);
  __syncthreads();

  // ---- producers: lane 0 of every warp of the group, round robin: warp w issues chunks
  // w, w + NCW, ...; chunk i goes out once the issuing warp has consumed chunk i - S + 1
  // (the stage's previous occupant, chunk i - S, was released a chunk earlier, so the
  // empty-barrier wait rarely blocks) and, for phase-2 chunks of tile k, once that tile's
  // G is parked (parked > k).  Spreading the TMA issue (~0.4k cycles per chunk) over the
  // warps keeps it off any single warp's critical path.
  // (the standalone K5, COLS, keeps one producer, thread 0, and the full ring lookahead:
  // its tiles are two chunks long and measured faster that way)
  constexpr int PSTEP = COLS ? 1 : NCW;
  int issued = COLS ? 0 : warp;  // next chunk this producer issues
  int parked = 0;      // tiles whose G has been parked (CTA-uniform)
  auto pump = [&](int done) {
    if (COLS ? gtid != 0 : lane != 0) return;
    while (issued < total && issued < done + (COLS ? S : S - 1)) {
      const int k = issued / T, c = issued - k * T;
      if (!REGP2 && c >= nX + nFk && parked <= k) break;
      const int s = issued % S;
      if (issued >= S) mbar_wait(&empty[s], ((issued / S) & 1) ^ 1);
      unsigned char* As = stages + s * C::STAGE;
      unsigned char* Bs = As + C::A_BYTES;
      const int r0 = (int)((vb + (int64_t)k * vgrid) * BM);
      const bool l_only = REGP2 && c >= nX && c < nX + nL;  // phase 2: the L^{-1} chunk only
      const bool c_only = REGP2 && nCk > 0 && c >= nX + nL;   // tensor-core residual chunk
      mbar_arrive_expect_tx(&full[s], l_only ? C::B_BYTES : c_only ? C::A_BYTES : C::STAGE);
      if (c_only) {
        tma_load_2d(As, &tmG, 16 * (c - nX - nL), r0, &full[s]);
      } else if (c < nX) {
        tma_load_2d(As, &tmX, 16 * c, r0, &full[s]);
        tma_load_2d(Bs, &tmXS, 16 * c, 0, &full[s]);
      } else if (l_only) {  // chunks J = nL-1 .. 0 (descending, see REGP2)
        tma_load_2d(Bs, &tmL, 16 * (nL - 1 - (c - nX)), 0, &full[s]);
      } else if (REGP2) {
        tma_load_2d(As, &tmF, 16 * (c - nX - nL), r0, &full[s]);
        tma_load_2d(Bs, &tmFS, 16 * (c - nX - nL), 0, &full[s]);
      } else if (c < nX + nFk) {
        tma_load_2d(As, &tmF, 16 * (c - nX), r0, &full[s]);
        tma_load_2d(Bs, &tmFS, 16 * (c - nX), 0, &full[s]);
      } else {
        tma_load_2d(As, &tmG, kcur - koff + 16 * (c - nX - nFk), r0, &full[s]);
        tma_load_2d(Bs, &tmL, 16 * (c - nX - nFk), 0, &full[s]);
      }
      issued += PSTEP;
    }
  };
  if (G > 1 && grp == 1) {  // offset group 1 so the two groups' non-DMMA phases interleave
    if (gtid == 0)
      while (!s_go) __nanosleep(200);
    named_bar_sync(1 + grp, GT);
  }
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
  // Two warp columns own interleaved fragments (global fragment q * WC + wc), so the skipped
  // upper triangle of L^{-T} in phase 2 is shared evenly between them.
  const uint32_t b_base = (uint32_t)wc * 1024u;

  double acc[2][NFW][2];

  // q_lo: first fragment that can be non-zero (phase 2 skips the zero upper triangle
  // of L^{-T}; phase 1 passes 0).
  // ks: k steps of the chunk that hold data (the Gram chunks skip steps made only of the
  // zero padding of X beyond d; the residual GEMM always passes 4)
  auto mma_stage = [&](uint32_t st_off, int q_lo, int ks) {
    const unsigned char* Aw = stages + st_off + a_base;
    const unsigned char* Bw = stages + st_off + C::A_BYTES + b_base;
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      if (s >= ks) break;
      double a[2];
#pragma unroll
      for (int fr = 0; fr < 2; ++fr) a[fr] = *reinterpret_cast<const double*>(Aw + fr * 1024 + foff[s]);
#pragma unroll
      for (int q = 0; q < NFW; ++q) {
        if (q < q_lo) continue;
        const double bv = *reinterpret_cast<const double*>(Bw + q * WC * 1024 + foff[s]);
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
    // fragment pairs (q, q+1), skipped whole below q_lo rounded down to even (at most one
    // all-zero fragment computed): four independent accumulators per branch block
#pragma unroll
    for (int q = 0; q < NFW; q += 2) {
      if (q + 1 < q_lo) continue;
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        const double bv0 = *reinterpret_cast<const double*>(Bw + q * WC * 1024 + foff[s]);
        double bv1 = 0.0;
        if (q + 1 < NFW) bv1 = *reinterpret_cast<const double*>(Bw + (q + 1) * WC * 1024 + foff[s]);
#pragma unroll
        for (int fr = 0; fr < 2; ++fr) {
          dmma884(acc[fr][q][0], acc[fr][q][1], a[s][fr], bv0);
          if (q + 1 < NFW) dmma884(acc[fr][q + 1][0], acc[fr][q + 1][1], a[s][fr], bv1);
        }
      }
    }
  };

  // c: the 16-coordinate chunk; its zero-padded coordinates (>= d) are skipped (they would
  // add exact zeros)
  auto dist_stage = [&](uint32_t st_off, int c) {
    const unsigned char* As = stages + st_off;
    const unsigned char* Bs = As + C::A_BYTES;
    const bool l1 = p.kind == kL1;
    const int jn = min(16, p.d - 16 * c);
#pragma unroll 1
    for (int j = 0; j < jn; ++j) {
      double xr[2];
#pragma unroll
      for (int fr = 0; fr < 2; ++fr) xr[fr] = *reinterpret_cast<const double*>(As + swz_off(arow[fr], j));
#pragma unroll
      for (int q = 0; q < NFW; ++q) {
        const int Q = q * WC + wc;
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

  // Optional phase timing (warp 0 lane 0 clocks; debug only).
  unsigned long long tclk = clock64();
  auto mark = [&](int ph) {
    if (p.phase_clk && tid == 0) {
      const unsigned long long now = clock64();
      p.phase_clk[(size_t)blockIdx.x * 8 + ph] += now - tclk;
      tclk = now;
    }
  };
  // RPC_DEBUG_TRACE: CTA 0 per-group, per-tile phase clocks
  auto trc = [&](int k, int ph) {
    if (p.trace && blockIdx.x == 0 && gtid == 0 && k < 64) p.trace[(grp * 64 + k) * 8 + ph] = clock64();
  };
  int cons = 0;  // chunks consumed by this warp so far (CTA-uniform in practice)
  // next_ready: the next stage's data was seen complete during the previous body (probed
  // with a non-blocking test right after that body's loads were issued), so its wait is skipped
  bool next_ready = false;
  auto consume = [&](auto&& body) {
    const int s = cons % S;
    if (!next_ready) mbar_wait(&full[s], (cons / S) & 1);
    __syncwarp();
    body((uint32_t)(s * C::STAGE));
    next_ready = mbar_test_wait(&full[(cons + 1) % S], ((cons + 1) / S) & 1);
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    ++cons;
    if (!COLS || warp == 0) pump(cons);
  };

#pragma unroll 1
  for (int k = 0; k < my_tiles; ++k) {
    const int tile = vb + k * vgrid;
    const int64_t tile_row0 = (int64_t)tile * BM;
    trc(k, 0);
#pragma unroll
    for (int fr = 0; fr < 2; ++fr)
#pragma unroll
      for (int q = 0; q < NFW; ++q) acc[fr][q][0] = acc[fr][q][1] = 0.0;

    // ---- phase 1a: kernel-column distances / Gram products (X tiles) -------------
#pragma unroll 1
    for (int c = 0; c < nX; ++c) {
      if constexpr (GRAM) {
        const int ks = min(4, (min(16, p.d - 16 * c) + 3) / 4);
        consume([&](uint32_t so) { mma_stage(so, 0, ks); });
      }
      else consume([&](uint32_t so) { dist_stage(so, c); });
    }
    mark(0);
    trc(k, 1);
    if (p.phase_clk) {  // debug: wait for every outstanding DMMA before timing the transform
      double s = 0.0;
#pragma unroll
      for (int fr = 0; fr < 2; ++fr)
#pragma unroll
        for (int q = 0; q < NFW; ++q) s += acc[fr][q][0] + acc[fr][q][1];
      if (s == 1.2345e300) p.phase_clk[0] = 1;
      mark(6);
    }
    // ---- acc (Gram dot / distance) -> -A(R, S) ------------------------------------
    // Rolled over the warp's column fragments: each pass transforms fragments 0 and 1 and
    // rotates the accumulator array by two fragments, so the code stays small while acc
    // never leaves registers.
    {
      // exponent = D * (-0.5 / sigma^2) (Gaussian) or D * (-1 / sigma) (l1): one multiply
      // instead of the reference's division, <= 1 ulp apart (kernel values agree to 1e-15).
      const double escale = p.escale;
      double sqr[2], gid[2];
      bool rin[2];
#pragma unroll
      for (int fr = 0; fr < 2; ++fr) {
        const int64_t grow = tile_row0 + arow[fr];
        rin[fr] = grow < p.n_loc;
        sqr[fr] = rin[fr] ? p.sqn[grow] : 0.0;
        gid[fr] = (double)(p.row0 + grow);
      }
      mark(7);
      // two fragments per pass (8 independent exp chains in flight), rotating by two
      auto xform = [&](double& a, int col, int fr, double sqc, double idc) {
        double dd = a;
        if (GRAM) {
          // dd = -2 x.y already (operand X(S,:) pre-scaled by -2, gram_xscale)
          dd = __dadd_rn(__dadd_rn(dd, sqr[fr]), sqc);
          dd = clamp_pin(dd, gid[fr], idc);
        }
        const double val = kfun_eval(dd, p.kfun, escale, s_exp2);
        a = (col < m && rin[fr]) ? (REGP2 ? val : -val) : 0.0;
      };
#pragma unroll 1
      for (int it = 0; it + 1 < NFW; it += 2) {
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int v = 0; v < 2; ++v) {
            const int col = 8 * ((it + h) * WC + wc) + 2 * t + v;
            const double sqc = s_sqnS[col], idc = s_idS[col];
#pragma unroll
            for (int fr = 0; fr < 2; ++fr) xform(acc[fr][h][v], col, fr, sqc, idc);
          }
#pragma unroll
        for (int fr = 0; fr < 2; ++fr) {
          const double t0 = acc[fr][0][0], t1 = acc[fr][0][1];
          const double t2 = acc[fr][NFW > 1 ? 1 : 0][0], t3 = acc[fr][NFW > 1 ? 1 : 0][1];
#pragma unroll
          for (int q = 0; q + 2 < NFW; ++q) {
            acc[fr][q][0] = acc[fr][q + 2][0];
            acc[fr][q][1] = acc[fr][q + 2][1];
          }
          if (NFW > 1) {
            acc[fr][NFW - 2][0] = t0;
            acc[fr][NFW - 2][1] = t1;
            acc[fr][NFW - 1][0] = t2;
            acc[fr][NFW - 1][1] = t3;
          }
        }
      }
      if (NFW & 1) {  // last fragment (now at position 0), then rotate by one
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          const int col = 8 * ((NFW - 1) * WC + wc) + 2 * t + v;
          const double sqc = s_sqnS[col], idc = s_idS[col];
#pragma unroll
          for (int fr = 0; fr < 2; ++fr) xform(acc[fr][0][v], col, fr, sqc, idc);
        }
#pragma unroll
        for (int fr = 0; fr < 2; ++fr) {
          const double t0 = acc[fr][0][0], t1 = acc[fr][0][1];
#pragma unroll
          for (int q = 0; q + 1 < NFW; ++q) {
            acc[fr][q][0] = acc[fr][q + 1][0];
            acc[fr][q][1] = acc[fr][q + 1][1];
          }
          acc[fr][NFW - 1][0] = t0;
          acc[fr][NFW - 1][1] = t1;
        }
      }
    }
    if (G > 1 && grp == 0 && k == 0 && gtid == 0) s_go = 1;
    mark(1);
    trc(k, 2);
    if (COLS || p.columns_only) {  // standalone K5: A(R, S) -> column-major output
#pragma unroll
      for (int fr = 0; fr < 2; ++fr) {
        const int64_t grow = tile_row0 + arow[fr];
        if (grow >= p.n_loc) continue;
#pragma unroll
        for (int q = 0; q < NFW; ++q)
#pragma unroll
          for (int v = 0; v < 2; ++v) {
            const int col = 8 * (q * WC + wc) + 2 * t + v;
            if (col < m) p.cols_out[(int64_t)col * p.ld_out + grow] = -acc[fr][q][v];
          }
      }
      continue;
    }

    if constexpr (REGP2) {
      // every warp of the group passes here before the group's next epilogue (s_rowg2)
      gsync();
      mark(2);
      trc(k, 3);
      // ---- phase 2 first, in place: acc = A(R, S) L^{-T} ---------------------------
      // Chunk J holds L^{-1}(:, 16J..16J+15) in kslot16 order, i.e. k step s of lane t is
      // column 16J + 8(s>>1) + 2t + (s&1): exactly the accumulator element
      // acc[fr][2J + (s>>1)][s&1] this lane holds, so the A operand needs no data movement.
      static_for_desc<(NFW + 1) / 2 - 1>([&](auto JC) {
        constexpr int J = decltype(JC)::value;
        constexpr int q0 = 2 * J, q1 = 2 * J + 1;
        if (J >= nL) return;
        consume([&](uint32_t so) {
          const unsigned char* Bw = stages + so + C::A_BYTES;
          double a[4][2];
#pragma unroll
          for (int fr = 0; fr < 2; ++fr) {
            a[0][fr] = acc[fr][q0][0];
            a[1][fr] = acc[fr][q0][1];
            acc[fr][q0][0] = acc[fr][q0][1] = 0.0;
            if constexpr (q1 < NFW) {
              a[2][fr] = acc[fr][q1][0];
              a[3][fr] = acc[fr][q1][1];
              acc[fr][q1][0] = acc[fr][q1][1] = 0.0;
            } else {
              a[2][fr] = a[3][fr] = 0.0;
            }
          }
#pragma unroll
          for (int q = q0; q < NFW; ++q)
#pragma unroll
            for (int s = 0; s < 4; ++s) {
              if (q1 >= NFW && s >= 2) continue;
              const double bv = *reinterpret_cast<const double*>(Bw + q * 1024 + foff[s]);
#pragma unroll
              for (int fr = 0; fr < 2; ++fr) dmma884(acc[fr][q][0], acc[fr][q][1], a[s][fr], bv);
            }
        });
      });
      mark(4);
      trc(k, 4);
      // ---- phase 1: acc += F(R,:) B'^T with B' = -L^{-1} F(S,:)  (K = kcur) ----------
#pragma unroll 1
      for (int c = 0; c + 1 < nFk; ++c) consume([&](uint32_t so) { mma_stage(so, 0, 4); });
      if (nFk > 0) {
        const int ks = (kcur - 16 * (nFk - 1) + 3) / 4;
        consume([&](uint32_t so) { mma_stage(so, 0, ks); });
      }
      // F B'^T from the tensor-core residual launch (i8gemm.cu): chunk J of C holds columns
      // 16 J .. 16 J + 15, i.e. this lane's fragments 2 J and 2 J + 1
      static_for_asc<(NFW + 1) / 2>([&](auto JC) {
        constexpr int J = decltype(JC)::value;
        if (J >= nCk) return;
        consume([&](uint32_t so) {
          const unsigned char* Aw = stages + so;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            if (2 * J + h >= NFW) continue;
#pragma unroll
            for (int fr = 0; fr < 2; ++fr)
#pragma unroll
              for (int v = 0; v < 2; ++v)
                acc[fr][2 * J + h][v] +=
                    *reinterpret_cast<const double*>(Aw + swz_off(arow[fr], 8 * h + 2 * t + v));
          }
        });
      });
      mark(3);
      trc(k, 5);
    } else {
    // ---- park A(R, S) in F(R, kcur:kcur+m): phase 2 streams it back as the A operand
    // of A L^{-T}.  Parking right after the transform lets the TMA round trip hide
    // behind the residual GEMM instead of stalling the end of the tile.
#pragma unroll
    for (int fr = 0; fr < 2; ++fr) {
      const int64_t grow = tile_row0 + arow[fr];
      double* frow = p.F + grow * p.ldf + kcur;
#pragma unroll
      for (int q = 0; q < NFW; ++q)
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          const int col = 8 * (q * WC + wc) + 2 * t + v;
          if (col < m && grow < p.n_loc) frow[col] = -acc[fr][q][v];
          acc[fr][q][v] = 0.0;
        }
    }
    fence_proxy_async_global();
    gsync();
    parked = k + 1;
    if (!COLS || warp == 0) pump(cons);
    mark(2);
    trc(k, 3);
    // ---- phase 1b: acc = F(R,:) B'^T with B' = -L^{-1} F(S,:)  (K = kcur) -------------
    //   G L^{-T} = (A - F F_S^T) L^{-T} = A L^{-T} + F (-L^{-1} F_S)^T
#pragma unroll 1
    for (int c = 0; c + 1 < nFk; ++c) consume([&](uint32_t so) { mma_stage(so, 0, 4); });
    if (nFk > 0) {  // last chunk: only the k steps below kcur hold data (TMA zero fill above)
      const int ks = (kcur - 16 * (nFk - 1) + 3) / 4;
      consume([&](uint32_t so) { mma_stage(so, 0, ks); });
    }

    mark(3);
    trc(k, 4);
    // ---- phase 2: acc += A L^{-T}  (K = m, A streamed back from F) --------------------
#pragma unroll 1
    for (int j = 0; j < nL; ++j) {
      // chunk j covers A columns [16j - koff, 16j + 16 - koff); L^{-T}[k][n] = 0 for n < k,
      // so fragments whose 8 columns all lie below 16j - koff contribute nothing.
      const int q_lo = max(0, ((16 * j - koff) / 8 - wc + WC - 1) / WC);
      consume([&](uint32_t so) { mma_stage_tri(so, q_lo); });
    }

    mark(4);
    trc(k, 5);
    }  // !REGP2
    // ---- epilogue ------------------------------------------------------------------
    double rs[2] = {0.0, 0.0};
    double unew[2] = {0.0, 0.0};  // new u of this lane's rows (t == 0 lanes; 0 past n_loc)
#pragma unroll
    for (int fr = 0; fr < 2; ++fr) {
      const int64_t grow = tile_row0 + arow[fr];
      const bool rin = grow < p.n_loc;
      double* frow = p.F + grow * p.ldf + kcur;
#pragma unroll
      for (int q = 0; q < NFW; ++q)
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          const int col = 8 * (q * WC + wc) + 2 * t + v;
          if (col < m && rin) {
            const double val = acc[fr][q][v];
            frow[col] = val;
            rs[fr] = fma(val, val, rs[fr]);
          }
        }
      rs[fr] += __shfl_xor_sync(0xffffffffu, rs[fr], 1);
      rs[fr] += __shfl_xor_sync(0xffffffffu, rs[fr], 2);
      if (WC == 1) {  // the quad's t == 0 lane holds the whole row: update u directly
        if (t == 0) {
          double s2 = rs[fr];
          if (rin) {
            const double un = __dsub_rn(p.u[grow], s2);
            unew[fr] = un < 0.0 ? 0.0 : un;
            p.u[grow] = unew[fr];
          } else {
            s2 = 0.0;
          }
          s_rowg2[arow[fr]] = s2;
        }
      } else if (t == 0) {
        s_rown[wc * BM + arow[fr]] = rs[fr];
      }
    }
    if (WC == 1 && !COLS && p.tsum) {
      // sequential sum of the warp's 16 rows in row order (row 8 fr + r sits in quad g with
      // perm8(g) == r): the per-thread sum of chunk_scan_core, zero past n_loc
      double ssum = 0.0;
#pragma unroll
      for (int fr = 0; fr < 2; ++fr)
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          const int gq = (r & 1) ? 4 + (r >> 1) : (r >> 1);  // perm8(gq) == r
          ssum = __dadd_rn(ssum, __shfl_sync(0xffffffffu, unew[fr], 4 * gq));
        }
      if (lane == 0) p.tsum[(tile_row0 >> 4) + wr] = ssum;
    }
    if (WC > 1) {
      gsync();
      if (gtid < BM) {
        const int64_t grow = tile_row0 + gtid;
        double s2 = 0.0;
#pragma unroll
        for (int w = 0; w < WC; ++w) s2 = __dadd_rn(s2, s_rown[w * BM + gtid]);
        if (grow < p.n_loc) {
          const double un = __dsub_rn(p.u[grow], s2);
          p.u[grow] = un < 0.0 ? 0.0 : un;
        } else {
          s2 = 0.0;
        }
        s_rowg2[gtid] = s2;
      }
    }
    // only the summing warp waits for the row partials; the others go on to the next tile
    // (s_rowg2 is next written after the next tile's park barrier).  A barrier id of its own
    // (not gsync's): the early warps' arrivals can then never be counted toward a later
    // gsync, and the next tile's epilogue arrivals come after warp 0 passed that tile's park.
    // (the tile's ||G||^2 is a fixed-order tree over the row sums — each lane adds rows
    // lane and lane + 32, then the xor butterfly, which every lane evaluates identically —
    // instead of a 64-long serial chain that kept warp 0, and through the ring the group,
    // waiting at every tile: 5.4k-cycle epilogues in the early rounds)
    if (warp == 0) {
      named_bar_sync(1 + G + grp, GT);
      double s2 = 0.0;
      for (int r = lane; r < BM; r += 32) s2 = __dadd_rn(s2, s_rowg2[r]);
      s2 = warp_sum_xor(s2);
      if (lane == 0) p.tile_g2[tile] = p.g2_accum ? __dadd_rn(p.tile_g2[tile], s2) : s2;

    } else {
      named_bar_arrive(1 + G + grp, GT);
    }
    mark(5);
    trc(k, 6);
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

template <int WC, int NFW, bool GRAM, int MINB, int G, bool COLS = false>
int launch_t(const UpdateParams& p, cudaStream_t st) {
  using C = UCfg<WC, NFW, G>;
  const void* kfn = (const void*)update_kernel<WC, NFW, GRAM, MINB, G, COLS>;
  static const bool dbg_launch = std::getenv("RPC_DEBUG_LAUNCH") != nullptr;
  const auto t0 = std::chrono::steady_clock::now();
  if (ensure_smem_attr(kfn, C::SMEM) != cudaSuccess) return -2;
  const auto t1 = std::chrono::steady_clock::now();
  CUtensorMap mX, mXS, mF, mFS, mG, mL;
  bool ok = make_map(&mX, p.X, p.dpad, p.n_loc, p.dpad, C::BM) &&
            make_map(&mXS, p.xs, p.dpad, C::NB, p.dpad, C::NB) &&
            make_map(&mF, p.F, p.kcur, p.n_loc, p.ldf, C::BM) &&
            make_map(&mFS, p.fs, p.kcur, C::NB, p.ldfs, C::NB) &&
            ((WC == 1 && !COLS && p.cext)  // tmG: C (tensor-core residual) when present
                 ? make_map(&mG, p.cext, p.ldce, p.n_loc, p.ldce, C::BM)
                 : make_map(&mG, p.F, p.kcur + p.m, p.n_loc, p.ldf, C::BM)) &&
            make_map(&mL, p.linv, p.ldl, C::NB, p.ldl, C::NB);
  if (!ok) return -3;
  const auto t2 = std::chrono::steady_clock::now();
  // persistent: one CTA per SM, tiles strided by the grid (p.tile_g2 is per tile)
  const int64_t ntiles = (p.n_loc + C::BM - 1) / C::BM;
  // persistent grid sized by occupancy: small m (early rounds, kernel-column bench) fits two
  // CTAs per SM, which hides the latency of the short per-tile chains
  const int occ = cached_occupancy(kfn, C::NT, C::SMEM, MINB);
  const unsigned grid = (unsigned)std::min<int64_t>((ntiles + G - 1) / G, (int64_t)occ * num_sms());
  const auto t3 = std::chrono::steady_clock::now();
  if (grid)
    update_kernel<WC, NFW, GRAM, MINB, G, COLS><<<grid, C::NT, C::SMEM, st>>>(p, mX, mXS, mF, mFS, mG, mL);
  if (dbg_launch) {
    const auto t4 = std::chrono::steady_clock::now();
    auto us = [](auto a, auto b) { return std::chrono::duration<double, std::micro>(b - a).count(); };
    std::fprintf(stderr, "[launch] attr %.2f maps %.2f occ %.2f launch %.2f us\n", us(t0, t1),
                 us(t1, t2), us(t2, t3), us(t3, t4));
  }
  return C::BM;
}

}  // namespace rpcb
