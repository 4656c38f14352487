#pragma once
// lowmem_impl.cuh — the round update of the low-memory variant
// (accelerated_rpcholesky_lowmem, rpcholesky.hpp:408-485), one fused kernel.
//
// The reference keeps O(N + k^2) state and, per round, regenerates the kernel block
// A(R, S_all) for every row chunk R, triangular-solves it against L and forms
//   g = (A(R, S_new) - (L^{-1} A(S_old, R))^T W_acc) L_sel^{-T},  u(R) -= rowsq(g)
// (rpcholesky.hpp:454-468).  With the new pivot block's inverse kept explicitly
// (Linv, lower triangular) that is one product
//   g = A(R, S_all) W^T,   W = rows [kold, kold+m) of L_new^{-1}
//     = [ -L_sel^{-1} F_S L_old^{-1} | L_sel^{-1} ]          (m x knew),
// so the per-row cost drops from the reference's k_old^2 (solve) to 2 k m (GEMM).
//
// Execution (B200): persistent CTAs walk 64-row tiles.  The tile's points X(R, :)
// stay resident in shared memory; the pivot axis is streamed in 16-column chunks:
// thread 0 of each warp group TMA-loads, per chunk, the 16 pivot points X(S_c, :)
// and the W chunk [m][16] into an S-stage ring (full/empty mbarriers).  The warps
// regenerate the 64 x 16 kernel tile in shared memory — Gaussian Gram products on
// the FP64 tensor cores (DMMA 8x8x4) + clamp / same-index pin / exp, or direct and
// l1 distances on the FP64 CUDA cores in ascending coordinate order — and feed it
// straight into the DMMA GEMM with the W chunk.  The kernel block never reaches
// HBM; the only N-sized traffic is X (read once per round) and u (read + write).
#include "update_impl.cuh"

namespace rpcb {

template <int WC, int NFW, int G>
struct LCfg {
  static constexpr int NT = 256;
  static constexpr int NCW = 8 / G;        // warps per group
  static constexpr int GT = 32 * NCW;
  static constexpr int WR = NCW / WC;
  static constexpr int BM = 16 * WR;       // 64
  static constexpr int NF = WC * NFW;
  static constexpr int NB = 8 * NF;        // W rows (m padded)
  static constexpr int NG = 2 / WC;        // 8-column generator fragments per warp
  static constexpr int A_BYTES = BM * 128;
  static constexpr int B_BYTES = NB * 128;
  static constexpr int GMISC = WC * BM * 8 + BM * 8 + 16 * 8;
  static constexpr int kMaxStages = 4;
  // per-group bytes for S stages and dchunks 16-coordinate slices
  static constexpr int stage_bytes(int dch) { return A_BYTES + B_BYTES + dch * 2048; }
  static constexpr int group_bytes(int S, int dch) { return S * stage_bytes(dch) + dch * A_BYTES; }
  static constexpr int smem_bytes(int S, int dch) {
    return G * group_bytes(S, dch) + 64 * 8 + G * GMISC + 1024;
  }
};

template <int WC, int NFW, bool GRAM, int G, int MINB>
__global__ void __launch_bounds__(256, MINB)
    lowmem_kernel(LowmemParams p, int S, const __grid_constant__ CUtensorMap tmX,
                  const __grid_constant__ CUtensorMap tmXS, const __grid_constant__ CUtensorMap tmW) {
  using C = LCfg<WC, NFW, G>;
  constexpr int BM = C::BM, NCW = C::NCW, GT = C::GT, NG = C::NG;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const uint32_t align = (1024u - (smem_u32(smem_raw) & 1023u)) & 1023u;
  const int tid = threadIdx.x, lane = tid & 31;
  const int grp = (tid >> 5) / NCW, warp = (tid >> 5) % NCW, gtid = tid % GT;
  const int nD = p.dchunks;
  const int STAGE = C::stage_bytes(nD);
  unsigned char* gbase = smem_raw + align + grp * C::group_bytes(S, nD);
  unsigned char* stages = gbase;
  unsigned char* xt = gbase + S * STAGE;  // resident X(R, :) tile, nD slices [BM][16]
  double* s_exp2 = reinterpret_cast<double*>(smem_raw + align + G * C::group_bytes(S, nD));
  unsigned char* gmisc = reinterpret_cast<unsigned char*>(s_exp2 + 64) + grp * C::GMISC;
  double* s_rown = reinterpret_cast<double*>(gmisc);  // [WC][BM]
  double* s_rowg2 = s_rown + WC * BM;
  uint64_t* full = reinterpret_cast<uint64_t*>(s_rowg2 + BM);
  uint64_t* empty = full + C::kMaxStages;
  uint64_t* xbar = empty + C::kMaxStages;
  auto gsync = [&]() { named_bar_sync(1 + grp, GT); };

  const int knew = p.knew, kold = p.kold;
  const int nK = (knew + 15) >> 4;
  const int ntiles = (int)((p.n_loc + BM - 1) / BM);
  const int vb = (int)blockIdx.x * G + grp, vgrid = (int)gridDim.x * G;
  const int my_tiles = vb < ntiles ? (ntiles - 1 - vb) / vgrid + 1 : 0;
  const int total = my_tiles * nK;

  if (gtid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCW);
    }
    mbar_init(xbar, 1);
    mbar_fence_init();
    tma_prefetch_desc(&tmX);
    tma_prefetch_desc(&tmXS);
    tma_prefetch_desc(&tmW);
  }
  if (tid < 64) s_exp2[tid] = exp2((double)tid / 64.0);
  __syncthreads();

  // producer: chunk i = (tile i / nK, pivot chunk i % nK); independent of the tile, so
  // the ring runs ahead across tile boundaries.
  // Round robin over the group's warps (lane 0 of warp w issues chunks w, w + NCW, ...),
  // one chunk behind the consumer so the stage is already released: the TMA issue cost is
  // spread over the warps instead of stalling one of them every chunk (update_impl.cuh).
  int issued = warp;
  auto pump = [&](int done) {
    if (lane != 0) return;
    while (issued < total && issued < done + (S > 2 ? S - 1 : S)) {
      const int c = issued % nK, s = issued % S;
      if (issued >= S) mbar_wait(&empty[s], ((issued / S) & 1) ^ 1);
      unsigned char* Bs = stages + s * STAGE + C::A_BYTES;
      unsigned char* XSs = Bs + C::B_BYTES;
      mbar_arrive_expect_tx(&full[s], C::B_BYTES + nD * 2048);
      tma_load_2d(Bs, &tmW, 16 * c, 0, &full[s]);
      for (int dc = 0; dc < nD; ++dc) tma_load_2d(XSs + dc * 2048, &tmXS, 16 * dc, 16 * c, &full[s]);
      issued += NCW;
    }
  };
  pump(0);

  const int g = lane >> 2, t = lane & 3;
  const int wr = warp / WC, wc = warp % WC;
  const int pg = perm8(g);
  int arow[2];
#pragma unroll
  for (int fr = 0; fr < 2; ++fr) arow[fr] = wr * 16 + 8 * fr + pg;
  // foffs: the pivot-point operand of the register-path Gram is read at row sigma(g) =
  // perm8^{-1}(g) of each 8-row group, so C-fragment column 2t+v of fragment j is chunk
  // column 8j + 4v + t = 4(2j+v) + t: exactly the A-operand k order of k-step 2j+v, and the
  // W operand keeps the conflict-free fragment loads (foff).
  uint32_t foff[4], foffs[4];
  const int sg = (g >> 1) + 4 * (g & 1);  // perm8^{-1}(g)
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    foff[s] = swz_off(pg, 4 * s + t);
    foffs[s] = swz_off(sg, 4 * s + t);
  }
  const uint32_t a_base = (uint32_t)(wr * 16) * 128u;
  const uint32_t b_base = (uint32_t)(wc * NFW) * 1024u;
  const double escale = p.escale;
  const bool l1 = p.kind == kL1;

  double acc[2][NFW][2];
  int cons = 0;

#pragma unroll 1
  for (int k = 0; k < my_tiles; ++k) {
    const int tile = vb + k * vgrid;
    const int64_t tile_row0 = (int64_t)tile * BM;
    // X(R, :) for this tile (every warp is past the previous tile's generation: the
    // previous epilogue ended with a group barrier)
    if (gtid == 0) {
      mbar_arrive_expect_tx(xbar, nD * C::A_BYTES);
      for (int dc = 0; dc < nD; ++dc) tma_load_2d(xt + dc * C::A_BYTES, &tmX, 16 * dc, (int)tile_row0, xbar);
    }
    double sqr[2], gid[2];
#pragma unroll
    for (int fr = 0; fr < 2; ++fr) {
      const int64_t grow = tile_row0 + arow[fr];
      sqr[fr] = grow < p.n_loc ? p.sqn[grow] : 0.0;
      gid[fr] = p.pin ? (double)(p.row0 + grow) : -2.0;  // ids are >= 0, padding -1
    }
#pragma unroll
    for (int fr = 0; fr < 2; ++fr)
#pragma unroll
      for (int q = 0; q < NFW; ++q) acc[fr][q][0] = acc[fr][q][1] = 0.0;
    mbar_wait(xbar, k & 1);

#pragma unroll 1
    for (int c = 0; c < nK; ++c) {
      const int s = cons % S;
      mbar_wait(&full[s], (cons / S) & 1);
      __syncwarp();
      unsigned char* As = stages + s * STAGE;
      const unsigned char* Bs = As + C::A_BYTES;
      const unsigned char* XSs = Bs + C::B_BYTES;
      const int z = 16 * c - kold;  // W rows n have zeros beyond column kold + n
      const int q_lo = z > 0 ? max(0, z / 8 - wc * NFW) : 0;
      const unsigned char* Bw = Bs + b_base;
      if constexpr (WC == 1) {
        // ---- one warp column: the warp's 16 x 16 kernel tile stays in registers ------
        // Lane (g, t) generates rows arow[fr] x chunk columns kc(j, v) = 8j + 4v + t, exactly
        // the C-fragment positions of a Gram DMMA against the TMA-staged pivot rows read at
        // foffs; these are the A operand of k-step s = 2j + v as they sit in registers.
        double gv[2][2][2];
        if constexpr (GRAM) {
          // pivot norms / ids of this lane's four columns: issued before the Gram products so
          // their L2 latency hides behind the DMMA chain
          double sqc4[2][2], idc4[2][2];
#pragma unroll
          for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int v = 0; v < 2; ++v) {
              const int col = 16 * c + 8 * j + 4 * v + t;
              const bool cin = col < knew;
              sqc4[j][v] = cin ? __ldg(p.piv + (int64_t)col * p.prec + 1) : 0.0;
              idc4[j][v] = cin ? __ldg(p.piv + (int64_t)col * p.prec) : -1.0;
            }
#pragma unroll
          for (int fr = 0; fr < 2; ++fr)
#pragma unroll
            for (int j = 0; j < 2; ++j) gv[fr][j][0] = gv[fr][j][1] = 0.0;
#pragma unroll 1
          for (int dc = 0; dc < nD; ++dc) {
            const unsigned char* Xw = xt + dc * C::A_BYTES + a_base;
            const unsigned char* Sw = XSs + dc * 2048;
#pragma unroll
            for (int s4 = 0; s4 < 4; ++s4) {
              double a[2];
#pragma unroll
              for (int fr = 0; fr < 2; ++fr) a[fr] = *reinterpret_cast<const double*>(Xw + fr * 1024 + foff[s4]);
#pragma unroll
              for (int j = 0; j < 2; ++j) {
                const double bv = *reinterpret_cast<const double*>(Sw + j * 1024 + foffs[s4]);
#pragma unroll
                for (int fr = 0; fr < 2; ++fr) dmma884(gv[fr][j][0], gv[fr][j][1], a[fr], bv);
              }
            }
          }
#pragma unroll
          for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int v = 0; v < 2; ++v) {
              const double sqc = sqc4[j][v], idc = idc4[j][v];
#pragma unroll
              for (int fr = 0; fr < 2; ++fr) {
                double dd = __dadd_rn(__dadd_rn(-2.0 * gv[fr][j][v], sqr[fr]), sqc);
                dd = clamp_pin(dd, gid[fr], idc);
                gv[fr][j][v] = kfun_eval(dd, p.kfun, escale, s_exp2);
              }
            }
        } else {
          // direct / l1 distances in the same fragment positions, ascending coordinates
          double dsum[2][2][2];
#pragma unroll
          for (int fr = 0; fr < 2; ++fr)
#pragma unroll
            for (int j = 0; j < 2; ++j) dsum[fr][j][0] = dsum[fr][j][1] = 0.0;
#pragma unroll 1
          for (int dc = 0; dc < nD; ++dc) {
            const unsigned char* Xw = xt + dc * C::A_BYTES;
            const unsigned char* Sw = XSs + dc * 2048;
            const int jn = min(16, p.d - 16 * dc);
#pragma unroll 2
            for (int jj = 0; jj < jn; ++jj) {
              double xr[2], xs[2][2];
#pragma unroll
              for (int fr = 0; fr < 2; ++fr) xr[fr] = *reinterpret_cast<const double*>(Xw + swz_off(arow[fr], jj));
#pragma unroll
              for (int j = 0; j < 2; ++j)
#pragma unroll
                for (int v = 0; v < 2; ++v)
                  xs[j][v] = *reinterpret_cast<const double*>(Sw + swz_off(8 * j + 4 * v + t, jj));
#pragma unroll
              for (int fr = 0; fr < 2; ++fr)
#pragma unroll
                for (int j = 0; j < 2; ++j)
#pragma unroll
                  for (int v = 0; v < 2; ++v) {
                    const double df = __dsub_rn(xr[fr], xs[j][v]);
                    dsum[fr][j][v] = l1 ? __dadd_rn(dsum[fr][j][v], fabs(df))
                                        : __dadd_rn(dsum[fr][j][v], __dmul_rn(df, df));
                  }
            }
          }
#pragma unroll
          for (int fr = 0; fr < 2; ++fr)
#pragma unroll
            for (int j = 0; j < 2; ++j)
#pragma unroll
              for (int v = 0; v < 2; ++v) gv[fr][j][v] = kfun_eval(dsum[fr][j][v], p.kfun, escale, s_exp2);
        }
        // ---- acc += A(R, S_c) W(:, S_c)^T from registers --------------------------------
#pragma unroll
        for (int s4 = 0; s4 < 4; ++s4) {
#pragma unroll
          for (int q = 0; q < NFW; ++q) {
            if (q < q_lo) continue;
            const double bv = *reinterpret_cast<const double*>(Bw + q * 1024 + foff[s4]);
#pragma unroll
            for (int fr = 0; fr < 2; ++fr)
              dmma884(acc[fr][q][0], acc[fr][q][1], gv[fr][s4 >> 1][s4 & 1], bv);
          }
        }
      } else {
      // ---- regenerate the kernel tile A(R, S_c) (64 x 16) into As -----------------
      if constexpr (GRAM) {
        double ga[2][NG][2];
#pragma unroll
        for (int fr = 0; fr < 2; ++fr)
#pragma unroll
          for (int j = 0; j < NG; ++j) ga[fr][j][0] = ga[fr][j][1] = 0.0;
#pragma unroll 1
        for (int dc = 0; dc < nD; ++dc) {
          const unsigned char* Xw = xt + dc * C::A_BYTES + a_base;
          const unsigned char* Sw = XSs + dc * 2048;
#pragma unroll
          for (int s4 = 0; s4 < 4; ++s4) {
            double a[2];
#pragma unroll
            for (int fr = 0; fr < 2; ++fr) a[fr] = *reinterpret_cast<const double*>(Xw + fr * 1024 + foff[s4]);
#pragma unroll
            for (int j = 0; j < NG; ++j) {
              const int jj = WC == 1 ? j : wc;
              const double bv = *reinterpret_cast<const double*>(Sw + jj * 1024 + foff[s4]);
#pragma unroll
              for (int fr = 0; fr < 2; ++fr) dmma884(ga[fr][j][0], ga[fr][j][1], a[fr], bv);
            }
          }
        }
#pragma unroll
        for (int j = 0; j < NG; ++j) {
          const int jj = WC == 1 ? j : wc;
#pragma unroll
          for (int v = 0; v < 2; ++v) {
            // fragment column 2t+v of B fragment jj came from pivot row 8 jj + perm8(2t+v)
            const int kc = 8 * jj + perm8(2 * t + v);
            const int col = 16 * c + kc;
            const bool cin = col < knew;
            const double sqc = cin ? p.piv[(int64_t)col * p.prec + 1] : 0.0;
            const double idc = cin ? p.piv[(int64_t)col * p.prec] : -1.0;
#pragma unroll
            for (int fr = 0; fr < 2; ++fr) {
              double dd = __dadd_rn(__dadd_rn(-2.0 * ga[fr][j][v], sqr[fr]), sqc);
              dd = clamp_pin(dd, gid[fr], idc);
              *reinterpret_cast<double*>(As + swz_off(arow[fr], kc)) = kfun_eval(dd, p.kfun, escale, s_exp2);
            }
          }
        }
      } else {
        // direct / l1 distances, ascending coordinates (bit-identical to the reference sums):
        // lane -> row wr*16 + (lane & 15), columns c0 .. c0 + EPT
        constexpr int EPT = 8 / WC;
        const int r = wr * 16 + (lane & 15);
        const int c0 = (WC == 1 ? 0 : 8 * wc) + EPT * (lane >> 4);
        double da[EPT];
#pragma unroll
        for (int e = 0; e < EPT; ++e) da[e] = 0.0;
#pragma unroll 1
        for (int dc = 0; dc < nD; ++dc) {
          const unsigned char* Xw = xt + dc * C::A_BYTES;
          const unsigned char* Sw = XSs + dc * 2048;
          const int jn = min(16, p.d - 16 * dc);
#pragma unroll 4
          for (int jj = 0; jj < jn; ++jj) {
            const double xr = *reinterpret_cast<const double*>(Xw + swz_off(r, jj));
#pragma unroll
            for (int e = 0; e < EPT; ++e) {
              const double df = __dsub_rn(xr, *reinterpret_cast<const double*>(Sw + swz_off(c0 + e, jj)));
              da[e] = l1 ? __dadd_rn(da[e], fabs(df)) : __dadd_rn(da[e], __dmul_rn(df, df));
            }
          }
        }
#pragma unroll
        for (int e = 0; e < EPT; ++e)
          *reinterpret_cast<double*>(As + swz_off(r, c0 + e)) = kfun_eval(da[e], p.kfun, escale, s_exp2);
      }
      gsync();
      // ---- acc += A(R, S_c) W(:, S_c)^T; W rows n have zeros beyond column kold + n ----
      {
        const unsigned char* Aw = As + a_base;
#pragma unroll
        for (int s4 = 0; s4 < 4; ++s4) {
          double a[2];
#pragma unroll
          for (int fr = 0; fr < 2; ++fr) a[fr] = *reinterpret_cast<const double*>(Aw + fr * 1024 + foff[s4]);
#pragma unroll
          for (int q = 0; q < NFW; ++q) {
            if (q < q_lo) continue;
            const double bv = *reinterpret_cast<const double*>(Bw + q * 1024 + foff[s4]);
#pragma unroll
            for (int fr = 0; fr < 2; ++fr) dmma884(acc[fr][q][0], acc[fr][q][1], a[fr], bv);
          }
        }
      }
      }  // WC == 2
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      ++cons;
      pump(cons);
    }

    if (p.out_mode) {  // product mode: out = A(R, S) W^T (+ add terms)
#pragma unroll
      for (int fr = 0; fr < 2; ++fr) {
        const int64_t grow = tile_row0 + arow[fr];
        if (grow >= p.n_loc) continue;
        const double add = (p.add_vec ? p.add_coef * p.add_vec[grow] : 0.0) + p.add_const;
#pragma unroll
        for (int q = 0; q < NFW; ++q)
#pragma unroll
          for (int v = 0; v < 2; ++v) {
            // C column 2t+v of fragment q came from W row 8 (wc NFW + q) + perm8(2t+v)
            const int col = 8 * (wc * NFW + q) + perm8(2 * t + v);
            if (col < p.m) p.out[grow * p.ld_out + col] = acc[fr][q][v] + add;
          }
      }
      gsync();  // the next tile's X load overwrites xt
      continue;
    }
    // ---- epilogue: u(R) = max(u - rowwise ||g||^2, 0); per-tile ||g||_F^2 ----------
    // (W rows >= m are zero-filled by TMA, so padded columns contribute exactly 0)
    double rs[2] = {0.0, 0.0};
#pragma unroll
    for (int fr = 0; fr < 2; ++fr) {
#pragma unroll
      for (int q = 0; q < NFW; ++q)
#pragma unroll
        for (int v = 0; v < 2; ++v) rs[fr] = fma(acc[fr][q][v], acc[fr][q][v], rs[fr]);
      rs[fr] += __shfl_xor_sync(0xffffffffu, rs[fr], 1);
      rs[fr] += __shfl_xor_sync(0xffffffffu, rs[fr], 2);
      if (t == 0) s_rown[wc * BM + arow[fr]] = rs[fr];
    }
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
    gsync();
    if (gtid < 32) {  // fixed-order tree over the row sums (as update_impl.cuh)
      double s2 = 0.0;
      for (int r = gtid; r < BM; r += 32) s2 = __dadd_rn(s2, s_rowg2[r]);
      s2 = warp_sum_xor(s2);
      if (gtid == 0) p.tile_g2[tile] = s2;
    }
  }
}

template <int WC, int NFW, bool GRAM, int G, int MINB = 1>
int launch_lowmem_t(const LowmemParams& p, cudaStream_t st) {
  using C = LCfg<WC, NFW, G>;
  constexpr int kMaxSmem = 227 * 1024;
  const int nD = (int)(p.dpad / 16);
  int S = C::kMaxStages;
  while (S >= 2 && C::smem_bytes(S, nD) > kMaxSmem) --S;
  if (S < 2) return -1;  // dimension too large for a resident tile
  const void* kfn = (const void*)lowmem_kernel<WC, NFW, GRAM, G, MINB>;
  if (ensure_smem_attr(kfn, kMaxSmem) != cudaSuccess) return -2;
  CUtensorMap mX, mXS, mW;
  bool ok = make_map(&mX, p.X, p.dpad, p.n_loc, p.dpad, C::BM) &&
            make_map(&mXS, p.piv + 2, p.dpad, p.knew, p.prec, 16) &&
            make_map(&mW, p.W, p.knew, p.m, p.ldw, C::NB);
  if (!ok) return -3;
  const int64_t ntiles = (p.n_loc + C::BM - 1) / C::BM;
  // persistent grid: as many CTAs per SM as registers and shared memory allow (small m, as in
  // the KRR product mode, fits two, which hides the latency of the short per-chunk chains)
  const int occ = cached_occupancy(kfn, C::NT, C::smem_bytes(S, nD), 1);
  const unsigned grid = (unsigned)std::min<int64_t>((ntiles + G - 1) / G, (int64_t)occ * num_sms());
  if (grid)
    lowmem_kernel<WC, NFW, GRAM, G, MINB><<<grid, C::NT, C::smem_bytes(S, nD), st>>>(p, S, mX, mXS, mW);
  return C::BM;
}

}  // namespace rpcb
