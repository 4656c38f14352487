// i8gemm.cu — the round's residual GEMM C = F(:, :kcur) B'^T on the 5th-generation tensor
// cores through int8 slices (Ozaki scheme I), for rounds where it beats the FP64 DMMA
// phase of the fused update (which then adds C instead of running its own GEMM).
//
// Representation.  |F_ij| <= 1 (unit-diagonal kernels: ||F_i||^2 = 1 - u_i <= 1), so F is
// held as kSlices signed base-2^7 digits of F * 2^6 at a fixed scale:
//   F_ij = sum_t f_t 2^(-6 - 7 t) + e,  |f_t| <= 64,  |e| <= 2^-49,
// kept beside F as int8 planes [kSlices][kcap / 64][rows][64] (each round appends its new
// columns: launch_slice_cols).  B' (m x kcur, per round) is scaled per row by 2^-e_c (max |B'_c,:| <
// 2^e_c) and sliced the same way.  Then
//   C_ic = 2^(e_c - 12) sum_{d < kSlices} 2^(-7 d) A_d(i, c),  A_d = sum_{t + u = d} f_t b_u^T,
// each A_d an exact int32 sum (|f_t b_u| <= 2^12, k <= 2^15 / (d + 1) terms) accumulated by
// tcgen05.mma.kind::i8 in tensor memory; the dropped digit products (t + u >= kSlices) and the
// representation error bound the result at ~6e-14 of sum_j |F_ij| |B'_cj| (tools/ozaki_probe.cu:
// 6.2e-14 measured at the C4 round-9 shape; the FP64 DMMA GEMM it replaces is ~1e-16 of that).
//
// Kernels (both persistent, one CTA per SM; warp 0 issues the TMA loads of 64-byte K blocks with
// the 64-byte swizzle, one elected thread of warp 1 the MMAs, the other warps drain tensor
// memory with tcgen05.ld, sum the diagonals in FP64 and apply the column scale, releasing each
// accumulator to the next MMAs as soon as it is read):
//   i8gemm_kernel   m <= 64: tiles of 128 rows x 64 columns, kSlices accumulators x 64 TMEM
//                   columns (448 of 512), two stages;
//   i8gemm2_kernel  64 < m <= 128: tiles of 128 rows x all columns, N = m rounded up to 16, two
//                   passes over K (diagonals 0-3, then 4-6) in four 128-column accumulators.
// DESIGN.md 4.6 has the measurements and the shared-memory-port bound.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <mutex>

#include "common.cuh"
#include "i8digits.cuh"
#include "kernels.h"

namespace rpcb {

constexpr int kSlices = kI8Slices;
constexpr int kI8BM = 128, kI8BN = 64, kI8KB = 64, kI8Nst = 2;
constexpr int kI8Apl = kI8BM * kI8KB, kI8Bpl = kI8BN * kI8KB;
constexpr int kI8Stage = kSlices * (kI8Apl + kI8Bpl);

__device__ __forceinline__ void tma_load_3d(void* smem_dst, const void* tmap, int c0, int c1, int c2,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

// K-major operand tile of 64-byte rows with the 64-byte swizzle (two MMA K steps per row)
__device__ __forceinline__ uint64_t umma_desc_sw64(uint32_t saddr) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1 << 16;           // leading byte offset (unused: swizzled K-major)
  d |= (uint64_t)(512 >> 4) << 32;  // stride byte offset: 8 rows x 64 B
  d |= (uint64_t)1 << 46;           // descriptor version (sm_100)
  d |= (uint64_t)4 << 61;           // SWIZZLE_64B
  return d;
}

// Persistent: a CTA per SM walks the (row tile, column half) tiles.  The epilogue drains the
// diagonals in order d = 0 .. 6 (C = sum_d 2^(-7 d) A_d accumulated in FP64 registers, 64
// columns a thread) and releases each diagonal's TMEM columns as soon as it has read them; the
// next tile's first K block issues its products diagonal by diagonal, each diagonal's first
// product (which overwrites) after that release, so the drain overlaps the next tile's MMAs.
__global__ void __launch_bounds__(192, 1) i8gemm_kernel(const __grid_constant__ CUtensorMap tmA,
                                                       const __grid_constant__ CUtensorMap tmB,
                                                       int a_nblk, int b_plane_rows,
                                                       int64_t n_rows, int m, int nkb, int ncolt,
                                                       int64_t ntiles,
                                                       const double* __restrict__ cscale,
                                                       double* __restrict__ C, int64_t ldc) {
  extern __shared__ __align__(1024) unsigned char smraw[];
  unsigned char* sm = smraw + ((1024u - (smem_u32(smraw) & 1023u)) & 1023u);
  __shared__ uint64_t full[kI8Nst], empty[kI8Nst], done, drained[kSlices];
  __shared__ uint32_t tmem_base_s;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kI8Nst; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&done, 1);
    for (int d = 0; d < kSlices; ++d) mbar_init(&drained[d], 4);
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
    if (elect_one()) {
      int it = 0;  // stage use counter across tiles
      for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int64_t row0 = (tile / ncolt) * kI8BM;
        const int col0 = (int)(tile % ncolt) * kI8BN;
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int s = it % kI8Nst;
          if (it >= kI8Nst) mbar_wait(&empty[s], ((it / kI8Nst) - 1) & 1);
          mbar_arrive_expect_tx(&full[s], kI8Stage);
          unsigned char* st = sm + s * kI8Stage;
          for (int t = 0; t < kSlices; ++t)
            tma_load_3d(st + t * kI8Apl, &tmA, 0, (int)row0, t * a_nblk + kb, &full[s]);
          for (int u = 0; u < kSlices; ++u)
            tma_load_2d(st + kSlices * kI8Apl + u * kI8Bpl, &tmB, kb * kI8KB,
                        u * b_plane_rows + col0, &full[s]);
        }
      }
    }
  } else if (warp == 1) {
    if (elect_one()) {
      // kind::i8: D s32, A and B signed int8, both K-major, M = 128, N = 64
      const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) |
                             ((uint32_t)(kI8BN >> 3) << 17) | ((uint32_t)(kI8BM >> 4) << 24);
      int it = 0, ti = 0;
      for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++ti) {
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int s = it % kI8Nst;
          mbar_wait(&full[s], (it / kI8Nst) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
          const uint32_t ba = smem_u32(sm + s * kI8Stage), bb = ba + kSlices * kI8Apl;
          // products diagonal by diagonal; in the first K block a diagonal's first product
          // overwrites it, once the previous tile's epilogue has drained it
#pragma unroll
          for (int d = 0; d < kSlices; ++d) {
            if (kb == 0 && ti > 0) {
              mbar_wait(&drained[d], (ti - 1) & 1);
              asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
            }
#pragma unroll
            for (int t = 0; t <= d; ++t)
#pragma unroll
              for (int ks = 0; ks < kI8KB / 32; ++ks) {
                const uint64_t da = umma_desc_sw64(ba + t * kI8Apl + ks * 32);
                const uint64_t db = umma_desc_sw64(bb + (d - t) * kI8Bpl + ks * 32);
                const uint32_t accum = (kb | ks | t) != 0;
                asm volatile(
                    "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                    "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(
                        tbase + (uint32_t)(d * kI8BN)),
                    "l"(da), "l"(db), "r"(idesc), "r"(accum));
              }
          }
          asm volatile(
              "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                  smem_u32(&empty[s])));
        }
        asm volatile(
            "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                smem_u32(&done)));
      }
    }
  } else {
    const int q = warp & 3;  // the TMEM lane quadrant this warp may read
    int ti = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++ti) {
      const int64_t r = (tile / ncolt) * kI8BM + q * 32 + lane;
      const int col0 = (int)(tile % ncolt) * kI8BN;
      mbar_wait(&done, ti & 1);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      double acc[kI8BN];
#pragma unroll
      for (int j = 0; j < kI8BN; ++j) acc[j] = 0.0;
      double wd = 1.0;  // 2^(-7 d)
#pragma unroll
      for (int d = 0; d < kSlices; ++d) {
#pragma unroll
        for (int cc = 0; cc < kI8BN / 16; ++cc) {
          uint32_t v[16];
          const uint32_t ta = tbase + ((uint32_t)(q * 32) << 16) + (uint32_t)(d * kI8BN + cc * 16);
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, "
              "%10, %11, %12, %13, %14, %15}, [%16];\n"
              : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
                "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]),
                "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
              : "r"(ta));
          asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
          for (int j = 0; j < 16; ++j) acc[cc * 16 + j] = fma((double)(int)v[j], wd, acc[cc * 16 + j]);
        }
        // this warp's reads of diagonal d are complete: release its TMEM columns
        asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&drained[d]);
        wd *= 0.0078125;
      }
      if (r < n_rows) {
        double* cr = C + r * ldc + col0;
#pragma unroll
        for (int j = 0; j < kI8BN; j += 2) {
          const int c = col0 + j;
          if (c + 1 < m)
            *reinterpret_cast<double2*>(cr + j) =
                make_double2(acc[j] * cscale[c], acc[j + 1] * cscale[c + 1]);
          else if (c < m)
            cr[j] = acc[j] * cscale[c];
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tbase));
}

// Two-pass variant for 64 < m <= 128: tiles of 128 F rows x all (<= 128) output columns, MMAs
// with N = m rounded up to 16.  By operand traffic the one-pass kernel above is bound by shared
// memory (an M = 128, N = 64, K = 32 product reads 4 KB of A and 2 KB of B for 32 cycles of
// tensor work); N = 128 halves the A reads per output, but seven 128-column accumulators do
// not fit tensor memory, so a tile makes two passes over K: diagonals 0 .. 3 (10 products; only
// digit planes 0 .. 3 of either operand are loaded) in four 128-column slots, then diagonals
// 4 .. 6 (18 products, all planes) in slots 0 .. 2.  Per 128 x 128 x 64-byte block that is
// 176 KB of TMA writes + 448 KB of operand reads against 168 + 672 KB for two one-pass tiles.
// The epilogue (8 warps: TMEM lane quadrant x column half) keeps its FP64 sums in registers
// across the two passes and releases each slot as soon as it is read, as above.
constexpr int kI8N2 = 128, kI8Bpl2 = kI8N2 * kI8KB;
constexpr int kI8Stage2 = kSlices * (kI8Apl + kI8Bpl2);
constexpr int kI8P1 = 4;  // diagonals (and digit planes) of the first pass

// The products of one K block of pass PASS (diagonals 0 .. 3 or 4 .. 6) from the stage at `ba`
// (a loop-invariant address: every descriptor is that base plus a constant).  Not the first K
// block of a pass (those products overwrite and wait for the drains).
template <int PASS>
__device__ __forceinline__ void i8_issue_kblock(uint32_t ba, uint32_t tbase, uint32_t idesc) {
  constexpr int d0 = PASS == 0 ? 0 : kI8P1, d1 = PASS == 0 ? kI8P1 : kSlices;
  const uint32_t bb = ba + kSlices * kI8Apl;
#pragma unroll
  for (int d = d0; d < d1; ++d)
#pragma unroll
    for (int t = 0; t <= d; ++t)
#pragma unroll
      for (int ks = 0; ks < kI8KB / 32; ++ks) {
        const uint64_t da = umma_desc_sw64(ba + t * kI8Apl + ks * 32);
        const uint64_t db = umma_desc_sw64(bb + (d - t) * kI8Bpl2 + ks * 32);
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(
                tbase + (uint32_t)((d - d0) * kI8N2)),
            "l"(da), "l"(db), "r"(idesc), "r"(1u));
      }
}

__global__ void __launch_bounds__(320, 1) i8gemm2_kernel(const __grid_constant__ CUtensorMap tmA,
                                                        const __grid_constant__ CUtensorMap tmB,
                                                        int a_nblk, int64_t n_rows, int m, int nkb,
                                                        int64_t ntiles,
                                                        const double* __restrict__ cscale,
                                                        double* __restrict__ C, int64_t ldc,
                                                        int dbg, long long* trace) {
  // RPC_I8_DEBUG bit 4: block 0 stamps its first tiles' pass transitions (16 slots per tile)
#define I8_STAMP(ev)                                                                       \
  do {                                                                                     \
    if (trace != nullptr && blockIdx.x == 0 && tile < 8 * (int64_t)gridDim.x)              \
      trace[(tile / gridDim.x) * 16 + (ev)] = clock64();                                   \
  } while (0)
  extern __shared__ __align__(1024) unsigned char smraw[];
  unsigned char* sm = smraw + ((1024u - (smem_u32(smraw) & 1023u)) & 1023u);
  __shared__ uint64_t full[kI8Nst], empty[kI8Nst], done, drained[kI8P1];
  __shared__ uint32_t tmem_base_s;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nmma = (m + 15) & ~15;  // MMA N: live columns rounded up to 16
  if (threadIdx.x == 0) {
    for (int s = 0; s < kI8Nst; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&done, 1);
    for (int d = 0; d < kI8P1; ++d) mbar_init(&drained[d], 8);
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
      int it = 0;  // stage use counter across tiles and passes
      for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int64_t row0 = tile * kI8BM;
        for (int pass = 0; pass < 2; ++pass) {
          const int np = pass == 0 ? kI8P1 : kSlices;
          for (int kb = 0; kb < nkb; ++kb, ++it) {
            const int s = it % kI8Nst;
            if (it >= kI8Nst) mbar_wait(&empty[s], ((it / kI8Nst) - 1) & 1);
            if (dbg & 1) {  // RPC_I8_DEBUG bit 0: no loads (the products read stale stages)
              mbar_arrive(&full[s]);
              continue;
            }
            mbar_arrive_expect_tx(&full[s], (uint32_t)np * (kI8Apl + kI8Bpl2));
            unsigned char* st = sm + s * kI8Stage2;
            for (int t = 0; t < np; ++t)
              tma_load_3d(st + t * kI8Apl, &tmA, 0, (int)row0, t * a_nblk + kb, &full[s]);
            for (int u = 0; u < np; ++u)
              tma_load_2d(st + kSlices * kI8Apl + u * kI8Bpl2, &tmB, kb * kI8KB, u * kI8N2,
                          &full[s]);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (elect_one()) {
      // kind::i8: D s32, A and B signed int8, both K-major, M = 128, N = nmma
      const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(nmma >> 3) << 17) |
                             ((uint32_t)(kI8BM >> 4) << 24);
      const uint32_t ba0 = smem_u32(sm), ba1 = ba0 + kI8Stage2;  // the two stages
      int it = 0;
      uint32_t uses[kI8P1] = {0, 0, 0, 0};  // completed uses of each accumulator slot
      for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        for (int pass = 0; pass < 2; ++pass) {
          const int d0 = pass == 0 ? 0 : kI8P1;
          for (int kb = 0; kb < nkb; ++kb, ++it) {
            const int s = it & 1;
            mbar_wait(&full[s], (it >> 1) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
            if (dbg & 2) {  // RPC_I8_DEBUG bit 1: no products (loads + drains only)
            } else if (kb > 0) {
              if (pass == 0) {
                if (s == 0) i8_issue_kblock<0>(ba0, tbase, idesc);
                else i8_issue_kblock<0>(ba1, tbase, idesc);
              } else {
                if (s == 0) i8_issue_kblock<1>(ba0, tbase, idesc);
                else i8_issue_kblock<1>(ba1, tbase, idesc);
              }
            } else {
              // first K block of the pass: a slot's first product overwrites it, after the
              // epilogue has drained its previous use
              const uint32_t ba = s == 0 ? ba0 : ba1, bb = ba + kSlices * kI8Apl;
#pragma unroll
              for (int sl = 0; sl < kI8P1; ++sl) {
                const int d = d0 + sl;
                if (d >= kSlices) break;
                if (uses[sl] > 0) {
                  if (sl == 0) I8_STAMP(pass * 4 + 0);
                  mbar_wait(&drained[sl], (uses[sl] - 1) & 1);
                  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
                  if (sl == 0) I8_STAMP(pass * 4 + 1);
                  if (sl == 2) I8_STAMP(pass * 4 + 2);
                }
                for (int t = 0; t <= d; ++t)
#pragma unroll
                  for (int ks = 0; ks < kI8KB / 32; ++ks) {
                    const uint64_t da = umma_desc_sw64(ba + t * kI8Apl + ks * 32);
                    const uint64_t db = umma_desc_sw64(bb + (d - t) * kI8Bpl2 + ks * 32);
                    const uint32_t accum = (ks | t) != 0;
                    asm volatile(
                        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(
                            tbase + (uint32_t)(sl * kI8N2)),
                        "l"(da), "l"(db), "r"(idesc), "r"(accum));
                  }
              }
            }
            asm volatile(
                "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                    smem_u32(&empty[s])));
          }
          asm volatile(
              "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                  smem_u32(&done)));
          I8_STAMP(pass * 4 + 3);
#pragma unroll
          for (int sl = 0; sl < kI8P1; ++sl)
            if (d0 + sl < kSlices) ++uses[sl];
        }
      }
    }
  } else {
    const int q = warp & 3;         // the TMEM lane quadrant this warp may read
    const int h = (warp - 2) >> 2;  // column half
    const int nch = min(4, max(0, (nmma - h * 64) >> 4));  // live 16-column chunks of this half
    uint32_t np = 0;                // passes seen (parity of `done`)
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      const int64_t r = tile * kI8BM + q * 32 + lane;
      double acc[64];
#pragma unroll
      for (int j = 0; j < 64; ++j) acc[j] = 0.0;
#pragma unroll
      for (int pass = 0; pass < 2; ++pass) {
        mbar_wait(&done, np & 1);
        ++np;
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        if (threadIdx.x == 64) I8_STAMP(8 + pass * 3);
        // slots drained in pairs: P = 128 A_d + A_(d+1) folded exactly in int64 (|A_d| < 2^28) and
        // converted through the 1.5 2^52 bit pattern: two full-rate FP64 operations per output
        // and pair instead of two I2F.F64 + two DFMA; both slots are released right after their
        // last TMEM read, ahead of that chunk's arithmetic
#pragma unroll
        for (int sl = 0; sl < (pass == 0 ? kI8P1 : kSlices - kI8P1); sl += 2) {
          const int d = pass * kI8P1 + sl;
          const bool pairq = d + 1 < kSlices;
          const double wd = 1.0 / (double)(1ull << (7 * (pairq ? d + 1 : d)));  // weight of the fold
#pragma unroll
          for (int cc = 0; cc < 4; ++cc) {
            if (cc < nch) {
              uint32_t v[16], w[16];
              const uint32_t ta = tbase + ((uint32_t)(q * 32) << 16) +
                                  (uint32_t)(sl * kI8N2 + h * 64 + cc * 16);
              asm volatile(
                  "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, "
                  "%10, %11, %12, %13, %14, %15}, [%16];\n"
                  : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
                    "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]),
                    "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                  : "r"(ta));
              if (pairq)
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, "
                    "%9, %10, %11, %12, %13, %14, %15}, [%16];\n"
                    : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]),
                      "=r"(w[6]), "=r"(w[7]), "=r"(w[8]), "=r"(w[9]), "=r"(w[10]), "=r"(w[11]),
                      "=r"(w[12]), "=r"(w[13]), "=r"(w[14]), "=r"(w[15])
                    : "r"(ta + (uint32_t)kI8N2));
              asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
              if (cc == nch - 1) {
                // this warp's reads of the slots are complete: release their TMEM columns
                asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
                __syncwarp();
                if (lane == 0) {
                  mbar_arrive(&drained[sl]);
                  if (pairq) mbar_arrive(&drained[sl + 1]);
                }
                if (threadIdx.x == 64) I8_STAMP(8 + pass * 3 + 1 + (sl >> 1));
              }
              if (dbg & 8) {  // RPC_I8_DEBUG bit 3: no conversions
                acc[cc * 16] += __longlong_as_double((long long)(v[0] ^ v[5] ^ w[10] ^ w[15]));
                continue;
              }
#pragma unroll
              for (int j = 0; j < 16; ++j) {
                double x;
                if (pairq) {
                  const long long P = (long long)(int)v[j] * 128 + (long long)(int)w[j];
                  x = __longlong_as_double(P + 0x4338000000000000LL) - 6755399441055744.0;
                } else {
                  x = __hiloint2double(0x43300000, (int)(v[j] ^ 0x80000000u)) - 4503601774854144.0;
                }
                acc[cc * 16 + j] = fma(x, wd, acc[cc * 16 + j]);
              }
            }
          }
        }
      }
      if (dbg & 4) {  // RPC_I8_DEBUG bit 2: no C stores
        double sacc = 0.0;
#pragma unroll
        for (int j = 0; j < 64; ++j) sacc += acc[j];
        if (sacc == 1.2345e300) C[0] = sacc;
      } else if (r < n_rows) {
        // a thread owns 512 contiguous bytes of its row of C: 256-bit stores (whole 32-byte
        // sectors; 16-byte stores at the 1 KB row stride cost 275 us of a 1.5 ms launch).
        // Columns from m on are written too (zeros: their cscale is 0, C is 128 columns wide).
        double* cr = C + r * ldc + h * 64;
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) {
          if (cc < nch) {
#pragma unroll
            for (int j = cc * 16; j < cc * 16 + 16; j += 4) {
              const int c = h * 64 + j;
              const double4 sc4 = *reinterpret_cast<const double4*>(cscale + c);
              asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(cr + j),
                           "d"(acc[j] * sc4.x), "d"(acc[j + 1] * sc4.y), "d"(acc[j + 2] * sc4.z),
                           "d"(acc[j + 3] * sc4.w)
                           : "memory");
            }
          }
        }
      }
      if (threadIdx.x == 64) I8_STAMP(14);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tbase));
}
#undef I8_STAMP

// kSlices digits of v * 2^6 (|v| <= 1) in base 2^7, each rounded to nearest (magic-number rint)
__device__ __forceinline__ void slice_value(double v, int8_t* out, int64_t pstride) {
  constexpr double kM = 6755399441055744.0;  // 1.5 * 2^52
  double r = v * 64.0;
#pragma unroll
  for (int t = 0; t < kSlices; ++t) {
    const double rr = r + kM;
    out[t * pstride] = (int8_t)__double2loint(rr);
    r = (r - (rr - kM)) * 128.0;
  }
}

// Appends F(:, c0:c0+nc) to the digit planes (i8digits.cuh): a thread per (row, 8-column
// group), two 256-bit loads of F, one 64-bit store per plane.  (Appending from the update
// kernel's epilogue — each warp re-reading its 16 rows of G through L2 — measured slower:
// C4 39.7 vs 37.4 ms.)
__global__ void __launch_bounds__(256) slice_cols_kernel(const double* __restrict__ F, int64_t ldf,
                                                         int64_t n, int c0, int nc,
                                                         int8_t* __restrict__ planes,
                                                         int64_t pstride, int64_t bstride) {
  const int g0 = c0 >> 3, ng = ((c0 + nc + 7) >> 3) - g0;
  const int64_t item = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (item >= n * ng) return;
  int64_t r;
  if (n * ng < (int64_t)1 << 31) r = (int64_t)((uint32_t)item / (uint32_t)ng);
  else r = item / ng;
  const int g = g0 + (int)(item - r * ng);
  i8_append_group(F + r * ldf, r, g, c0, c0 + nc, planes, pstride, bstride);
}

// B' rows (logical a < m at bp[perm_row(a)], columns < kcur): per-row scale 2^-e (max < 2^e),
// planes [t][a][k] zero for k >= kcur and for rows m <= a < rows_pad; cscale[a] = 2^(e - 12)
__global__ void __launch_bounds__(256) slice_bprime_kernel(const double* __restrict__ bp,
                                                           int64_t ldbp, int m, int kcur,
                                                           int kpad, int8_t* __restrict__ planes,
                                                           int64_t pstride,
                                                           double* __restrict__ cscale) {
  const int a = blockIdx.x;
  __shared__ double s_max[8];
  const double* row = bp + (int64_t)perm_row(a) * ldbp;
  double mx = 0.0;
  if (a < m)
    for (int k = threadIdx.x; k < kcur; k += blockDim.x) mx = fmax(mx, fabs(__ldg(row + k)));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) s_max[threadIdx.x >> 5] = mx;
  __syncthreads();
  mx = 0.0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) mx = fmax(mx, s_max[w]);
  int e = 0;
  if (mx > 0.0) frexp(mx, &e);  // mx = f 2^e, f in [0.5, 1)
  const double sc = ldexp(1.0, -e);
  if (threadIdx.x == 0) cscale[a] = a < m ? ldexp(1.0, e - 12) : 0.0;
  for (int k = threadIdx.x; k < kpad; k += blockDim.x) {
    const double v = (a < m && k < kcur) ? __ldg(row + k) * sc : 0.0;
    slice_value(v, planes + (int64_t)a * kpad + k, pstride);
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 i8_encode_fn() {
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

// F's planes as a 3D tensor {64 bytes, plane_rows, kI8Slices * nblk}: box {64, 128, 1}
static bool i8_map_a(CUtensorMap* mp, const void* base, int64_t plane_rows, int64_t nblk_all) {
  auto fn = i8_encode_fn();
  if (!fn) return false;
  cuuint64_t dims[3] = {64, (cuuint64_t)plane_rows, (cuuint64_t)nblk_all};
  cuuint64_t strides[2] = {64, (cuuint64_t)(plane_rows * 64)};
  cuuint32_t box[3] = {(cuuint32_t)kI8KB, (cuuint32_t)kI8BM, 1};
  cuuint32_t es[3] = {1, 1, 1};
  return fn(mp, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<void*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static bool i8_map(CUtensorMap* mp, const void* base, int64_t inner, int64_t rows, int64_t pitch,
                   int box_rows) {
  auto fn = i8_encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)pitch};
  cuuint32_t box[2] = {(cuuint32_t)kI8KB, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  return fn(mp, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

void launch_slice_cols(const double* F, int64_t ldf, int64_t n, int c0, int nc, int8_t* planes,
                       int64_t plane_rows, int64_t kcap, cudaStream_t st) {
  if (n <= 0 || nc <= 0) return;
  const int ng = ((c0 + nc + 7) >> 3) - (c0 >> 3);
  const int64_t items = n * ng;
  slice_cols_kernel<<<(unsigned)((items + 255) / 256), 256, 0, st>>>(
      F, ldf, n, c0, nc, planes, plane_rows * kcap, plane_rows * 64);
}

int launch_i8_residual(const int8_t* fplanes, int64_t plane_rows, int64_t kcap, int64_t n_rows,
                       const double* bp, int64_t ldbp, int m, int kcur, int8_t* bplanes,
                       double* cscale, double* C, int64_t ldc, cudaStream_t st) {
  if (m < 1 || m > kI8MaxCols || kcur < 1 || n_rows <= 0) return -1;
  const int kpad = (kcur + kI8KB - 1) / kI8KB * kI8KB;
  if (kpad > kcap) return -1;
  const int mpad = (m + kI8BN - 1) / kI8BN * kI8BN;  // B plane rows (zeros beyond m)
  slice_bprime_kernel<<<mpad, 256, 0, st>>>(bp, ldbp, m, kcur, kpad, bplanes,
                                            (int64_t)mpad * kpad, cscale);
  // 64 < m <= 128: the two-pass kernel (RPC_I8_ONEPASS keeps the one-pass tiles for comparison)
  static const bool one_pass = std::getenv("RPC_I8_ONEPASS") != nullptr;
  const bool two_pass = mpad == kI8N2 && !one_pass;
  CUtensorMap mA, mB;
  if (!i8_map_a(&mA, fplanes, plane_rows, (int64_t)kSlices * (kcap / 64)) ||
      !i8_map(&mB, bplanes, kpad, (int64_t)kSlices * mpad, kpad, two_pass ? kI8N2 : kI8BN))
    return -3;
  const int a_nblk = (int)(kcap / 64), nkb = kpad / kI8KB, ncolt = mpad / kI8BN;
  if (two_pass) {
    const size_t smem2 = (size_t)kI8Nst * kI8Stage2 + 1024;
    const int64_t ntiles2 = (n_rows + kI8BM - 1) / kI8BM;
    if (ensure_smem_attr((const void*)i8gemm2_kernel, (int)smem2) != cudaSuccess) return -2;
    const unsigned grid2 = (unsigned)std::min<int64_t>(ntiles2, num_sms());
    // RPC_I8_DEBUG (timing experiments only, wrong results): 1 = no TMA loads, 2 = no products
    static const int dbg = [] {
      const char* e = std::getenv("RPC_I8_DEBUG");
      return e ? std::atoi(e) : 0;
    }();
    static long long* trace = nullptr;
    if ((dbg & 16) && trace == nullptr) {
      cudaMalloc(&trace, sizeof(long long) * 128);
      cudaMemset(trace, 0, sizeof(long long) * 128);
    }
    i8gemm2_kernel<<<grid2, 320, smem2, st>>>(mA, mB, a_nblk, n_rows, m, nkb, ntiles2, cscale, C,
                                              ldc, dbg, trace);
    if (dbg & 16) {
      long long h[128];
      cudaStreamSynchronize(st);
      cudaMemcpy(h, trace, sizeof(h), cudaMemcpyDeviceToHost);
      for (int t = 0; t < 8; ++t) {
        std::fprintf(stderr, "[i8 trace] tile %d nkb %d:", t, nkb);
        for (int e = 0; e < 16; ++e) std::fprintf(stderr, " %lld", h[t * 16 + e] ? h[t * 16 + e] - h[3] : 0);
        std::fprintf(stderr, "\n");
      }
    }
    return 0;
  }
  const size_t smem = (size_t)kI8Nst * kI8Stage + 1024;
  const int64_t ntiles = (n_rows + kI8BM - 1) / kI8BM * ncolt;
  if (ensure_smem_attr((const void*)i8gemm_kernel, (int)smem) != cudaSuccess) return -2;
  const unsigned grid = (unsigned)std::min<int64_t>(ntiles, num_sms());
  i8gemm_kernel<<<grid, 192, smem, st>>>(mA, mB, a_nblk, mpad, n_rows, m, nkb, ncolt, ntiles,
                                         cscale, C, ldc);
  return 0;
}

}  // namespace rpcb
