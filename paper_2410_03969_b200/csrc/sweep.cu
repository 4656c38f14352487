// sweep.cu — K3 (proposal block H), K4 (rejection-sampling Cholesky sweep in one
// CTA) and the accepted block's inverse L^{-1} used by the fused update (K6).
//
// H (rpcholesky.hpp:366-371) = A(S', S') - F(S', :) F(S', :)^T over the b
// proposals in draw order (duplicates included).  The kernel part follows
// oracle.hpp:71-90 / 103-112 and kernels.hpp:60-64 operation by operation
// without FMA contraction, so given identical inputs it matches the CPU oracle
// up to the last-ulp difference between CUDA's and glibc's exp().
//
// The sweep (rpcholesky.hpp:167-201) replays the reference's exact operation
// order: accept iff u_i * r_i < h_ii (u = diag(H) at entry, one draw per
// proposal, counters draw0 + i), root = sqrt(h_ii), l_j = h_ji / root,
// h_pq -= l_p * l_q with two roundings.  Only the lower triangle of H is ever
// read by the reference sweep, so it is held packed in shared memory.
#include <algorithm>

#include "common.cuh"
#include "kentry.cuh"
#include "kernels.h"

namespace rpcb {

// One 16 x 16 tile of H per CTA (lower-triangle tiles only: the sweep reads q <= p), its
// k range split over gridDim.z CTAs so the dependent add chains are short: CTA z sums
// k in its slab sequentially (no FMA) into part[z][tile][256]; the last CTA of a tile to
// finish (ticket counter, self-resetting) adds the slab partials in slab order and writes
// H = A(S', S') - total.  The order is fixed, so H is the same on every shard and run.
// The 128-wide k slabs are double-buffered through registers so the L2 latency of slab
// s + 1 hides behind the dependent add chain of slab s.
__global__ void __launch_bounds__(256) hblock_kernel(const double* __restrict__ prop,
                                                     RecordLayout lay, int b, int d, int kcur,
                                                     int kind, int kfun, double sigma,
                                                     double* __restrict__ H, int kslab,
                                                     double* __restrict__ part,
                                                     unsigned* __restrict__ tickets) {
  if (blockIdx.x > blockIdx.y) return;
  __shared__ double sp[16][129];
  __shared__ double sq[16][129];
  __shared__ int s_last;
  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * 16 + tx;
  const int p = blockIdx.y * 16 + ty, q = blockIdx.x * 16 + tx;
  const int ks0 = blockIdx.z * kslab, ks1 = min(kcur, ks0 + kslab);
  // this thread's share of a slab: rows rr0 + 2 e, column kk
  const int kk = tid & 127, rr0 = tid >> 7;
  const double* rp[8];
  const double* rq[8];
  bool vp[8], vq[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const int rr = rr0 + 2 * e;
    const int pp = blockIdx.y * 16 + rr, qq = blockIdx.x * 16 + rr;
    vp[e] = pp < b;
    vq[e] = qq < b;
    rp[e] = prop + (int64_t)(vp[e] ? pp : 0) * lay.rec + lay.foff + kk;
    rq[e] = prop + (int64_t)(vq[e] ? qq : 0) * lay.rec + lay.foff + kk;
  }
  double np[8], nq[8];
  auto fetch = [&](int k0) {
    const bool kin = k0 + kk < ks1;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      np[e] = (vp[e] && kin) ? __ldg(rp[e] + k0) : 0.0;
      nq[e] = (vq[e] && kin) ? __ldg(rq[e] + k0) : 0.0;
    }
  };
  double acc = 0.0;
  if (ks0 < ks1) fetch(ks0);
  for (int k0 = ks0; k0 < ks1; k0 += 128) {
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      sp[rr0 + 2 * e][kk] = np[e];
      sq[rr0 + 2 * e][kk] = nq[e];
    }
    __syncthreads();
    if (k0 + 128 < ks1) fetch(k0 + 128);
    const int kend = min(128, ks1 - k0);
#pragma unroll 8
    for (int k = 0; k < kend; ++k) acc = __dadd_rn(acc, __dmul_rn(sp[ty][k], sq[tx][k]));
    __syncthreads();
  }
  const int nz = gridDim.z;
  if (nz > 1) {
    const int tile = blockIdx.y * gridDim.x + blockIdx.x;
    part[((int64_t)blockIdx.z * gridDim.x * gridDim.y + tile) * 256 + tid] = acc;
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = atomicAdd(&tickets[tile], 1u) == (unsigned)(nz - 1);
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    acc = 0.0;
    for (int z = 0; z < nz; ++z)
      acc = __dadd_rn(acc, __ldcg(part + ((int64_t)z * gridDim.x * gridDim.y + tile) * 256 + tid));
    if (tid == 0) tickets[tile] = 0u;
  }
  if (p < b && q < b && q <= p) {
    const double a = kernel_entry(prop + (int64_t)p * lay.rec, prop + (int64_t)q * lay.rec, lay,
                                  d, kind, kfun, sigma);
    H[(int64_t)p * b + q] = __dsub_rn(a, acc);
  }
}

int hblock_splits(int b, int kcur) {
  const int nb = (b + 15) / 16, tiles = nb * (nb + 1) / 2;
  const int by_k = (kcur + 127) / 128;
  const int by_grid = std::max(1, 296 / tiles);  // ~2 CTAs per SM
  return std::max(1, std::min(by_k, by_grid));
}

void launch_hblock(const double* prop, RecordLayout lay, int b, int dpad, int d, int kcur,
                   int kind, int kfun, double sigma, double* H, cudaStream_t st, double* part,
                   unsigned* tickets) {
  (void)dpad;
  const int nb = (b + 15) / 16;
  const int nz = part && tickets ? hblock_splits(b, kcur) : 1;
  const int kslab = nz > 1 ? (((kcur + nz - 1) / nz + 127) / 128) * 128 : std::max(kcur, 1);
  hblock_kernel<<<dim3(nb, nb, nz), dim3(16, 16), 0, st>>>(prop, lay, b, d, kcur, kind, kfun,
                                                            sigma, H, kslab, part, tickets);
}

#ifdef RPC_SWEEP_PROBE  // debug aid (tools/sweep_probe.cu): per-block phase clocks
__device__ unsigned long long g_sweep_clk[32][4];
__device__ unsigned long long g_step_clk[256][4];
#define STEP_CLK_ON(i, k)                            \
  {                                                  \
    if (lane == 0) g_step_clk[i][k] = clock64();     \
    __syncwarp();                                    \
  }
#ifdef RPC_SWEEP_STEP_PROBE
#define STEP_CLK(i, k) STEP_CLK_ON(i, k)
#else
#define STEP_CLK(i, k)
#endif
#define SWEEP_CLK(blk, ph)                                   \
  {                                                          \
    if (threadIdx.x == 0) g_sweep_clk[blk][ph] = clock64(); \
    __syncwarp();                                            \
  }
#else
#define SWEEP_CLK(blk, ph)
#define STEP_CLK(i, k)
#endif

constexpr int kSweepThreads = 512;
constexpr int kSweepBlock = 16;

__device__ __forceinline__ int64_t tri(int p) { return (int64_t)p * (p + 1) / 2; }

// Blocked form of the reference's right-looking sweep with the identical per-entry
// operation sequence: every h_pq still receives  h_pq - l_c(p) l_c(q)  for the
// accepted steps c in sweep order, with the same two roundings, so the decisions,
// L and the accepted list are bit-identical to rpcholesky.hpp:174-199.
//   1. warp 0 runs the 16 decisions of a block on the 16x16 diagonal block only
//      (a decision needs h_ii, which depends only on in-block l values);
//   2. all threads form the accepted columns below the block (panel) row by row;
//   3. all threads apply the block's accepted rank-1 updates to the trailing
//      triangle, in acceptance order per entry.
// Three CTA barriers per 16 steps instead of two per step.
// Progress publication for the fused sweep + round-prep launch (sweep_prep_kernel): after
// every 16-step block the sweep CTA releases (epoch << 32) | accepted-count, with the block's
// L columns (lcol), positions (pos) and acceptance indices (aidx) written before; the final
// count carries bit 31.  The prep workers acquire it and run their substitutions behind the
// sweep.
struct SweepProgress {
  unsigned long long* prog;
  int* aidx;  // [b] acceptance index of proposal j, -1 if rejected
  unsigned epoch;
};

__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void sweep_body(
    const double* __restrict__ H, int b, uint64_t seed, uint64_t draw0,
    const double* __restrict__ prop, RecordLayout lay, int* __restrict__ pos,
    int64_t* __restrict__ acc_ids, double* __restrict__ lcol, double* __restrict__ lacc_cm,
    SweepOut* out, double* hp_global, int accept_all, const ScanStatus* pub_scan,
    char* pub_host, const SweepProgress* prg) {
  extern __shared__ double sm[];
  __shared__ int s_m, s_nacc, s_acc[kSweepBlock];
  __shared__ double s_root[kSweepBlock];
  __shared__ int s_pos[kMaxBlock];
  double* rdraw = sm;
  double* udiag = sm + b;
  double* lblk = sm + 2 * b;                       // [kSweepBlock][kSweepBlock] in-block l values
  double* lpan = lblk + kSweepBlock * kSweepBlock;  // [kSweepBlock][b] panel l values
  double* hp = hp_global ? hp_global : lpan + kSweepBlock * b;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int nwarps = kSweepThreads / 32;
  for (int p = warp; p < b; p += nwarps) {
#pragma unroll 4
    for (int q = lane; q <= p; q += 32) hp[tri(p) + q] = __ldg(H + (int64_t)p * b + q);
  }
  for (int i = tid; i < b; i += kSweepThreads) {
    // accept_all (block / simple RPCholesky): r = 0, so a row is kept iff h_ii > 0 — the
    // LLT success condition (Eigen fails on the first pivot <= 0)
    rdraw[i] = accept_all ? 0.0 : u01(splitmix64_draw(seed, draw0 + (uint64_t)i));
    udiag[i] = H[(int64_t)i * b + i];
    if (prg) prg->aidx[i] = -1;
  }
  if (tid == 0) s_m = 0;
  __syncthreads();
  for (int i0 = 0; i0 < b; i0 += kSweepBlock) {
    const int i1 = min(b, i0 + kSweepBlock);
    SWEEP_CLK(i0 / kSweepBlock, 0)
    // ---- 1. decisions on the diagonal block (warp 0, registers + shuffles) ----
    // The per-step critical path is  h_ii -> sqrt -> l_(i+1) = h_(i+1,i) / root ->
    // h_(i+1,i+1) -= l_(i+1)^2 -> next decision.  The next diagonal is therefore formed and
    // broadcast right after the division, ahead of the block's other rank-1 updates (lane
    // i+1 computes exactly the value its row update below produces), and the u_i r_i
    // products of the block are read before the chain starts.
    if (warp == 0) {
      int nacc = 0;
      const int p = i0 + lane;               // this lane's row inside the block
      const bool live = lane < kSweepBlock && p < i1;
      double row[kSweepBlock];               // h(p, i0 + q), q <= p - i0
#pragma unroll
      for (int q = 0; q < kSweepBlock; ++q)
        row[q] = (live && i0 + q <= p) ? hp[tri(p) + i0 + q] : 0.0;
      double ur[kSweepBlock];                // u_i * r_i (rounded), uniform across lanes
#pragma unroll
      for (int q = 0; q < kSweepBlock; ++q)
        ur[q] = i0 + q < i1 ? __dmul_rn(udiag[i0 + q], rdraw[i0 + q]) : 0.0;
      double hnext = __shfl_sync(0xffffffffu, row[0], 0);
#pragma unroll
      for (int ii = 0; ii < kSweepBlock; ++ii) {
        const int i = i0 + ii;
        if (i >= i1) break;
        STEP_CLK(i, 0)
        const double hii = hnext;                 // h(i, i) after the previous steps
        if (!(ur[ii] < hii)) {                    // uniform in the warp
          if (ii + 1 < kSweepBlock) hnext = __shfl_sync(0xffffffffu, row[ii + 1], ii + 1);
          continue;
        }
        const double root = __dsqrt_rn(hii);
        // lanes outside the column divide 1.0: a zero dividend would send them down the
        // division's slow path and leave the warp diverged for the shuffles below
        const bool own = live && p >= i;
        const double lp_div = __ddiv_rn(own ? row[ii] : 1.0, root);
        const double lp = own ? lp_div : 0.0;
        STEP_CLK(i, 2)
        __syncwarp();
        if (ii + 1 < kSweepBlock)
          hnext = __shfl_sync(0xffffffffu, __dsub_rn(row[ii + 1], __dmul_rn(lp, lp)), ii + 1);
        STEP_CLK(i, 3)
        if (live && p >= i) lblk[nacc * kSweepBlock + (p - i0)] = lp;
        __syncwarp();
        // lanes q's l values from the in-block store above (broadcast LDS.128 pairs instead of
        // 32-bit shuffles; read only where lane q was live), all loads issued before the
        // updates so they overlap instead of queueing behind one temporary register
        {
          const double2* lb2 = reinterpret_cast<const double2*>(lblk + nacc * kSweepBlock);
          double2 lqp[kSweepBlock / 2];
#pragma unroll
          for (int h = 0; h < kSweepBlock / 2; ++h)
            if (2 * h + 1 > ii) lqp[h] = lb2[h];
#pragma unroll
          for (int q = 0; q < kSweepBlock; ++q) {
            if (q <= ii) continue;
            const double lq = (q & 1) ? lqp[q >> 1].y : lqp[q >> 1].x;
            if (live && i0 + q <= p) row[q] = __dsub_rn(row[q], __dmul_rn(lp, lq));
          }
        }
        if (lane == 0) {
          s_acc[nacc] = i;
          s_root[nacc] = root;
        }
        STEP_CLK(i, 1)
        ++nacc;
      }
      if (lane == 0) s_nacc = nacc;
    }
    __syncthreads();
    SWEEP_CLK(i0 / kSweepBlock, 1)
    const int nacc = s_nacc;
    const int m0 = s_m;
    if (nacc > 0) {
      // ---- 2. panel: l_c(p) for rows p >= i1, accepted c in order ----
      // (the row's l values stay in registers and both loops are unrolled to the block
      // size, so the shared-memory operand loads issue ahead of the subtraction chain; the
      // operation sequence per entry is unchanged)
      for (int p = i1 + tid; p < b; p += kSweepThreads) {
        double lrow[kSweepBlock];
        const int64_t bp = tri(p);
#pragma unroll
        for (int k = 0; k < kSweepBlock; ++k) {
          if (k >= nacc) break;
          const int c = s_acc[k];
          double t = hp[bp + c];
#pragma unroll
          for (int k2 = 0; k2 < k; ++k2)
            t = __dsub_rn(t, __dmul_rn(lrow[k2], lblk[k2 * kSweepBlock + (c - i0)]));
          lrow[k] = __ddiv_rn(t, s_root[k]);
          lpan[k * b + p] = lrow[k];
        }
      }
      __syncthreads();
      // global L columns (c-th acceptance): rows in the block and below
      for (int idx = tid; idx < nacc * b; idx += kSweepThreads) {
        const int k = idx / b, j = idx % b, c = s_acc[k];
        if (j < c) continue;
        lcol[(int64_t)(m0 + k) * b + j] = j < i1 ? lblk[k * kSweepBlock + (j - i0)] : lpan[k * b + j];
      }
      SWEEP_CLK(i0 / kSweepBlock, 2)
      // ---- 3. trailing update, acceptance order per entry ----
      // Each lane carries four independent entries — rows p0, p0 + nwarps, columns q, q + 32 —
      // so four dependent subtract chains are in flight instead of one (the chain of a single
      // entry, not the FP64 throughput, bounded this phase: b = 120 probe 37.7k -> 31.6k
      // cycles; eight entries per lane or four columns of one row measured slower); each entry
      // still receives h - l_k(p) l_k(q) for the block's accepted steps k in order.
      for (int p0 = i1 + warp; p0 < b; p0 += 2 * nwarps) {
        const int p1 = p0 + nwarps;
        const bool v1 = p1 < b;
        const int pr1 = v1 ? p1 : p0;
        const int64_t b0 = tri(p0), b1 = tri(pr1);
        for (int q = i1 + lane; q <= pr1; q += 64) {
          const int q2 = q + 32, qb = q2 < b ? q2 : q;
          const bool e00 = q <= p0, e01 = q2 <= p0, e10 = v1 && q <= p1, e11 = v1 && q2 <= p1;
          double h00 = e00 ? hp[b0 + q] : 0.0, h01 = e01 ? hp[b0 + q2] : 0.0;
          double h10 = e10 ? hp[b1 + q] : 0.0, h11 = e11 ? hp[b1 + q2] : 0.0;
#pragma unroll 4
          for (int k = 0; k < nacc; ++k) {
            const double* lk = lpan + k * b;
            const double l0 = lk[p0], l1 = lk[pr1], la = lk[q], lb = lk[qb];
            h00 = __dsub_rn(h00, __dmul_rn(l0, la));
            h01 = __dsub_rn(h01, __dmul_rn(l0, lb));
            h10 = __dsub_rn(h10, __dmul_rn(l1, la));
            h11 = __dsub_rn(h11, __dmul_rn(l1, lb));
          }
          if (e00) hp[b0 + q] = h00;
          if (e01) hp[b0 + q2] = h01;
          if (e10) hp[b1 + q] = h10;
          if (e11) hp[b1 + q2] = h11;
        }
      }
      if (tid < nacc) {
        s_pos[m0 + tid] = s_acc[tid];
        if (prg) {
          pos[m0 + tid] = s_acc[tid];
          prg->aidx[s_acc[tid]] = m0 + tid;
        }
      }
      if (tid == 0) s_m = m0 + nacc;
    }
    __syncthreads();
    SWEEP_CLK(i0 / kSweepBlock, 3)
    // (warp 1 publishes: warp 0 goes straight on to the next block's decisions; the barrier
    // above ordered every thread's lcol / pos / aidx writes before this fence)
    if (prg && tid == 32 && (nacc > 0 || i1 == b)) {
      __threadfence();
      st_release_u64(prg->prog, ((unsigned long long)prg->epoch << 32) | (unsigned)s_m |
                                    (i1 == b ? 0x80000000u : 0u));
    }
  }
  const int m = s_m;
  for (int a = tid; a < m; a += kSweepThreads) {
    pos[a] = s_pos[a];
    acc_ids[a] = (int64_t)prop[(int64_t)s_pos[a] * lay.rec];
  }
  // chol_factor(a, c) = l(pos_a, pos_c)  (rpcholesky.hpp:192-199), column-major
  for (int idx = tid; idx < m * m; idx += kSweepThreads) {
    const int c = idx / m, a = idx % m;
    lacc_cm[idx] = (a >= c) ? lcol[(int64_t)c * b + s_pos[a]] : 0.0;
  }
  if (tid == 0) out->m = m;
  if (pub_host) {  // round status -> mapped pinned host memory: ScanStatus | SweepOut | ids
    ScanStatus* hs = reinterpret_cast<ScanStatus*>(pub_host);
    SweepOut* hw = reinterpret_cast<SweepOut*>(hs + 1);
    double* hpid = reinterpret_cast<double*>(hw + 1);
    int64_t* haid = reinterpret_cast<int64_t*>(hpid + b);
    if (tid == 0) {
      *hs = *pub_scan;
      hw->m = m;
    }
    for (int j = tid; j < b; j += kSweepThreads) {
      hpid[j] = prop[(int64_t)j * lay.rec];
      haid[j] = j < m ? (int64_t)prop[(int64_t)s_pos[j] * lay.rec] : 0;
    }
    if (prg) {
      // sequence word last: the host spins on it instead of waiting for the launch to end
      __syncthreads();
      if (tid == 0) {
        __threadfence_system();
        *reinterpret_cast<volatile int32_t*>(&hw->pad) = (int32_t)prg->epoch;
      }
    }
  }
}

__global__ void __launch_bounds__(kSweepThreads) sweep_kernel(
    const double* __restrict__ H, int b, uint64_t seed, uint64_t draw0,
    const double* __restrict__ prop, RecordLayout lay, int* __restrict__ pos,
    int64_t* __restrict__ acc_ids, double* __restrict__ lcol, double* __restrict__ lacc_cm,
    SweepOut* out, double* hp_global, int accept_all, const ScanStatus* pub_scan,
    char* pub_host) {
  sweep_body(H, b, seed, draw0, prop, lay, pos, acc_ids, lcol, lacc_cm, out, hp_global,
             accept_all, pub_scan, pub_host, nullptr);
}

void launch_sweep(const double* H, int b, uint64_t seed, uint64_t draw0, const double* prop,
                  RecordLayout lay, int* pos, int64_t* acc_ids, double* lcol, double* lacc_cm,
                  SweepOut* out, double* scratch_hp, cudaStream_t st, int accept_all,
                  const ScanStatus* pub_scan, char* pub_host) {
  const size_t packed = (size_t)b * (b + 1) / 2;
  size_t smem = sizeof(double) * (2 * (size_t)b + kSweepBlock * kSweepBlock + kSweepBlock * (size_t)b);
  double* hpg = nullptr;
  if (smem + packed * sizeof(double) <= 210 * 1024) {
    smem += packed * sizeof(double);
  } else {
    hpg = scratch_hp;  // global (L2-resident) fallback for large blocks
  }
  ensure_smem_attr((const void*)sweep_kernel, 214 * 1024);
  sweep_kernel<<<1, kSweepThreads, smem, st>>>(H, b, seed, draw0, prop, lay, pos, acc_ids, lcol,
                                                lacc_cm, out, hpg, accept_all, pub_scan,
                                                pub_host);
}

// L^{-1} by forward substitution L x = e_c, one warp per column c (8 columns per
// CTA), with L staged in shared memory (column-major, when it fits; else read from L2).
// No CTA-wide barriers inside the substitution, and no branches: each step loads the next
// column of L unconditionally (clamped rows) one step ahead of its use and applies the
// update as a select, so a step costs its dependency chain (FMA, multiply, shuffle) only
// (measured 78 -> 19 us at m = 116 against the branchy form, bitwise-identical results).
constexpr int kLinvWarps = 8;
template <int NQ>
__global__ void __launch_bounds__(32 * kLinvWarps) linv_kernel(const double* __restrict__ lacc_cm,
                                                               int m_host, const int* m_dev,
                                                               int nb, int64_t ldl, int koff,
                                                               int perm, int in_smem,
                                                               double* __restrict__ linv_rm) {
  extern __shared__ double smem_l[];  // column-major m x m copy when it fits
  const int m = m_dev ? *m_dev : m_host;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int c = blockIdx.x * kLinvWarps + warp;
  if ((int)blockIdx.x * kLinvWarps >= m) return;  // whole CTA beyond m (device-side m)
  const double* sL = lacc_cm;
  if (in_smem) {
    // independent 16-byte loads, eight in flight per thread (the copy is latency bound)
    const int n2 = (m * m) >> 1;
    const double2* src2 = reinterpret_cast<const double2*>(lacc_cm);
    double2* dst2 = reinterpret_cast<double2*>(smem_l);
    double2 buf[8];
    for (int i0 = tid; i0 < n2; i0 += 8 * (int)blockDim.x) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = i0 + u * (int)blockDim.x;
        if (i < n2) buf[u] = __ldg(src2 + i);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = i0 + u * (int)blockDim.x;
        if (i < n2) dst2[i] = buf[u];
      }
    }
    if (tid == 0 && ((m * m) & 1)) smem_l[m * m - 1] = lacc_cm[m * m - 1];
    __syncthreads();
    sL = smem_l;
  }
  if (c >= m) return;
  // lane owns rows a = lane + 32 q; reciprocals of its diagonal entries up front so the
  // serial substitution chain has no divisions.
  double x[NQ], rd[NQ], ln[NQ];
  int ar[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    const int a = lane + 32 * q;
    ar[q] = a < m ? a : m - 1;
    x[q] = (a == c) ? 1.0 : 0.0;
    rd[q] = 1.0 / sL[(int64_t)ar[q] * m + ar[q]];
    ln[q] = sL[(int64_t)c * m + ar[q]];
  }
  for (int t = c; t < m; ++t) {
    double lc[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) lc[q] = ln[q];
    const int tn = t + 1 < m ? t + 1 : t;
#pragma unroll
    for (int q = 0; q < NQ; ++q) ln[q] = sL[(int64_t)tn * m + ar[q]];
    const int ql = t >> 5, ll = t & 31;
    double xt_own = x[0] * rd[0];
#pragma unroll
    for (int q = 1; q < NQ; ++q) xt_own = (q == ql) ? x[q] * rd[q] : xt_own;
    const double xt = __shfl_sync(0xffffffffu, xt_own, ll);
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int a = lane + 32 * q;
      const double nx = fma(-lc[q], xt, x[q]);
      x[q] = (a == t) ? xt : ((a > t) ? nx : x[q]);
    }
  }
  const int col = linv_slot(c, m, koff, perm);
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    const int a = lane + 32 * q;
    if (a < nb) linv_rm[(int64_t)perm_row(a) * ldl + col] = (a >= c && a < m) ? x[q] : 0.0;
  }
  for (int a = lane + 32 * NQ; a < nb; a += 32) linv_rm[(int64_t)perm_row(a) * ldl + col] = 0.0;
}

// ---- round prep: L^{-1}, B' and the accepted operands in one launch ----------------
// Three independent roles over one grid, all reading the sweep's outputs (m on the device):
//   CTAs [0, nA)        : L^{-1} columns (as linv_kernel: one warp per column),
//   CTAs [nA, nA + nB)  : B' = -L^{-1} F_S by forward substitution L x = -F_S(:, k), one warp
//                         per column k (no dependency on L^{-1}, so it runs beside it),
//   CTAs [nA + nB, ...) : the accepted pivots' X rows (pre-scaled), norms and ids.
// Replaces linv -> gather -> bprime (three dependent launches) on the accelerated path.
template <int NQ>
__device__ __forceinline__ void warp_lower_solve(const double* sL, int m, int t0, double (&x)[NQ]) {
  const int lane = threadIdx.x & 31;
  double rd[NQ], ln[NQ];
  int ar[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    const int a = lane + 32 * q;
    ar[q] = a < m ? a : m - 1;
    rd[q] = 1.0 / sL[(int64_t)ar[q] * m + ar[q]];
    ln[q] = sL[(int64_t)t0 * m + ar[q]];
  }
  for (int t = t0; t < m; ++t) {
    double lc[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) lc[q] = ln[q];
    const int tn = t + 1 < m ? t + 1 : t;
#pragma unroll
    for (int q = 0; q < NQ; ++q) ln[q] = sL[(int64_t)tn * m + ar[q]];
    const int ql = t >> 5, ll = t & 31;
    double xt_own = x[0] * rd[0];
#pragma unroll
    for (int q = 1; q < NQ; ++q) xt_own = (q == ql) ? x[q] * rd[q] : xt_own;
    const double xt = __shfl_sync(0xffffffffu, xt_own, ll);
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int a = lane + 32 * q;
      const double nx = fma(-lc[q], xt, x[q]);
      x[q] = (a == t) ? xt : ((a > t) ? nx : x[q]);
    }
  }
}

template <int NQ>
__global__ void __launch_bounds__(32 * kLinvWarps) round_prep_kernel(
    const double* __restrict__ lacc_cm, int m_host, const int* m_dev, int nA, int nB, int nb,
    int64_t ldl, int koff, int in_smem, double* __restrict__ linv_rm,
    const double* __restrict__ prop, RecordLayout lay, const int* __restrict__ pos, int kcur,
    double* __restrict__ bp, int64_t ldbp, int dpad, double* __restrict__ xs,
    double* __restrict__ sqnS, double* __restrict__ idS, double xscale, int n_rows) {
  extern __shared__ double smem_l[];
  const int m = m_dev ? *m_dev : m_host;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int bid = blockIdx.x;
  if (bid >= nA + nB) {  // ---- operands of accepted pivot n (rows perm_row(n)), a warp each ----
    const int n = (bid - nA - nB) * kLinvWarps + warp;
    if (n >= n_rows) return;
    const int dst = perm_row(n);
    double* xr = xs + (int64_t)dst * dpad;
    if (n < m) {
      const double* rec = prop + (int64_t)pos[n] * lay.rec;
      for (int i = lane; i < dpad; i += 32) xr[i] = xscale * rec[lay.xoff + i];
      if (lane == 0) {
        sqnS[n] = rec[1];
        idS[n] = rec[0];
      }
    } else {
      for (int i = lane; i < dpad; i += 32) xr[i] = 0.0;
      if (lane == 0) {
        sqnS[n] = 0.0;
        idS[n] = -1.0;
      }
    }
    return;
  }
  const bool inv = bid < nA;
  const int c = inv ? bid * kLinvWarps + warp : 0;
  const int k = inv ? 0 : (bid - nA) * kLinvWarps + warp;
  if (m <= 0) return;
  if (inv && bid * kLinvWarps >= m) {
    // columns [m, round16(m)) of the last 16-column chunk the update reads: zeros
    if (c < ((m + 15) & ~15))
      for (int a = lane; a < nb; a += 32) linv_rm[(int64_t)perm_row(a) * ldl + linv_slot(c, m, koff, 1)] = 0.0;
    return;
  }
  const double* sL = lacc_cm;
  if (in_smem) {
    const int n2 = (m * m) >> 1;
    const double2* src2 = reinterpret_cast<const double2*>(lacc_cm);
    double2* dst2 = reinterpret_cast<double2*>(smem_l);
    double2 buf[8];
    for (int i0 = tid; i0 < n2; i0 += 8 * (int)blockDim.x) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = i0 + u * (int)blockDim.x;
        if (i < n2) buf[u] = __ldg(src2 + i);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = i0 + u * (int)blockDim.x;
        if (i < n2) dst2[i] = buf[u];
      }
    }
    if (tid == 0 && ((m * m) & 1)) smem_l[m * m - 1] = lacc_cm[m * m - 1];
    __syncthreads();
    sL = smem_l;
  }
  double x[NQ];
  if (inv) {
    if (c >= m) {
      if (c < ((m + 15) & ~15))
        for (int a = lane; a < nb; a += 32) linv_rm[(int64_t)perm_row(a) * ldl + linv_slot(c, m, koff, 1)] = 0.0;
      return;
    }
#pragma unroll
    for (int q = 0; q < NQ; ++q) x[q] = (lane + 32 * q == c) ? 1.0 : 0.0;
    warp_lower_solve<NQ>(sL, m, c, x);
    const int col = linv_slot(c, m, koff, 1);
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int a = lane + 32 * q;
      if (a < nb) linv_rm[(int64_t)perm_row(a) * ldl + col] = (a >= c && a < m) ? x[q] : 0.0;
    }
    for (int a = lane + 32 * NQ; a < nb; a += 32) linv_rm[(int64_t)perm_row(a) * ldl + col] = 0.0;
    return;
  }
  if (k >= kcur) return;
  // B'(:, k) = -L^{-1} F_S(:, k): forward substitution from the right-hand side -F_S(:, k)
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    const int a = lane + 32 * q;
    x[q] = a < m ? -__ldg(prop + (int64_t)pos[a] * lay.rec + lay.foff + k) : 0.0;
  }
  warp_lower_solve<NQ>(sL, m, 0, x);
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    const int a = lane + 32 * q;
    if (a < m) bp[(int64_t)perm_row(a) * ldbp + k] = x[q];
  }
  for (int a = m + lane; a < n_rows; a += 32) bp[(int64_t)perm_row(a) * ldbp + k] = 0.0;
}

template <int NQ>
static void prep_launch(const double* lacc_cm, int m_host, const int* m_dev, int m_max, int nb,
                        int64_t ldl, int koff, double* linv_rm, const double* prop,
                        RecordLayout lay, const int* pos, int kcur, double* bp, int64_t ldbp,
                        int dpad, double* xs, double* sqnS, double* idS, double xscale,
                        int n_rows, cudaStream_t st) {
  ensure_smem_attr((const void*)round_prep_kernel<NQ>, 200 * 1024);
  const size_t bytes = sizeof(double) * (size_t)m_max * m_max;
  const int in_smem = bytes <= 200 * 1024;
  const int nA = (((m_max + 15) & ~15) + kLinvWarps - 1) / kLinvWarps;  // through round16(m)
  const int nB = (kcur + kLinvWarps - 1) / kLinvWarps;
  const int nC = (n_rows + kLinvWarps - 1) / kLinvWarps;  // operand rows, a warp each
  // (every CTA of the launch reserves the L copy's shared memory: few operand CTAs keep the
  // whole grid in one wave)
  round_prep_kernel<NQ><<<nA + nB + nC, 32 * kLinvWarps, in_smem ? bytes : 0, st>>>(
      lacc_cm, m_host, m_dev, nA, nB, nb, ldl, koff, in_smem, linv_rm, prop, lay, pos, kcur, bp,
      ldbp, dpad, xs, sqnS, idS, xscale, n_rows);
}

void launch_round_prep(const double* lacc_cm, int m_host, const int* m_dev, int m_max, int nb,
                       int64_t ldl, int koff, double* linv_rm, const double* prop,
                       RecordLayout lay, const int* pos, int kcur, double* bp, int64_t ldbp,
                       int dpad, double* xs, double* sqnS, double* idS, double xscale,
                       int n_rows, cudaStream_t st) {
  if (m_max <= 0) return;
#define RPCB_PREP(NQ)                                                                         \
  prep_launch<NQ>(lacc_cm, m_host, m_dev, m_max, nb, ldl, koff, linv_rm, prop, lay, pos, kcur, \
                  bp, ldbp, dpad, xs, sqnS, idS, xscale, n_rows, st)
  if (m_max <= 32) RPCB_PREP(1);
  else if (m_max <= 64) RPCB_PREP(2);
  else if (m_max <= 128) RPCB_PREP(4);
  else RPCB_PREP(8);
#undef RPCB_PREP
}

// ---- fused sweep + round prep --------------------------------------------------------
// CTA 0 runs the sweep (sweep_body, publishing its progress after every 16-step block);
// every other warp of the grid runs one item of the round prep behind it:
//   items [0, kcur)             B'(:, k) = -L^{-1} F_S(:, k)   (forward substitution),
//   items [kcur, kcur + nc16)   L^{-1}(:, c), c = item - kcur   (c < round16(b)),
// then the accepted operand rows once the final count is out.  The substitution runs over
// proposal rows j (lane j & 31, slot j >> 5) instead of acceptance indices: accepted column c
// (position p_c) updates x_j for j > p_c with exactly the operations of warp_lower_solve
// (x_t = x_(p_c) * (1 / L_cc), x_j = fma(-L(j, c), x_t, x_j)), so B' and L^{-1} are the
// round_prep_kernel's bit for bit; rejected rows carry values nobody reads.  Columns arrive
// 16 at a time, so a warp's chain trails the sweep by one block and the prep work leaves
// the round's critical path (it ran after the sweep: ~25 us per C4 round).
struct PrepArgs {
  const double* lcol;
  int b;
  const double* prop;
  RecordLayout lay;
  int kcur;
  double* bp;
  int64_t ldbp;
  double* linv_rm;
  int64_t ldl;
  int nb;
  int dpad;
  double* xs;
  double* sqnS;
  double* idS;
  double xscale;
  int n_rows;
  const int* pos;
  const int* aidx;
  const unsigned long long* prog;
  unsigned epoch;
};

// lane 0 polls the progress word until at least `need` columns are out or the sweep is done;
// returns the count, `done` set with the final one
__device__ __forceinline__ int prep_wait(const PrepArgs& a, int need, bool& done) {
  unsigned long long v = 0;
  if ((threadIdx.x & 31) == 0) {
    for (;;) {
      v = ld_acquire_u64(a.prog);
      if ((unsigned)(v >> 32) == a.epoch &&
          ((int)(v & 0x7fffffffu) >= need || (v & 0x80000000ull)))
        break;
      __nanosleep(64);
    }
  }
  __syncwarp();
  v = __shfl_sync(0xffffffffu, v, 0);
  done = (v & 0x80000000ull) != 0;
  return (int)(v & 0x7fffffffu);
}

template <int NQ>
__device__ __forceinline__ void prep_solve(const PrepArgs& a, int item) {
  const int lane = threadIdx.x & 31;
  const bool inv = item >= a.kcur;
  const int c = inv ? item - a.kcur : 0, k = inv ? 0 : item;
  bool done = false;
  int avail = prep_wait(a, inv ? c + 1 : 1, done);
  double x[NQ];
  int t = 0;
  if (inv) {
    if (avail <= c) {  // c >= m: zero column inside the last 16-column chunk the update reads
      if (c < ((avail + 15) & ~15))
        for (int r = lane; r < a.nb; r += 32) a.linv_rm[(int64_t)perm_row(r) * a.ldl + kslot16(c)] = 0.0;
      return;
    }
    const int pc = __ldcg(a.pos + c);
#pragma unroll
    for (int q = 0; q < NQ; ++q) x[q] = (lane + 32 * q == pc) ? 1.0 : 0.0;
    t = c;
  } else {
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int j = lane + 32 * q;
      x[q] = j < a.b ? -__ldg(a.prop + (int64_t)j * a.lay.rec + a.lay.foff + k) : 0.0;
    }
  }
  constexpr int kB = 8;  // columns whose loads are issued together
  for (;;) {
    if (t >= avail) {
      if (done) break;
      avail = prep_wait(a, t + 1, done);
      if (t >= avail) break;
    }
    while (t < avail) {
      const int nbt = min(kB, avail - t);
      int pp[kB];
      double dd[kB], lc[kB][NQ];
#pragma unroll
      for (int u = 0; u < kB; ++u) pp[u] = u < nbt ? __ldcg(a.pos + t + u) : 0;
#pragma unroll
      for (int u = 0; u < kB; ++u) {
        const double* col = a.lcol + (int64_t)(t + u) * a.b;
        dd[u] = u < nbt ? __ldcg(col + pp[u]) : 1.0;
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
          const int j = lane + 32 * q;
          lc[u][q] = (u < nbt && j < a.b) ? __ldcg(col + j) : 0.0;
        }
      }
#pragma unroll
      for (int u = 0; u < kB; ++u) {
        if (u >= nbt) break;
        const double rd = 1.0 / dd[u];
        const int p = pp[u], ql = p >> 5;
        double own = x[0];
#pragma unroll
        for (int q = 1; q < NQ; ++q) own = (q == ql) ? x[q] : own;
        const double xt = __shfl_sync(0xffffffffu, own * rd, p & 31);
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
          const int j = lane + 32 * q;
          const double nx = fma(-lc[u][q], xt, x[q]);
          x[q] = (j == p) ? xt : ((j > p) ? nx : x[q]);
        }
      }
      t += nbt;
    }
  }
  const int m = avail;
  if (inv) {
    const int col = kslot16(c);
    for (int r = lane; r < a.nb; r += 32)
      if (r < c || r >= m) a.linv_rm[(int64_t)perm_row(r) * a.ldl + col] = 0.0;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int j = lane + 32 * q;
      const int r = j < a.b ? __ldcg(a.aidx + j) : -1;
      if (r >= c) a.linv_rm[(int64_t)perm_row(r) * a.ldl + col] = x[q];
    }
  } else {
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int j = lane + 32 * q;
      const int r = j < a.b ? __ldcg(a.aidx + j) : -1;
      if (r >= 0) a.bp[(int64_t)perm_row(r) * a.ldbp + k] = x[q];
    }
    for (int r = m + lane; r < a.n_rows; r += 32) a.bp[(int64_t)perm_row(r) * a.ldbp + k] = 0.0;
  }
}

__device__ __forceinline__ void prep_operand(const PrepArgs& a, int n) {
  const int lane = threadIdx.x & 31;
  bool done = false;
  const int m = prep_wait(a, 1 << 30, done);  // the final count
  const int dst = perm_row(n);
  double* xr = a.xs + (int64_t)dst * a.dpad;
  if (n < m) {
    const double* rec = a.prop + (int64_t)__ldcg(a.pos + n) * a.lay.rec;
    for (int i = lane; i < a.dpad; i += 32) xr[i] = a.xscale * rec[a.lay.xoff + i];
    if (lane == 0) {
      a.sqnS[n] = rec[1];
      a.idS[n] = rec[0];
    }
  } else {
    for (int i = lane; i < a.dpad; i += 32) xr[i] = 0.0;
    if (lane == 0) {
      a.sqnS[n] = 0.0;
      a.idS[n] = -1.0;
    }
  }
}

template <int NQ>
__global__ void __launch_bounds__(kSweepThreads) sweep_prep_kernel(
    const double* __restrict__ H, int b, uint64_t seed, uint64_t draw0,
    const double* __restrict__ prop, RecordLayout lay, int* __restrict__ pos,
    int64_t* __restrict__ acc_ids, double* __restrict__ lcol, double* __restrict__ lacc_cm,
    SweepOut* out, const ScanStatus* pub_scan, char* pub_host, SweepProgress prg, PrepArgs pa) {
  if (blockIdx.x == 0) {
    sweep_body(H, b, seed, draw0, prop, lay, pos, acc_ids, lcol, lacc_cm, out, nullptr, 0,
               pub_scan, pub_host, &prg);
    return;
  }
  const int nw = (gridDim.x - 1) * (kSweepThreads / 32);
  const int gw = (blockIdx.x - 1) * (kSweepThreads / 32) + (threadIdx.x >> 5);
  const int nitems = pa.kcur + ((b + 15) & ~15);
  for (int it = gw; it < nitems; it += nw) prep_solve<NQ>(pa, it);
  for (int n = nw - 1 - gw; n < pa.n_rows; n += nw) prep_operand(pa, n);
}

int launch_sweep_prep(const double* H, int b, uint64_t seed, uint64_t draw0, const double* prop,
                      RecordLayout lay, int* pos, int64_t* acc_ids, double* lcol,
                      double* lacc_cm, SweepOut* out, const ScanStatus* pub_scan,
                      char* pub_host, unsigned long long* prog, int* aidx, unsigned epoch,
                      int nb, int64_t ldl, double* linv_rm, int kcur, double* bp, int64_t ldbp,
                      int dpad, double* xs, double* sqnS, double* idS, double xscale,
                      int n_rows, cudaStream_t st) {
  if (b < 1 || b > 128) return -1;
  const size_t packed = (size_t)b * (b + 1) / 2;
  const size_t smem = sizeof(double) * (2 * (size_t)b + kSweepBlock * kSweepBlock +
                                        kSweepBlock * (size_t)b + packed);
  SweepProgress prg{prog, aidx, epoch};
  PrepArgs pa{lcol, b,      prop, lay,  kcur, bp,     ldbp, linv_rm, ldl,  nb,
              dpad, xs,     sqnS, idS,  xscale, n_rows, pos,  aidx,    prog, epoch};
  auto go = [&](auto kfn) -> int {
    if (ensure_smem_attr((const void*)kfn, (int)smem) != cudaSuccess) return -2;
    const int occ = cached_occupancy((const void*)kfn, kSweepThreads, smem, 1);
    const int items = kcur + ((b + 15) & ~15);
    const int want = 1 + std::max(1, (std::max(items, n_rows) + kSweepThreads / 32 - 1) /
                                         (kSweepThreads / 32));
    const int grid = std::min(want, occ * num_sms());
    if (grid < 2) return -3;
    void* args[] = {(void*)&H,   (void*)&b,       (void*)&seed,  (void*)&draw0,   (void*)&prop,
                    (void*)&lay, (void*)&pos,     (void*)&acc_ids, (void*)&lcol, (void*)&lacc_cm,
                    (void*)&out, (void*)&pub_scan, (void*)&pub_host, (void*)&prg,  (void*)&pa};
    // cooperative: every CTA co-resident, so the prep warps can wait on the sweep CTA
    return cudaLaunchCooperativeKernel((const void*)kfn, dim3(grid), dim3(kSweepThreads), args,
                                       smem, st) == cudaSuccess
               ? grid
               : -4;
  };
  if (b <= 32) return go(sweep_prep_kernel<1>);
  if (b <= 64) return go(sweep_prep_kernel<2>);
  return go(sweep_prep_kernel<4>);
}

template <int NQ>
static void linv_launch(const double* lacc_cm, int m_host, const int* m_dev, int m_max, int nb,
                        int64_t ldl, int koff, int perm, double* linv_rm, cudaStream_t st) {
  ensure_smem_attr((const void*)linv_kernel<NQ>, 200 * 1024);
  const size_t bytes = sizeof(double) * (size_t)m_max * m_max;
  const int in_smem = bytes <= 200 * 1024;
  linv_kernel<NQ><<<(m_max + kLinvWarps - 1) / kLinvWarps, 32 * kLinvWarps, in_smem ? bytes : 0, st>>>(
      lacc_cm, m_host, m_dev, nb, ldl, koff, perm, in_smem, linv_rm);
}

static void linv_dispatch(const double* lacc_cm, int m_host, const int* m_dev, int m_max, int nb,
                          int64_t ldl, int koff, int perm, double* linv_rm, cudaStream_t st) {
  if (m_max <= 32) linv_launch<1>(lacc_cm, m_host, m_dev, m_max, nb, ldl, koff, perm, linv_rm, st);
  else if (m_max <= 64) linv_launch<2>(lacc_cm, m_host, m_dev, m_max, nb, ldl, koff, perm, linv_rm, st);
  else if (m_max <= 128) linv_launch<4>(lacc_cm, m_host, m_dev, m_max, nb, ldl, koff, perm, linv_rm, st);
  else linv_launch<8>(lacc_cm, m_host, m_dev, m_max, nb, ldl, koff, perm, linv_rm, st);
}

void launch_linv(const double* lacc_cm, int m, int nb, int64_t ldl, int koff, double* linv_rm,
                 cudaStream_t st, int perm) {
  if (m <= 0) return;
  linv_dispatch(lacc_cm, m, nullptr, m, nb, ldl, koff, perm, linv_rm, st);
}

void launch_linv_dev(const double* lacc_cm, const int* m_dev, int m_max, int nb, int64_t ldl,
                     int koff, double* linv_rm, cudaStream_t st, int perm) {
  if (m_max <= 0) return;
  linv_dispatch(lacc_cm, 0, m_dev, m_max, nb, ldl, koff, perm, linv_rm, st);
}

}  // namespace rpcb

namespace rpcb {

__global__ void add_diag_shift_kernel(double* H, int b, double shift) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < b) H[(int64_t)i * b + i] += shift;
}

void launch_add_diag(double* H, int b, double shift, cudaStream_t st) {
  add_diag_shift_kernel<<<(b + 127) / 128, 128, 0, st>>>(H, b, shift);
}

__global__ void gather_records_kernel(const double* __restrict__ prop, int64_t rec, int64_t words,
                                      const int* __restrict__ idx, double* __restrict__ out) {
  const double* src = prop + (int64_t)idx[blockIdx.x] * rec;
  double* dst = out + (int64_t)blockIdx.x * rec;
  for (int64_t w = threadIdx.x; w < words; w += blockDim.x) dst[w] = src[w];
}

void launch_gather_records(const double* prop, int64_t rec, int64_t words, const int* idx, int m,
                           double* out, cudaStream_t st) {
  if (m > 0) gather_records_kernel<<<m, 256, 0, st>>>(prop, rec, words, idx, out);
}

}  // namespace rpcb
