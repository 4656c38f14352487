// sampling.cu — K1/K2: SplitMix64 counter draws, residual-diagonal scan and
// inverse-CDF proposal sampling; plus small utility kernels.
//
// Reference semantics (rng.hpp:67-96, rpcholesky.hpp:361-365): cumsum is the
// inclusive prefix of u; a draw maps r = next_double() to target = r * total,
// idx = first i with cumsum[i] > target, clamped to N-1, then walked back over
// a zero-weight plateau.  Draw j of round t is SplitMix64 counter 2*b*t + j.
//
// Fast mode replaces the strictly sequential scan by a fixed, p-invariant
// two-level sequence that is still a monotone prefix sum with the zero-plateau
// property (adding a zero weight never changes the running value):
//   global chunks of kChunk = 4096 rows; inside a chunk thread t owns rows
//   [16t, 16t+16) and runs s_e = s_{e-1} + u_e; thread bases B_0 = 0,
//   B_{t+1} = B_t + s_15(t) (serial); local_e = B_t + s_e; chunk offsets
//   off_0 = 0, chunk_end[c] = off_c + local_last(c), off_{c+1} = chunk_end[c];
//   cumsum_i = off_c + local_i.
// Every addition is one IEEE rounding, so cumsum differs from the reference's
// sequential sum only by association.  Replay mode runs the
// reference's exact sequential scan and std::upper_bound on one thread.
#include <climits>

#include "common.cuh"
#include "kernels.h"

namespace rpcb {

// Per-thread sequential partials and serial thread bases for one chunk.
// sh must hold kScanThreads + 1 doubles.  Returns this thread's base B_t.
__device__ __forceinline__ double chunk_scan_core(const double* __restrict__ uc, int n_valid,
                                                  double (&s)[16], double* sh) {
  const int t = threadIdx.x;
  const int e0 = t * 16;
  double acc = 0.0;
  if (e0 + 16 <= n_valid) {
    const double2* v2 = reinterpret_cast<const double2*>(uc + e0);
    double v[16];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const double2 w = __ldg(v2 + q);
      v[2 * q] = w.x;
      v[2 * q + 1] = w.y;
    }
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      acc = __dadd_rn(acc, v[e]);
      s[e] = acc;
    }
  } else {
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      const double v = (e0 + e < n_valid) ? __ldg(uc + e0 + e) : 0.0;
      acc = __dadd_rn(acc, v);
      s[e] = acc;
    }
  }
  sh[t] = acc;
  __syncthreads();
  if (t == 0) {
    double b = 0.0;
    for (int i = 0; i < kScanThreads; i += 8) {
      double tt[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) tt[q] = sh[i + q];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        sh[i + q] = b;
        b = __dadd_rn(b, tt[q]);
      }
    }
    sh[kScanThreads] = b;
  }
  __syncthreads();
  return sh[t];
}

// Also folds the previous update's per-tile ||G||^2 partials into this chunk's partial
// (tile_g2 != nullptr; same serial order as tile_to_chunk_kernel), saving a launch per round.
__global__ void __launch_bounds__(kScanThreads) chunk_totals_kernel(const double* __restrict__ u,
                                                                    int64_t n_loc,
                                                                    double* __restrict__ totals,
                                                                    const double* __restrict__ tile_g2,
                                                                    int n_tiles,
                                                                    double* __restrict__ chunk_g2,
                                                                    FusedPrefix fp,
                                                                    double* __restrict__ tb) {
  __shared__ double sh[kScanThreads + 1];
  const int c = blockIdx.x;
  const int64_t r0 = (int64_t)c * kChunk;
  const int n_valid = (int)lmin(kChunk, n_loc - r0);
  double s[16];
  const double base = chunk_scan_core(u + r0, n_valid, s, sh);
  if (tb) tb[(int64_t)c * kScanThreads + threadIdx.x] = sh[threadIdx.x + 1];  // B_(t+1)
  const int last = n_valid - 1;
  if (threadIdx.x == (last >> 4)) {
    double v = 0.0;
#pragma unroll
    for (int e = 0; e < 16; ++e)
      if (e == (last & 15)) v = s[e];
    totals[c] = __dadd_rn(base, v);
  }
  if (tile_g2) {
    // previous update's per-tile ||G||^2 partials of this chunk: loaded by 64 threads in
    // parallel, then summed in tile order by one thread (a dependent chain of global loads
    // was most of this kernel's time)
    constexpr int kTilesPerChunk = kChunk / 64;
    __shared__ double s_tg[kTilesPerChunk];
    const int t0 = c * kTilesPerChunk;
    const int t1 = min(n_tiles, t0 + kTilesPerChunk);
    if (threadIdx.x < kTilesPerChunk) s_tg[threadIdx.x] = t0 + (int)threadIdx.x < t1 ? tile_g2[t0 + threadIdx.x] : 0.0;
    __syncthreads();
    if (threadIdx.x == kScanThreads - 1) {
      double g = 0.0;
      for (int t = 0; t < t1 - t0; ++t) g = __dadd_rn(g, s_tg[t]);
      chunk_g2[c] = g;
    }
  }
  if (fp.counter) {
    // single shard: the last CTA to finish runs the serial chunk-offset chain of
    // chunk_prefix_kernel (same order, same results) — one launch fewer per round
    __shared__ int s_last;
    __shared__ double s_tot[kFusedPrefixMax], s_g2[kFusedPrefixMax];
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(fp.counter, 1u) == gridDim.x - 1;
    __syncthreads();
    if (s_last) {
      __threadfence();
      // stage with the whole CTA (loads in parallel), then the serial chain from smem
      for (int k = threadIdx.x; k < fp.n_chunks; k += blockDim.x) {
        s_tot[k] = __ldcg(totals + k);
        s_g2[k] = fp.g2_all ? __ldcg(fp.g2_all + k) : 0.0;
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        double off = 0.0, g2 = 0.0;
        for (int k = 0; k < fp.n_chunks; ++k) {
          off = __dadd_rn(off, s_tot[k]);
          s_tot[k] = off;
          g2 = __dadd_rn(g2, s_g2[k]);
        }
        fp.status->total = off;
        fp.status->g2_prev = g2;
        fp.status->exhausted = !(off > 0.0);
        *fp.counter = 0u;
      }
      __syncthreads();
      for (int k = threadIdx.x; k < fp.n_chunks; k += blockDim.x) fp.chunk_end[k] = s_tot[k];
    }
  }
}

void launch_chunk_totals(const double* u, int64_t n_loc, int n_chunks, double* totals,
                         cudaStream_t st, const double* tile_g2, int n_tiles, double* chunk_g2,
                         FusedPrefix fp, double* tb) {
  if (n_chunks > 0)
    chunk_totals_kernel<<<n_chunks, kScanThreads, 0, st>>>(u, n_loc, totals, tile_g2, n_tiles,
                                                           chunk_g2, fp, tb);
}

// One warp per chunk: lane l holds runs 8l .. 8l + 7 and tiles 2l, 2l + 1; the serial chains
// B_(t+1) = B_t + s_t and g = g + tile_g2 pass from lane to lane in order.
__global__ void __launch_bounds__(32) chunk_chain_kernel(const double* __restrict__ tsum,
                                                         const double* __restrict__ tile_g2,
                                                         int64_t n_loc, double* __restrict__ tb,
                                                         double* __restrict__ totals,
                                                         double* __restrict__ chunk_g2) {
  constexpr int kTiles = kChunk / 64;
  const int c = blockIdx.x, lane = threadIdx.x;
  const int64_t r0 = (int64_t)c * kChunk;
  const int nrun = (int)((lmin(kChunk, n_loc - r0) + 15) / 16);   // runs holding rows
  const int ntl = (int)((lmin(kChunk, n_loc - r0) + 63) / 64);    // tiles holding rows
  double v[8], gt[2];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int t = 8 * lane + i;
    v[i] = t < nrun ? __ldg(tsum + (int64_t)c * kScanThreads + t) : 0.0;
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int tl = 2 * lane + i;
    gt[i] = tl < ntl ? __ldg(tile_g2 + (int64_t)c * kTiles + tl) : 0.0;
  }
  double bsum = 0.0, gsum = 0.0;
  for (int L = 0; L < 32; ++L) {
    if (lane == L) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        bsum = __dadd_rn(bsum, v[i]);
        v[i] = bsum;
      }
      if (2 * L < ntl) gsum = __dadd_rn(gsum, gt[0]);
      if (2 * L + 1 < ntl) gsum = __dadd_rn(gsum, gt[1]);
    }
    bsum = __shfl_sync(0xffffffffu, bsum, L);
    gsum = __shfl_sync(0xffffffffu, gsum, L);
  }
  double2* o2 = reinterpret_cast<double2*>(tb + (int64_t)c * kScanThreads + 8 * lane);
#pragma unroll
  for (int i = 0; i < 4; ++i) o2[i] = make_double2(v[2 * i], v[2 * i + 1]);
  if (lane == 0) {
    totals[c] = bsum;
    chunk_g2[c] = gsum;
  }
}

void launch_chunk_chain(const double* tsum, const double* tile_g2, int64_t n_loc, int n_chunks,
                        double* tb, double* totals, double* chunk_g2, cudaStream_t st) {
  if (n_chunks > 0)
    chunk_chain_kernel<<<n_chunks, 32, 0, st>>>(tsum, tile_g2, n_loc, tb, totals, chunk_g2);
}

// Serial chunk-offset chain (fixed order => p-invariant).  The totals are staged in
// shared memory by the whole CTA, one fixed-size tile at a time, so the single-thread
// chain never waits on HBM and any number of chunks (any N) fits; the chain carries
// across tiles in the same order, so the results do not depend on the tile size.
constexpr int kPrefixTile = 2048;
__global__ void __launch_bounds__(1024) chunk_prefix_kernel(const double* __restrict__ totals,
                                                            const double* g2_all, int n_chunks,
                                                            double* __restrict__ chunk_end,
                                                            ScanStatus* status) {
  __shared__ double st[kPrefixTile], sg[kPrefixTile];
  double off = 0.0, g2 = 0.0;  // live in thread 0
  for (int t0 = 0; t0 < n_chunks; t0 += kPrefixTile) {
    const int nt = min(kPrefixTile, n_chunks - t0);
    for (int c = threadIdx.x; c < nt; c += blockDim.x) {
      st[c] = totals[t0 + c];
      sg[c] = g2_all ? g2_all[t0 + c] : 0.0;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int c = 0; c < nt; ++c) {
        off = __dadd_rn(off, st[c]);
        st[c] = off;
        g2 = __dadd_rn(g2, sg[c]);
      }
    }
    __syncthreads();
    for (int c = threadIdx.x; c < nt; c += blockDim.x) chunk_end[t0 + c] = st[c];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    status->total = off;
    status->g2_prev = g2;
    status->exhausted = !(off > 0.0);
  }
}

void launch_chunk_prefix(const double* totals_all, const double* g2_all, int n_chunks,
                         double* chunk_end, ScanStatus* status, cudaStream_t st) {
  chunk_prefix_kernel<<<1, 1024, 0, st>>>(totals_all, g2_all, n_chunks, chunk_end, status);
}

// Copies the sampled point's record (id, ||x||^2, x, F row) into rec.
__device__ __forceinline__ void write_record(const SampleParams& p, int64_t lrow, double* rec) {
  if (threadIdx.x == 0) {
    rec[0] = (double)(p.row0 + lrow);
    rec[1] = p.sqn[lrow];
  }
  const double* xr = p.X + lrow * p.dpad;
  for (int i = threadIdx.x; i < p.dpad; i += blockDim.x) rec[p.lay.xoff + i] = xr[i];
  const double* fr = p.F + lrow * p.ldf;
  for (int k = threadIdx.x; k < p.kcur; k += blockDim.x) rec[p.lay.foff + k] = fr[k];
}

constexpr int kSampleStageMax = 4096;  // chunk ends staged in shared memory (N <= 16.7M)
__global__ void __launch_bounds__(kScanThreads) sample_kernel(SampleParams p) {
  __shared__ double sh[kScanThreads + 1];
  __shared__ int s_chunk, s_mode, s_owner, s_best;
  __shared__ double s_off, s_target;
  extern __shared__ double s_ends[];  // [nc] when staged
  const int j = blockIdx.x;
  const int nc = p.n_chunks_global;
  // the chunk ends go to shared memory in one parallel pass, so the draw's binary search
  // costs shared-memory latency per probe instead of a dependent L2 round trip
  const bool staged = nc <= kSampleStageMax;
  if (staged) {
    for (int c = threadIdx.x; c < nc; c += blockDim.x) s_ends[c] = p.chunk_end[c];
    __syncthreads();
  }
  const double* ends = staged ? s_ends : p.chunk_end;
  if (threadIdx.x == 0) {
    const double r = u01(splitmix64_draw(p.seed, p.draw0 + (uint64_t)j));
    const double total = ends[nc - 1];
    const double target = __dmul_rn(r, total);
    int lo = 0, hi = nc;  // upper_bound over chunk ends
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (target < ends[mid]) hi = mid; else lo = mid + 1;
    }
    int mode = 0;
    if (lo == nc) {  // clamp to N-1, then walk back over the zero plateau
      int c = nc - 1;
      while (c > 0 && ends[c] == ends[c - 1]) --c;
      lo = c;
      mode = 1;
    }
    int o = 0;
    while (o + 1 < p.n_shards && p.shard_chunk0[o + 1] <= lo) ++o;
    s_chunk = lo;
    s_mode = mode;
    s_target = target;
    s_off = lo ? ends[lo - 1] : 0.0;
    s_owner = o;
    s_best = mode ? -1 : INT_MAX;
    p.owner[j] = o;
  }
  __syncthreads();
  if (s_owner != p.shard) return;
  const int lc = s_chunk - p.chunk0;
  const int64_t r0 = (int64_t)lc * kChunk;
  const int n_valid = (int)lmin(kChunk, p.n_loc - r0);
  double s[16];
  const double base = chunk_scan_core(p.u + r0, n_valid, s, sh);
  const double off = s_off, target = s_target;
  const int e0 = threadIdx.x * 16;
  if (s_mode == 0) {
    int best = INT_MAX;
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      const double cum = __dadd_rn(off, __dadd_rn(base, s[e]));
      if (e0 + e < n_valid && cum > target && best == INT_MAX) best = e0 + e;
    }
    if (best != INT_MAX) atomicMin(&s_best, best);
  } else {
    int best = -1;
    double prev = __dadd_rn(off, base);
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      const double cum = __dadd_rn(off, __dadd_rn(base, s[e]));
      if (e0 + e < n_valid && cum > prev) best = e0 + e;
      prev = cum;
    }
    if (best >= 0) atomicMax(&s_best, best);
  }
  __syncthreads();
  int best = s_best;
  if (best == INT_MAX || best < 0) best = 0;  // unreachable when total > 0
  write_record(p, r0 + best, p.records + (int64_t)j * p.lay.rec);
}

// Same draws from the stored thread bases (p.tb): thread t of the drawn chunk knows where
// its 16-row run starts (B_t) and ends (B_(t+1)), so the run holding the first cumsum > target
// is found without rescanning the chunk (no 256-long base chain per draw); only that thread
// re-adds its 16 rows.  Identical result: the fast cumsum is monotone, cum_i =
// off + (B_t + s_e), and a run contains the first index above the target iff its end is
// above it and its start is not (plateau mode: iff its end exceeds its start).
__global__ void __launch_bounds__(kScanThreads) sample_tb_kernel(SampleParams p) {
  __shared__ int s_chunk, s_mode, s_owner, s_best;
  __shared__ double s_off, s_target;
  extern __shared__ double s_ends[];  // [nc] when staged (+ [nc] g2 partials, CTA 0, fused)
  const int j = blockIdx.x;
  const int nc = p.n_chunks_global;
  const bool staged = nc <= kSampleStageMax;
  if (p.totals) {
    // fused scan: the chunk offsets from the previous update's chunk totals, chained in
    // chunk_prefix_kernel's order by every CTA (thread 0, out of shared memory); draw 0's CTA
    // also chains the ||G||^2 partials and publishes the offsets and the round status
    double* s_g2 = s_ends + nc;
    for (int c = threadIdx.x; c < nc; c += blockDim.x) {
      s_ends[c] = __ldg(p.totals + c);
      if (j == 0) s_g2[c] = __ldg(p.chunk_g2 + c);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double off = 0.0;
      for (int c = 0; c < nc; ++c) {
        off = __dadd_rn(off, s_ends[c]);
        s_ends[c] = off;
      }
    } else if (j == 0 && threadIdx.x == 32) {
      double g2 = 0.0;
      for (int c = 0; c < nc; ++c) g2 = __dadd_rn(g2, s_g2[c]);
      s_g2[0] = g2;
    }
    __syncthreads();
    if (j == 0) {
      for (int c = threadIdx.x; c < nc; c += blockDim.x) p.chunk_end_out[c] = s_ends[c];
      if (threadIdx.x == 0) {
        p.status->total = s_ends[nc - 1];
        p.status->g2_prev = s_g2[0];
        p.status->exhausted = !(s_ends[nc - 1] > 0.0);
      }
    }
  } else if (staged) {
    for (int c = threadIdx.x; c < nc; c += blockDim.x) s_ends[c] = p.chunk_end[c];
    __syncthreads();
  }
  const double* ends = staged ? s_ends : p.chunk_end;
  if (threadIdx.x == 0) {
    const double r = u01(splitmix64_draw(p.seed, p.draw0 + (uint64_t)j));
    const double total = ends[nc - 1];
    const double target = __dmul_rn(r, total);
    int lo = 0, hi = nc;  // upper_bound over chunk ends
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (target < ends[mid]) hi = mid; else lo = mid + 1;
    }
    int mode = 0;
    if (lo == nc) {  // clamp to N-1, then walk back over the zero plateau
      int c = nc - 1;
      while (c > 0 && ends[c] == ends[c - 1]) --c;
      lo = c;
      mode = 1;
    }
    int o = 0;
    while (o + 1 < p.n_shards && p.shard_chunk0[o + 1] <= lo) ++o;
    s_chunk = lo;
    s_mode = mode;
    s_target = target;
    s_off = lo ? ends[lo - 1] : 0.0;
    s_owner = o;
    s_best = -1;
    p.owner[j] = o;
  }
  __syncthreads();
  if (s_owner != p.shard) return;
  const int lc = s_chunk - p.chunk0;
  const int64_t r0 = (int64_t)lc * kChunk;
  const int n_valid = (int)lmin(kChunk, p.n_loc - r0);
  const int t = threadIdx.x, e0 = 16 * t;
  const double* tbc = p.tb + (int64_t)lc * kScanThreads;
  const double bend = __ldg(tbc + t), bstart = t ? __ldg(tbc + t - 1) : 0.0;
  const double off = s_off, target = s_target;
  const double cend = __dadd_rn(off, bend), cstart = __dadd_rn(off, bstart);
  if (s_mode == 0) {
    if (e0 < n_valid && cend > target && !(t > 0 && cstart > target)) {
      double acc = 0.0;
      int best = -1;
      for (int e = 0; e < 16 && e0 + e < n_valid; ++e) {
        acc = __dadd_rn(acc, __ldg(p.u + r0 + e0 + e));
        if (__dadd_rn(off, __dadd_rn(bstart, acc)) > target) {
          best = e0 + e;
          break;
        }
      }
      s_best = best;  // one run qualifies
    }
  } else if (e0 < n_valid && cend > cstart) {
    atomicMax(&s_best, t);  // the last run with an increase
  }
  __syncthreads();
  if (s_mode != 0 && t == s_best) {
    double acc = 0.0, prev = cstart;
    int best = -1;
    for (int e = 0; e < 16 && e0 + e < n_valid; ++e) {
      acc = __dadd_rn(acc, __ldg(p.u + r0 + e0 + e));
      const double cum = __dadd_rn(off, __dadd_rn(bstart, acc));
      if (cum > prev) best = e0 + e;
      prev = cum;
    }
    s_best = best;
  }
  __syncthreads();
  int best = s_best;
  if (best < 0) best = 0;  // unreachable when total > 0
  write_record(p, r0 + best, p.records + (int64_t)j * p.lay.rec);
}

void launch_sample(const SampleParams& p, cudaStream_t st) {
  const int nc = p.n_chunks_global;
  const size_t smem = nc <= kSampleStageMax ? sizeof(double) * (size_t)nc : 0;
  if (p.tb) sample_tb_kernel<<<p.b, kScanThreads, p.totals ? 2 * smem : smem, st>>>(p);
  else sample_kernel<<<p.b, kScanThreads, smem, st>>>(p);
}

// ---- replay mode -----------------------------------------------------------
// The reference's strictly sequential scan (acc += w[i], rng.hpp:67-75) on one thread,
// fed from shared memory: while thread 0 runs the dependent add chain over block b, the
// other warps stage block b+1 from HBM and write block b-1's prefix out (coalesced), so
// the chain never waits on a global load.
constexpr int kReplayBlk = 1024;
__global__ void __launch_bounds__(256) replay_scan_kernel(const double* __restrict__ u, int64_t n,
                                                          double* __restrict__ cumsum,
                                                          ScanStatus* status) {
  __shared__ double in[2][kReplayBlk], out[2][kReplayBlk];
  const int64_t nblk = (n + kReplayBlk - 1) / kReplayBlk;
  const int tid = threadIdx.x;
  for (int i = tid; i < kReplayBlk; i += blockDim.x) in[0][i] = i < n ? __ldg(u + i) : 0.0;
  __syncthreads();
  double acc = 0.0;  // thread 0
  for (int64_t b = 0; b < nblk; ++b) {
    const int cur = (int)(b & 1);
    if (tid == 0) {
      const int nv = (int)lmin(kReplayBlk, n - b * kReplayBlk);
      const double* src = in[cur];
      double* dst = out[cur];
      int i = 0;
      for (; i + 16 <= nv; i += 16) {
        double v[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) v[q] = src[i + q];
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          acc = __dadd_rn(acc, v[q]);
          dst[i + q] = acc;
        }
      }
      for (; i < nv; ++i) {
        acc = __dadd_rn(acc, src[i]);
        dst[i] = acc;
      }
    } else if (tid >= 32) {
      const int t = tid - 32, nt = blockDim.x - 32;
      const int64_t nb0 = (b + 1) * kReplayBlk;  // stage the next block
      if (b + 1 < nblk)
        for (int i = t; i < kReplayBlk; i += nt) in[cur ^ 1][i] = nb0 + i < n ? __ldg(u + nb0 + i) : 0.0;
      if (b > 0) {  // write the previous block's prefix
        const int64_t pb0 = (b - 1) * kReplayBlk;
        for (int i = t; i < kReplayBlk; i += nt) cumsum[pb0 + i] = out[cur ^ 1][i];
      }
    }
    __syncthreads();
  }
  const int64_t lb0 = (nblk - 1) * kReplayBlk;  // last block
  for (int64_t i = tid; i < n - lb0; i += blockDim.x) cumsum[lb0 + i] = out[(nblk - 1) & 1][i];
  if (tid == 0) {
    status->total = acc;
    status->exhausted = !(acc > 0.0);
  }
}

void launch_replay_scan(const double* u, int64_t n, double* cumsum, ScanStatus* status,
                        cudaStream_t st) {
  replay_scan_kernel<<<1, 256, 0, st>>>(u, n, cumsum, status);
}

__global__ void replay_sample_kernel(SampleParams p, const double* __restrict__ cumsum) {
  __shared__ int64_t s_idx;
  __shared__ int s_owner;
  const int j = blockIdx.x;
  if (threadIdx.x == 0) {
    const int64_t n = p.n_global;
    const double total = cumsum[n - 1];
    const double target = __dmul_rn(u01(splitmix64_draw(p.seed, p.draw0 + (uint64_t)j)), total);
    int64_t lo = 0, hi = n;
    while (lo < hi) {
      const int64_t mid = lo + ((hi - lo) >> 1);
      if (target < cumsum[mid]) hi = mid; else lo = mid + 1;
    }
    int64_t idx = lo;
    if (idx >= n) idx = n - 1;
    while (idx > 0 && cumsum[idx] == cumsum[idx - 1]) --idx;
    // owner: the shard whose chunk range holds the drawn row
    const int64_t chunk = idx / kChunk;
    int o = 0;
    while (o + 1 < p.n_shards && p.shard_chunk0[o + 1] <= chunk) ++o;
    s_idx = idx;
    s_owner = o;
    p.owner[j] = o;
  }
  __syncthreads();
  if (s_owner != p.shard) return;
  write_record(p, s_idx - p.row0, p.records + (int64_t)j * p.lay.rec);
}

void launch_replay_sample(const SampleParams& p, const double* cumsum, cudaStream_t st) {
  replay_sample_kernel<<<p.b, 128, 0, st>>>(p, cumsum);
}

// ---- utilities ---------------------------------------------------------------
__global__ void tile_to_chunk_kernel(const double* __restrict__ tile_g2, int n_tiles,
                                     int tiles_per_chunk, int n_chunks,
                                     double* __restrict__ chunk_g2) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n_chunks) return;
  double s = 0.0;
  const int t0 = c * tiles_per_chunk;
  const int t1 = min(n_tiles, t0 + tiles_per_chunk);
  for (int t = t0; t < t1; ++t) s = __dadd_rn(s, tile_g2[t]);
  chunk_g2[c] = s;
}

void launch_tile_to_chunk(const double* tile_g2, int n_tiles, int tiles_per_chunk,
                          int n_chunks_local, double* chunk_g2, cudaStream_t st) {
  if (n_chunks_local > 0)
    tile_to_chunk_kernel<<<(n_chunks_local + 127) / 128, 128, 0, st>>>(
        tile_g2, n_tiles, tiles_per_chunk, n_chunks_local, chunk_g2);
}

__global__ void __launch_bounds__(256) fsq_chunks_kernel(const double* __restrict__ F,
                                                         int64_t ldf, int64_t n_loc, int k,
                                                         double* __restrict__ out) {
  __shared__ double sh[256];
  const int64_t r0 = (int64_t)blockIdx.x * kChunk;
  const int64_t r1 = lmin(n_loc, r0 + kChunk);
  double acc = 0.0;
  for (int64_t r = r0 + threadIdx.x; r < r1; r += 256) {
    const double* fr = F + r * ldf;
    double s = 0.0;
    for (int c = 0; c < k; ++c) s = __dadd_rn(s, __dmul_rn(fr[c], fr[c]));
    acc = __dadd_rn(acc, s);
  }
  sh[threadIdx.x] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < 256; ++i) t = __dadd_rn(t, sh[i]);
    out[blockIdx.x] = t;
  }
}

void launch_fsq_chunks(const double* F, int64_t ldf, int64_t n_loc, int k, int n_chunks_local,
                       double* chunk_out, cudaStream_t st) {
  if (n_chunks_local > 0)
    fsq_chunks_kernel<<<n_chunks_local, 256, 0, st>>>(F, ldf, n_loc, k, chunk_out);
}

__global__ void f_to_colmajor_kernel(const double* __restrict__ F, int64_t ldf, int64_t n_loc,
                                     int c0, int nc, double* __restrict__ out, int64_t ld_out) {
  __shared__ double tile[32][33];
  const int64_t rb = (int64_t)blockIdx.x * 32;
  const int cb = blockIdx.y * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t r = rb + i;
    const int c = cb + threadIdx.x;
    tile[i][threadIdx.x] = (r < n_loc && c < nc) ? F[r * ldf + c0 + c] : 0.0;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int c = cb + i;
    const int64_t r = rb + threadIdx.x;
    if (r < n_loc && c < nc) out[(int64_t)c * ld_out + r] = tile[threadIdx.x][i];
  }
}

void launch_f_to_colmajor(const double* F, int64_t ldf, int64_t n_loc, int c0, int nc,
                          double* out, int64_t ld_out, cudaStream_t st) {
  if (n_loc <= 0 || nc <= 0) return;
  dim3 grid((unsigned)((n_loc + 31) / 32), (unsigned)((nc + 31) / 32)), block(32, 8);
  f_to_colmajor_kernel<<<grid, block, 0, st>>>(F, ldf, n_loc, c0, nc, out, ld_out);
}

// src: this shard's rows, either row-major [n_loc][ld_src] or column-major
// [d][ld_src].  Output padded row-major X and ||x||^2 in ascending coordinate
// order without FMA contraction (oracle.hpp:252).  A CTA stages `rows` rows
// through shared memory so both the read and the padded write are coalesced; the
// row count shrinks with d so the tile fits, and very wide points (one row > the
// shared-memory budget) take the per-row kernel below.
constexpr int kPackRows = 64;
constexpr int kPackSmem = 200 * 1024;
__global__ void __launch_bounds__(256) pack_points_kernel(const double* __restrict__ src,
                                                          int64_t n_loc, int d, int64_t ld_src,
                                                          int src_row_major, int64_t dpad,
                                                          int rows, double* __restrict__ X,
                                                          double* __restrict__ sqn,
                                                          int* nonfinite) {
  extern __shared__ double tile[];  // [rows][dpad + 1] (odd stride: per-row reads of one
                                    // column by 32 lanes hit distinct banks)
  const int64_t r0 = (int64_t)blockIdx.x * rows;
  const int nr = (int)lmin(rows, n_loc - r0);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const int dp = (int)dpad, ts = dp + 1;
  bool bad = false;
  // (no 64-bit index divisions: a warp per row for row-major sources, whose rows are
  // contiguous, a warp per column for column-major ones)
  if (src_row_major) {
    for (int r = warp; r < nr; r += nw) {
      const double* sr = src + (r0 + r) * ld_src;
      for (int c = lane; c < dp; c += 32) {
        const double v = c < d ? __ldg(sr + c) : 0.0;
        bad |= !isfinite(v);
        tile[r * ts + c] = v;
      }
    }
  } else {
    for (int c = warp; c < dp; c += nw) {
      const double* sc = src + (int64_t)c * ld_src + r0;
      for (int r = lane; r < nr; r += 32) {
        const double v = c < d ? __ldg(sc + r) : 0.0;
        bad |= !isfinite(v);
        tile[r * ts + c] = v;
      }
    }
  }
  __syncthreads();
  for (int r = warp; r < nr; r += nw) {
    double* xr = X + (r0 + r) * dpad;
    for (int c = lane; c < dp; c += 32) xr[c] = tile[r * ts + c];
  }
  if (tid < nr) {
    double s = 0.0;
    for (int c = 0; c < d; ++c) {
      const double v = tile[tid * ts + c];
      s = __dadd_rn(s, __dmul_rn(v, v));
    }
    sqn[r0 + tid] = s;
  }
  if (bad && nonfinite) atomicOr(nonfinite, 1);
}

// One CTA per point for dpad beyond the shared-memory tile: copy (coalesced for row-major
// sources), then the ascending-order norm by one thread from the packed row.
__global__ void __launch_bounds__(256) pack_row_kernel(const double* __restrict__ src, int d,
                                                       int64_t ld_src, int src_row_major,
                                                       int64_t dpad, double* __restrict__ X,
                                                       double* __restrict__ sqn, int* nonfinite) {
  const int64_t r = blockIdx.x;
  bool bad = false;
  double* xr = X + r * dpad;
  for (int64_t c = threadIdx.x; c < dpad; c += blockDim.x) {
    double v = 0.0;
    if (c < d) v = src_row_major ? src[r * ld_src + c] : src[c * ld_src + r];
    bad |= !isfinite(v);
    xr[c] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int c = 0; c < d; ++c) s = __dadd_rn(s, __dmul_rn(xr[c], xr[c]));
    sqn[r] = s;
  }
  if (bad && nonfinite) atomicOr(nonfinite, 1);
}

void launch_pack_points(const double* src, int64_t n_loc, int d, int64_t ld_src,
                        int src_row_major, int64_t dpad, double* X, double* sqn,
                        int* nonfinite, cudaStream_t st) {
  if (n_loc <= 0) return;
  const int rows = (int)lmin(kPackRows, kPackSmem / (int64_t)(sizeof(double) * (dpad + 1)));
  if (rows < 1) {
    pack_row_kernel<<<(unsigned)n_loc, 256, 0, st>>>(src, d, ld_src, src_row_major, dpad, X, sqn,
                                                     nonfinite);
    return;
  }
  const size_t smem = sizeof(double) * rows * (size_t)(dpad + 1);
  ensure_smem_attr((const void*)pack_points_kernel, kPackSmem);
  pack_points_kernel<<<(unsigned)((n_loc + rows - 1) / rows), 256, smem, st>>>(
      src, n_loc, d, ld_src, src_row_major, dpad, rows, X, sqn, nonfinite);
}

__global__ void fill_kernel(double* p, int64_t n, double v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}

void launch_fill(double* p, int64_t n, double v, cudaStream_t st) {
  if (n > 0) fill_kernel<<<(unsigned)lmin(4096, (n + 255) / 256), 256, 0, st>>>(p, n, v);
}

}  // namespace rpcb
