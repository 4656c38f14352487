// common.cuh — shared device helpers for the B200 accelerated-RPCholesky path.
//
// Layout conventions:
//   * X shard   : [n_loc][dpad] row-major fp64, dpad = d rounded up to 16 (zero pad)
//   * F shard   : [n_loc][ldf]  row-major fp64, ldf even (16-byte rows); only
//                 columns < kcur are ever read (loads beyond kcur are zero-filled)
//   * u shard   : [n_loc] residual diagonal
//   * staged tiles in shared memory are [rows][16 doubles] = 128-byte rows with
//     the TMA 128B swizzle (16-byte chunk c of row r stored at chunk c ^ (r & 7)),
//     read by DMMA fragments with the stride-2 row map (see frag_row) that makes
//     every 64-bit fragment load bank-conflict free.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include <map>
#include <mutex>
#include <tuple>

namespace rpcb {

// ---- per-device launch settings (host) --------------------------------------
// cudaFuncSetAttribute is per device, so the opt-in to > 48 KB of dynamic shared memory,
// the occupancy that sizes persistent grids and the SM count are cached per (kernel,
// device[, smem]) under one mutex: several contexts on different GPUs may launch from
// different threads of one process (rpchol_b200.hpp).
struct LaunchCache {
  std::mutex mu;
  std::map<std::tuple<const void*, int, size_t>, int> occ;
  std::map<std::pair<const void*, int>, int> smem;
  std::map<int, int> sms;
};
inline LaunchCache& launch_cache() {
  static LaunchCache c;
  return c;
}
inline int current_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev;
}
// Raise the kernel's dynamic shared-memory limit on the current device to at least `bytes`.
inline cudaError_t ensure_smem_attr(const void* fn, int bytes) {
  if (bytes <= 48 * 1024) return cudaSuccess;
  LaunchCache& c = launch_cache();
  std::lock_guard<std::mutex> lk(c.mu);
  int& have = c.smem[{fn, current_device()}];
  if (have >= bytes) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) have = bytes;
  return e;
}
// Resident CTAs per SM for (kernel, threads, smem) on the current device (>= 1).
inline int cached_occupancy(const void* fn, int threads, size_t smem, int fallback) {
  LaunchCache& c = launch_cache();
  std::lock_guard<std::mutex> lk(c.mu);
  auto key = std::make_tuple(fn, current_device(), smem);
  auto it = c.occ.find(key);
  if (it != c.occ.end()) return it->second;
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, threads, smem) != cudaSuccess ||
      occ < 1) {
    cudaGetLastError();
    occ = fallback;
  }
  c.occ[key] = occ;
  return occ;
}
inline int num_sms() {
  LaunchCache& c = launch_cache();
  std::lock_guard<std::mutex> lk(c.mu);
  const int dev = current_device();
  int& n = c.sms[dev];
  if (!n) {
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

constexpr int kChunk = 4096;       // rows per scan chunk (global, p-invariant)
constexpr int kScanThreads = 256;  // 16 elements per thread
constexpr int kBK = 16;            // k-extent of one staged tile (128 B rows)

__host__ __device__ __forceinline__ int64_t lmin(int64_t a, int64_t b) { return a < b ? a : b; }

// ---- SplitMix64 (reference rng.hpp:27-42), counter form -------------------
__host__ __device__ __forceinline__ uint64_t splitmix64_draw(uint64_t seed, uint64_t n) {
  uint64_t z = seed + (n + 1) * 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ double u01(uint64_t z) {
  return (double)(z >> 11) * 0x1.0p-53;
}

// ---- shared-memory tile addressing (128B swizzle, TMA-compatible) ---------
// byte offset of element (row, k) in a [rows][16] fp64 tile
__device__ __forceinline__ uint32_t swz_off(int row, int k) {
  const int chunk = (k >> 1) ^ (row & 7);
  return (uint32_t)(row * 128 + chunk * 16 + (k & 1) * 8);
}

// ---- cp.async (LDGSTS) with zero fill --------------------------------------
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
  const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem),
               "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// ---- FP64 tensor core: DMMA 8x8x4 ------------------------------------------
// D(8x8) += A(8x4, row) * B(4x8, col); lane l holds A[l/4][l%4], B[l%4][l/4],
// C[l/4][2(l%4)], C[l/4][2(l%4)+1].
__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

// Row of a 16-row group used by fragment `f` (0/1) lane-group g (0..7):
// paired fragments interleave rows (stride 2) so that a half-warp touches
// rows {f, 2+f, 4+f, 6+f} whose swizzled chunks are all distinct.
__device__ __forceinline__ int frag_row(int g, int f, bool paired) {
  return paired ? (2 * g + f) : g;
}

// Position of logical row n8 (0..7) inside its 8-row group in shared memory:
// {0,1,2,3} -> {0,2,4,6}, {4,5,6,7} -> {1,3,5,7}.  A half-warp's fragment rows
// then have distinct (row & 7) >> 1, so the 128B-swizzled fp64 fragment loads
// of a DMMA m8n8k4 operand are bank-conflict free.
__host__ __device__ __forceinline__ int perm8(int n8) { return n8 < 4 ? 2 * n8 : 2 * (n8 - 4) + 1; }
__host__ __device__ __forceinline__ int perm_row(int n) { return (n & ~7) + perm8(n & 7); }

// ---- mbarrier + TMA (sm_90+/sm_100a) ----------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      "selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// Non-blocking probe of a phase (no suspend): lets a consumer check the next stage's
// barrier while its DMMAs for the current stage are still in flight.
__device__ __forceinline__ bool mbar_test_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      "selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// The retry loop is plain C++ so the compiler sees the branch and reconverges the
// warp before any following .aligned instruction (mma.sync, shfl.sync).
// One lane of the (converged) warp.  Single-thread TMA / MMA roles run under elect.sync so the
// compiler knows one lane is active and keeps addresses and descriptors in uniform registers
// (an `if (lane == 0)` region gets an election loop and broadcast moves around every TMA or
// MMA instruction).
__device__ __forceinline__ bool elect_one() {
  uint32_t p;
  asm volatile(
      "{\n.reg .pred P;\nelect.sync _|P, 0xffffffff;\nselp.u32 %0, 1, 0, P;\n}\n"
      : "=r"(p));
  return p != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}
// 2D tiled TMA load: box at (c0 = inner element, c1 = row) into shared memory,
// completion signalled on `bar` via complete_tx.
__device__ __forceinline__ void tma_load_2d(void* smem_dst, const void* tmap, int c0, int c1,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];\n" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_prefetch_desc(const void* tmap) {
  asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(tmap)) : "memory");
}
// Generic-proxy global writes made visible to later async-proxy (TMA) reads.
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;\n" ::: "memory");
}
__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ void named_bar_arrive(int id, int nthreads) {
  asm volatile("bar.arrive %0, %1;\n" ::"r"(id), "r"(nthreads) : "memory");
}

// ---- reductions -----------------------------------------------------------
__device__ __forceinline__ double warp_sum_xor(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace rpcb
