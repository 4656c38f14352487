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

namespace rpcb {

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
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// Row of a 16-row group used by fragment `f` (0/1) lane-group g (0..7):
// paired fragments interleave rows (stride 2) so that a half-warp touches
// rows {f, 2+f, 4+f, 6+f} whose swizzled chunks are all distinct.
__device__ __forceinline__ int frag_row(int g, int f, bool paired) {
  return paired ? (2 * g + f) : g;
}

// ---- reductions -----------------------------------------------------------
__device__ __forceinline__ double warp_sum_xor(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace rpcb
