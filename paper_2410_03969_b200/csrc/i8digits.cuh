// i8digits.cuh — F's int8 digit planes: layout and the per-group append used
// by the update kernel's epilogue (update_impl.cuh) and by slice_cols_kernel (i8gemm.cu).
//   planes[t][blk][row][64]: digit t of F(row, 64 blk + j), kcap / 64 blocks, plane stride
//   pstride = (kcap / 64) * plane_rows * 64, block stride bstride = plane_rows * 64.
//   V = rint(F 2^48) (|F| <= 1); d_0 = V >> 42 (signed, |d_0| <= 64), d_1 .. d_6 the unsigned
//   7-bit chunks below it: F = sum_t d_t 2^(-6 - 7 t) within 2^-49.
#pragma once
#include <cstdint>

#include "kernels.h"

namespace rpcb {

// Digits of F(r, 8 g .. 8 g + 7) for the columns in [c0, c1) into the planes (one 64-bit store
// per plane); bytes of columns below c0 are kept (earlier rounds'), those from c1 on are
// don't-care (the next round rewrites them).  frow: F's row r.
__device__ __forceinline__ void i8_append_group(const double* frow, int64_t r, int g, int c0,
                                                int c1, int8_t* planes, int64_t pstride,
                                                int64_t bstride) {
  int8_t* base = planes + (int64_t)(g >> 3) * bstride + r * 64 + 8 * (g & 7);
  uint32_t wl[kI8Slices], wh[kI8Slices];
  const bool head = 8 * g < c0;
#pragma unroll
  for (int t = 0; t < kI8Slices; ++t) {
    uint64_t w = head ? *reinterpret_cast<const uint64_t*>(base + t * pstride) : 0ull;
    wl[t] = (uint32_t)w;
    wh[t] = (uint32_t)(w >> 32);
  }
  // the group's 64 bytes of F as two 256-bit loads (F rows are 128-byte aligned and padded to
  // 16 columns, so the whole group is readable); entries outside [c0, c1) are not used
  double v[8];
  asm volatile("ld.global.cg.v4.f64 {%0, %1, %2, %3}, [%4];"
               : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3])
               : "l"(frow + 8 * g));
  asm volatile("ld.global.cg.v4.f64 {%0, %1, %2, %3}, [%4];"
               : "=d"(v[4]), "=d"(v[5]), "=d"(v[6]), "=d"(v[7])
               : "l"(frow + 8 * g + 4));
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const int c = 8 * g + e;
    if (!(c >= c0 && c < c1)) v[e] = 0.0;
  }
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const int c = 8 * g + e;
    if (c < c0) continue;
    const double q = fma(v[e], 281474976710656.0, 6755399441055744.0);  // v 2^48 + 1.5 2^52
    const long long V = __double_as_longlong(q) - 0x4338000000000000LL;
    const uint32_t lo = (uint32_t)V, hi = (uint32_t)((unsigned long long)V >> 32);
    uint32_t dg[kI8Slices];
    dg[6] = lo & 127u;
    dg[5] = (lo >> 7) & 127u;
    dg[4] = (lo >> 14) & 127u;
    dg[3] = (lo >> 21) & 127u;
    dg[2] = __funnelshift_r(lo, hi, 28) & 127u;
    dg[1] = (hi >> 3) & 127u;
    dg[0] = (uint32_t)((int)hi >> 10) & 0xffu;  // V >> 42, two's complement byte
    const int sh = 8 * (e & 3);
#pragma unroll
    for (int t = 0; t < kI8Slices; ++t) {
      if (e < 4) wl[t] = (wl[t] & ~(0xffu << sh)) | (dg[t] << sh);
      else wh[t] = (wh[t] & ~(0xffu << sh)) | (dg[t] << sh);
    }
  }
#pragma unroll
  for (int t = 0; t < kI8Slices; ++t)
    *reinterpret_cast<uint64_t*>(base + t * pstride) = ((uint64_t)wh[t] << 32) | wl[t];
}

}  // namespace rpcb
