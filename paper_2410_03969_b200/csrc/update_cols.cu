// update_cols.cu — standalone K5 (kernel columns A(:, S), m <= 128) instantiations: the
// fused update kernel compiled with only its kernel-column phase, two warp groups of 4
// warps, and two CTAs per SM where registers allow (bench_column_throughput,
// rpc_kernel_columns).
#include "update_impl.cuh"

namespace rpcb {

int launch_update_cols(const UpdateParams& p, int nf, cudaStream_t st) {
#define RPCB_CASE(N)                                                                          \
  case N:                                                                                     \
    return p.kind == kGaussGram ? launch_t<1, N, true, (N <= 8 ? 2 : 1), 2, true>(p, st)                   \
                                : launch_t<1, N, false, (N <= 8 ? 2 : 1), 2, true>(p, st);
  if (nf <= 8 || p.kind != kGaussGram) {
    switch (nf) {
      RPCB_CASE(1) RPCB_CASE(2) RPCB_CASE(3) RPCB_CASE(4) RPCB_CASE(5) RPCB_CASE(6) RPCB_CASE(7)
      RPCB_CASE(8) RPCB_CASE(9) RPCB_CASE(10) RPCB_CASE(11) RPCB_CASE(12) RPCB_CASE(13)
      RPCB_CASE(14) RPCB_CASE(15) RPCB_CASE(16)
    }
  }
#undef RPCB_CASE
  // Gram, 8 < nf <= 16: one group of 8 warps in two warp columns (half the accumulators per
  // warp), two CTAs per SM
#define RPCB_CASE2(N) \
  case N:             \
    return launch_t<2, N, true, 2, 1, true>(p, st);
  switch ((nf + 1) / 2) {
    RPCB_CASE2(5) RPCB_CASE2(6) RPCB_CASE2(7) RPCB_CASE2(8)
  }
#undef RPCB_CASE2
  return -1;
}

}  // namespace rpcb
