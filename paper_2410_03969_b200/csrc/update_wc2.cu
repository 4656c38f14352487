// update_wc2.cu — instantiations for 128 < m <= 256 (one CTA per SM) and 64 < m <= 96 (two
// CTAs per SM): one warp group of 8 warps, two warp columns (BM = 64).
#include "update_impl.cuh"

namespace rpcb {

int launch_update_wc2(const UpdateParams& p, int nfw, cudaStream_t st) {
#define RPCB_CASE(N, MB)                                                        \
  case N:                                                                       \
    return p.kind == kGaussGram ? launch_t<2, N, true, MB, 1>(p, st) : launch_t<2, N, false, MB, 1>(p, st);
  switch (nfw) {
    RPCB_CASE(9, 1) RPCB_CASE(10, 1)
    RPCB_CASE(11, 1) RPCB_CASE(12, 1) RPCB_CASE(13, 1) RPCB_CASE(14, 1) RPCB_CASE(15, 1)
    RPCB_CASE(16, 1)
  }
#undef RPCB_CASE
  return -1;
}

}  // namespace rpcb
