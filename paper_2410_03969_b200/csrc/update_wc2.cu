// update_wc2.cu — instantiations: two warp columns, BM = 64: two CTAs per SM for
// m <= 128 (even fragment counts), one CTA per SM for 128 < m <= 256.
#include "update_impl.cuh"

namespace rpcb {

int launch_update_wc2(const UpdateParams& p, int nfw, cudaStream_t st) {
#define RPCB_CASE(N, MB)                                                        \
  case N:                                                                       \
    return p.kind == kGaussGram ? launch_t<2, N, true, MB>(p, st) : launch_t<2, N, false, MB>(p, st);
  switch (nfw) {
    RPCB_CASE(1, 2) RPCB_CASE(2, 2) RPCB_CASE(3, 2) RPCB_CASE(4, 2) RPCB_CASE(5, 2)
    RPCB_CASE(6, 2) RPCB_CASE(7, 2) RPCB_CASE(8, 2) RPCB_CASE(9, 1) RPCB_CASE(10, 1)
    RPCB_CASE(11, 1) RPCB_CASE(12, 1) RPCB_CASE(13, 1) RPCB_CASE(14, 1) RPCB_CASE(15, 1)
    RPCB_CASE(16, 1)
  }
#undef RPCB_CASE
  return -1;
}

}  // namespace rpcb
