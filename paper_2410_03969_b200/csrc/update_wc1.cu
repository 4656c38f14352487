// update_wc1.cu — instantiations for m <= 128: two warp groups of 4 warps per CTA
// (ping-pong), one warp column each (BM = 64 per group tile, no column padding).
#include "update_impl.cuh"

namespace rpcb {

int launch_update_wc1(const UpdateParams& p, int nf, cudaStream_t st) {
#define RPCB_CASE(N)                                                            \
  case N:                                                                       \
    return p.kind == kGaussGram ? launch_t<1, N, true, (N <= 6 ? 2 : 1), 2>(p, st)              \
                                : launch_t<1, N, false, (N <= 6 ? 2 : 1), 2>(p, st);
  switch (nf) {
    RPCB_CASE(1) RPCB_CASE(2) RPCB_CASE(3) RPCB_CASE(4) RPCB_CASE(5) RPCB_CASE(6) RPCB_CASE(7)
    RPCB_CASE(8) RPCB_CASE(9) RPCB_CASE(10) RPCB_CASE(11) RPCB_CASE(12) RPCB_CASE(13)
    RPCB_CASE(14) RPCB_CASE(15) RPCB_CASE(16)
  }
#undef RPCB_CASE
  return -1;
}

}  // namespace rpcb
