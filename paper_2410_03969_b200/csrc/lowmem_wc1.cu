// lowmem_wc1.cu — low-memory update instantiations for m <= 128: two warp groups of
// 4 warps per CTA, one warp column each (64-row tiles).
#include "lowmem_impl.cuh"

namespace rpcb {

int launch_lowmem_wc1(const LowmemParams& p, int nf, cudaStream_t st) {
#define RPCB_CASE(N)                                                                          \
  case N:                                                                                     \
    return p.kind == kGaussGram ? launch_lowmem_t<1, N, true, 2, (N <= 4 ? 2 : 1)>(p, st)     \
                                : launch_lowmem_t<1, N, false, 2, (N <= 4 ? 2 : 1)>(p, st);
  switch (nf) {
    RPCB_CASE(1) RPCB_CASE(2) RPCB_CASE(3) RPCB_CASE(4) RPCB_CASE(5) RPCB_CASE(6) RPCB_CASE(7)
    RPCB_CASE(8) RPCB_CASE(9) RPCB_CASE(10) RPCB_CASE(11) RPCB_CASE(12) RPCB_CASE(13)
    RPCB_CASE(14) RPCB_CASE(15) RPCB_CASE(16)
  }
#undef RPCB_CASE
  return -1;
}

}  // namespace rpcb
