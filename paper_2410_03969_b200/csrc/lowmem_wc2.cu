// lowmem_wc2.cu — low-memory update instantiations for 128 < m <= 256, and for any m when
// the two-group configuration's resident X tiles do not fit (large d): one group of 8 warps,
// two warp columns (64-row tiles).
#include "lowmem_impl.cuh"

namespace rpcb {

int launch_lowmem_wc2(const LowmemParams& p, int nfw, cudaStream_t st) {
#define RPCB_CASE(N)                                                                          \
  case N:                                                                                     \
    return p.kind == kGaussGram ? launch_lowmem_t<2, N, true, 1>(p, st)                       \
                                : launch_lowmem_t<2, N, false, 1>(p, st);
  switch (nfw) {
    RPCB_CASE(1) RPCB_CASE(2) RPCB_CASE(3) RPCB_CASE(4) RPCB_CASE(5) RPCB_CASE(6) RPCB_CASE(7)
    RPCB_CASE(8) RPCB_CASE(9) RPCB_CASE(10) RPCB_CASE(11) RPCB_CASE(12) RPCB_CASE(13)
    RPCB_CASE(14) RPCB_CASE(15) RPCB_CASE(16)
  }
#undef RPCB_CASE
  return -1;
}

}  // namespace rpcb
