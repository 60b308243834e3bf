// saim_mkp_spec_replay.cu -- exact-replay instantiations of the speculative sub-warp MKP kernel
// (saim_mkp_spec.cuh, RP = true; DESIGN.md 6.1 "Exact replay").
#include "saim_mkp_spec.cuh"

namespace saim {
mkpx_kernel_t mkpx_replay_kernel_for(int MM, int M, int G) { return mkpx_kernel_for_t<true>(MM, M, G); }
}  // namespace saim
