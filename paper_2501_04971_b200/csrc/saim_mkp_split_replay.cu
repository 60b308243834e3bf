// saim_mkp_split_replay.cu -- exact-replay instantiations of the MKP row-split kernel
// (saim_mkp_split.cuh, RP = true; DESIGN.md 6.1 "Exact replay").
#include "saim_mkp_split.cuh"

namespace saim {
mkps_kernel_t mkps_replay_kernel_for(int MM, int M) { return mkps_kernel_for_t<true>(MM, M); }
}  // namespace saim
