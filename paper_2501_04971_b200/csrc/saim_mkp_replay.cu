// saim_mkp_replay.cu -- exact-replay instantiations of the MKP lockstep kernel (saim_mkp.cuh, RP =
// true; DESIGN.md 6.1 "Exact replay").  A separate translation unit so it compiles in parallel.
#include "saim_mkp.cuh"

namespace saim {
mkp_kernel_t mkp_replay_kernel_for(int MM, int M, bool prod) { return mkp_kernel_for_t<true>(MM, M, prod); }
}  // namespace saim
