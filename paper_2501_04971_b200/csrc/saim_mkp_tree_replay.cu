// saim_mkp_tree_replay.cu -- exact-replay instantiations of the MKP outcome-tree kernel
// (saim_mkp_tree.cuh, RP = true; DESIGN.md 6.1 "Exact replay").
#include "saim_mkp_tree.cuh"

namespace saim {
mkpt_kernel_t mkpt_replay_kernel_for(int MM, int M, int L) { return mkpt_kernel_for_t<true>(MM, M, L); }
}  // namespace saim
