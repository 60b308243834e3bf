// saim_qkp_replay.cu -- instantiations of the QKP exact-replay kernel (saim_qkp.cuh, RP = true):
// the replicas whose run met a decision the fp64 level could not certify are re-run with the
// double-double level (R18, 6.1 "Exact replay").  A separate translation unit so the
// two kernel families compile in parallel.
#undef SAIM_PROF
#include "saim_qkp.cuh"

namespace saim {

typedef void (*qkp_kernel_t)(const RunArgs);

template <int NPL, int QB, bool PK>
static qkp_kernel_t pick_rp() { return saim_qkp_kernel<NPL, QB, PK, true>; }

qkp_kernel_t qkp_replay_kernel_for(int npl, int qb, int pk) {
#define SAIM_QKP_CASE(P)                                \
  if (npl <= P) return qb == 1 ? (pk ? pick_rp<P, 1, true>() : pick_rp<P, 1, false>()) : pick_rp<P, 2, false>();
  SAIM_QKP_CASE(1) SAIM_QKP_CASE(2) SAIM_QKP_CASE(3) SAIM_QKP_CASE(4) SAIM_QKP_CASE(6)
  SAIM_QKP_CASE(8) SAIM_QKP_CASE(10) SAIM_QKP_CASE(12) SAIM_QKP_CASE(16)
#undef SAIM_QKP_CASE
  return nullptr;
}

}  // namespace saim
