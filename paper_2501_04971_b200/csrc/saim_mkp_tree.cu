// saim_mkp_tree.cu -- launch planning of the MKP outcome-tree kernel (saim_mkp_tree.cuh).
#include "saim_mkp_tree.cuh"

namespace saim {

mkpt_kernel_t mkpt_replay_kernel_for(int MM, int M, int L);   // saim_mkp_tree_replay.cu
static mkpt_kernel_t mkpt_kernel_for(int MM, int M, int L) { return mkpt_kernel_for_t<false>(MM, M, L); }

// Plan for L lanes per replica: per-warp shared bytes and the largest warps-per-CTA that fit.
int mkpt_plan(int M, int N_max, int smem_optin, int MM, uint32_t blob_bytes, int L, uint32_t *per_warp, int *max_wpc) {
  mkpt_kernel_t k = mkpt_kernel_for(MM, M, L);
  if (!k) return -1;
  cudaFuncAttributes attr;
  if (cudaFuncGetAttributes(&attr, k) != cudaSuccess) return -1;
  const int WN = (N_max + 31) / 32;
  const uint32_t pw = mkpt_warp_bytes(WN, L, MM);
  int wpc = attr.maxThreadsPerBlock / 32;
  const long long by_smem = ((long long)smem_optin - blob_bytes - attr.sharedSizeBytes - 64) / pw;
  if (by_smem < wpc) wpc = (int)by_smem;
  if (wpc < 1) return -1;
  if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(blob_bytes + wpc * pw)) != cudaSuccess)
    return -1;
  *per_warp = pw;
  *max_wpc = wpc;
  return 0;
}

cudaError_t mkpt_launch(const RunArgs &a, int n_inst, int MM, int L, int wpc, uint32_t per_warp, cudaStream_t st,
                        bool replay) {
  mkpt_kernel_t k = replay ? mkpt_replay_kernel_for(MM, a.M, L) : mkpt_kernel_for(MM, a.M, L);
  if (!k) return cudaErrorInvalidValue;
  const int G = 32 / L;
  const int warps_inst = (a.R + G - 1) / G;
  dim3 grid((warps_inst + wpc - 1) / wpc, n_inst);
  const int smem = (int)(a.blob_bytes + wpc * per_warp);
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);  // see qkp_launch
  if (e != cudaSuccess) return e;
  k<<<grid, wpc * 32, smem, st>>>(a);
  return cudaGetLastError();
}

}  // namespace saim
