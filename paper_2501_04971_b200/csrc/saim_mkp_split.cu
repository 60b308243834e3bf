// saim_mkp_split.cu -- launch planning of the MKP row-split kernel (saim_mkp_split.cuh).
#include "saim_mkp_split.cuh"

namespace saim {

mkps_kernel_t mkps_replay_kernel_for(int MM, int M);   // saim_mkp_split_replay.cu
static mkps_kernel_t mkps_kernel_for(int MM, int M) { return mkps_kernel_for_t<false>(MM, M); }

// Plan for the row-split kernel (S = 2): per-warp shared bytes and max warps per CTA.
int mkps_plan(int M, int N_max, int smem_optin, int MM, uint32_t blob_bytes, uint32_t *per_warp, int *max_wpc) {
  mkps_kernel_t k = mkps_kernel_for(MM, M);
  if (!k) return -1;
  cudaFuncAttributes attr;
  if (cudaFuncGetAttributes(&attr, k) != cudaSuccess) return -1;
  const int WN = (N_max + 31) / 32;
  const uint32_t pw = mkps_warp_bytes(WN, 2, MM);
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

cudaError_t mkps_launch(const RunArgs &a, int n_inst, int MM, int wpc, uint32_t per_warp, cudaStream_t st, bool replay) {
  mkps_kernel_t k = replay ? mkps_replay_kernel_for(MM, a.M) : mkps_kernel_for(MM, a.M);
  if (!k) return cudaErrorInvalidValue;
  const int warps_inst = (a.R + 15) / 16;
  dim3 grid((warps_inst + wpc - 1) / wpc, n_inst);
  const int smem = (int)(a.blob_bytes + wpc * per_warp);
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);  // see qkp_launch
  if (e != cudaSuccess) return e;
  k<<<grid, wpc * 32, smem, st>>>(a);
  return cudaGetLastError();
}

}  // namespace saim
