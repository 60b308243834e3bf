// saim_mkp.cu -- launch planning of the MKP lockstep kernel (saim_mkp.cuh).
#include "saim_mkp.cuh"

namespace saim {

mkp_kernel_t mkp_replay_kernel_for(int MM, int M, bool prod);   // saim_mkp_replay.cu

// (MM, M) -> main kernel: exact arithmetic widths for the paper's MKP sizes (M = 5, 10, 30).
static mkp_kernel_t mkp_kernel_for(int MM, int M, bool prod = false) { return mkp_kernel_for_t<false>(MM, M, prod); }

static int mm_for(int M) { return M <= 4 ? 4 : (M <= 8 ? 8 : (M <= 16 ? 16 : (M <= 32 ? 32 : -1))); }

// Plan the MKP launch: padded constraint count MM, blob layout, per-warp bytes and the maximum
// warps per CTA allowed by threads/registers and shared memory.  Returns 0 or -1 (does not fit).
int mkp_plan(int n, int M, int N_max, int smem_optin, int *MM_out, uint32_t *blob_bytes, uint32_t *per_warp,
             int *max_wpc, uint32_t *per_warp_prod, int *max_wpc_prod) {
  const int MM = mm_for(M);
  if (MM < 0) return -1;
  mkp_kernel_t k = mkp_kernel_for(MM, M);
  cudaFuncAttributes attr;
  if (cudaFuncGetAttributes(&attr, k) != cudaSuccess) return -1;
  const MkpLayout L = mkp_layout(n, MM);
  const int WN = (N_max + 31) / 32;
  const uint32_t pw = mkp_warp_bytes(WN, MM);
  int wpc = attr.maxThreadsPerBlock / 32;
  const long long by_smem = ((long long)smem_optin - L.bytes - attr.sharedSizeBytes - 64) / pw;
  if (by_smem < wpc) wpc = (int)by_smem;
  if (wpc < 1) return -1;
  if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(L.bytes + wpc * pw)) != cudaSuccess)
    return -1;
  // with producer warps (M <= 8): 2 warps per consumer, larger per-consumer region
  *per_warp_prod = mkp_warp_bytes(WN, MM, 1);
  *max_wpc_prod = 0;
  mkp_kernel_t kp = mkp_kernel_for(MM, M, true);
  cudaFuncAttributes attrp;
  if (kp && cudaFuncGetAttributes(&attrp, kp) == cudaSuccess) {
    int wpcp = attrp.maxThreadsPerBlock / 64;
    const long long by_smem_p = ((long long)smem_optin - L.bytes - attrp.sharedSizeBytes - 64) / *per_warp_prod;
    if (by_smem_p < wpcp) wpcp = (int)by_smem_p;
    if (wpcp >= 1 && cudaFuncSetAttribute(kp, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)(L.bytes + wpcp * *per_warp_prod)) == cudaSuccess)
      *max_wpc_prod = wpcp;
  }
  *MM_out = MM;
  *blob_bytes = L.bytes;
  *per_warp = pw;
  *max_wpc = wpc;
  return 0;
}

// wpc consumer warps per CTA (plus as many producer warps if a.mkp_prod; per_warp is then the
// producer-mode per-consumer region).
cudaError_t mkp_launch(const RunArgs &a, int n_inst, int MM, int wpc, uint32_t per_warp, cudaStream_t st, bool replay) {
  mkp_kernel_t k = replay ? mkp_replay_kernel_for(MM, a.M, a.mkp_prod != 0) : mkp_kernel_for(MM, a.M, a.mkp_prod != 0);
  if (!k) return cudaErrorInvalidValue;
  const int warps_per_inst = (a.R + 31) / 32;
  dim3 grid((warps_per_inst + wpc - 1) / wpc, n_inst);
  const int smem = (int)(a.blob_bytes + wpc * per_warp);
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);  // see qkp_launch
  if (e != cudaSuccess) return e;
  k<<<grid, wpc * 32 * (a.mkp_prod ? 2 : 1), smem, st>>>(a);
  return cudaGetLastError();
}

}  // namespace saim
