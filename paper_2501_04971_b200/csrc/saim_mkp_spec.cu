// saim_mkp_spec.cu -- launch planning of the speculative sub-warp MKP kernel (saim_mkp_spec.cuh).
#include "saim_mkp_spec.cuh"

namespace saim {

mkpx_kernel_t mkpx_replay_kernel_for(int MM, int M, int G);   // saim_mkp_spec_replay.cu
static mkpx_kernel_t mkpx_kernel_for(int MM, int M, int G) { return mkpx_kernel_for_t<false>(MM, M, G); }

// Plan for G lanes per chain: bytes of the per-CTA spin table, per-warp shared bytes and the
// largest warps-per-CTA that fit.  Returns 0, or -1 (no instantiation / does not fit).
int mkpx_plan(int M, int N_max, int smem_optin, int MM, uint32_t blob_bytes, int G, uint32_t *table_bytes,
              uint32_t *per_warp, int *max_wpc, int *regs) {
  mkpx_kernel_t k = mkpx_kernel_for(MM, M, G);
  if (!k) return -1;
  cudaFuncAttributes attr;
  if (cudaFuncGetAttributes(&attr, k) != cudaSuccess) return -1;
  const int WN = (N_max + 31) / 32;
  const uint32_t tb = mkpx_table_bytes(WN, MM), pw = mkpx_warp_bytes(WN, G, MM);
  int wpc = attr.maxThreadsPerBlock / 32;
  const long long by_smem = ((long long)smem_optin - blob_bytes - tb - attr.sharedSizeBytes - 64) / pw;
  if (by_smem < wpc) wpc = (int)by_smem;
  if (wpc < 1) return -1;
  *table_bytes = tb;
  *per_warp = pw;
  *max_wpc = wpc;
  *regs = attr.numRegs;
  return 0;
}

cudaError_t mkpx_launch(const RunArgs &a, int n_inst, int MM, int G, int wpc, uint32_t per_warp, cudaStream_t st,
                        bool replay) {
  mkpx_kernel_t k = replay ? mkpx_replay_kernel_for(MM, a.M, G) : mkpx_kernel_for(MM, a.M, G);
  if (!k) return cudaErrorInvalidValue;
  const int C = 32 / G;
  const int warps_inst = (a.R + C - 1) / C;
  dim3 grid((warps_inst + wpc - 1) / wpc, n_inst);
  const int smem = (int)(a.blob_bytes + mkpx_table_bytes(a.WN, MM) + wpc * per_warp);
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);  // see qkp_launch
  if (e != cudaSuccess) return e;
  k<<<grid, wpc * 32, smem, st>>>(a);
  return cudaGetLastError();
}

}  // namespace saim
