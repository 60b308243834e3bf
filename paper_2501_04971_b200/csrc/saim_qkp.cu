// saim_qkp.cu -- launch code of the QKP kernel (saim_qkp.cuh) and the device self-tests.
#include "saim_qkp.cuh"

#ifdef SAIM_PROF
// Development profiling build only (-DSAIM_PROF): per-sweep clock64 totals by phase of the anneal.
extern "C" int saim_prof_read(unsigned long long *h, int reset) {
  cudaMemcpyFromSymbol(h, saim_prof, sizeof(saim_prof));
  if (reset) {
    unsigned long long z[48] = {0};
    cudaMemcpyToSymbol(saim_prof, z, sizeof(z));
  }
  return 0;
}
#endif

namespace saim {

// ---------------------------------------------------------------------------------------------
// Launch: grid (ceil(R / wpc), n_inst), wpc warps per CTA.
typedef void (*qkp_kernel_t)(const RunArgs);

template <int NPL, int QB, bool PK>
static qkp_kernel_t pick() { return saim_qkp_kernel<NPL, QB, PK, false>; }

qkp_kernel_t qkp_replay_kernel_for(int npl, int qb, int pk);   // saim_qkp_replay.cu

static qkp_kernel_t qkp_kernel_for(int npl, int qb, int pk) {
#define SAIM_QKP_CASE(P)                                \
  if (npl <= P) return qb == 1 ? (pk ? pick<P, 1, true>() : pick<P, 1, false>()) : pick<P, 2, false>();
  SAIM_QKP_CASE(1) SAIM_QKP_CASE(2) SAIM_QKP_CASE(3) SAIM_QKP_CASE(4) SAIM_QKP_CASE(6)
  SAIM_QKP_CASE(8) SAIM_QKP_CASE(10) SAIM_QKP_CASE(12) SAIM_QKP_CASE(16)
#undef SAIM_QKP_CASE
  return nullptr;
}

static int qkp_warp_bytes(int npl) {
  switch (npl) {
    case 1: return qkp_warp_smem_bytes<1>();   case 2: return qkp_warp_smem_bytes<2>();
    case 3: return qkp_warp_smem_bytes<3>();   case 4: return qkp_warp_smem_bytes<4>();
    case 6: return qkp_warp_smem_bytes<6>();   case 8: return qkp_warp_smem_bytes<8>();
    case 10: return qkp_warp_smem_bytes<10>(); case 12: return qkp_warp_smem_bytes<12>();
    default: return qkp_warp_smem_bytes<16>();
  }
}

int qkp_npl_bucket(int npl) {
  const int b[] = {1, 2, 3, 4, 6, 8, 10, 12, 16};
  for (int v : b)
    if (npl <= v) return v;
  return -1;
}

// max_wpc: warps per CTA limited by threads (launch bounds), registers and shared memory
// (blob + per-warp phi).  Sets the kernel's dynamic shared-memory limit accordingly.
cudaError_t qkp_configure(int npl, int qb, int pk, int blob_bytes, int smem_optin, int *max_wpc) {
  qkp_kernel_t k = qkp_kernel_for(npl, qb, pk);
  if (!k) return cudaErrorInvalidValue;
  cudaFuncAttributes attr;
  cudaError_t e = cudaFuncGetAttributes(&attr, k);
  if (e != cudaSuccess) return e;
  int wpc = attr.maxThreadsPerBlock / 32;
  if (wpc > 32) wpc = 32;
  const int per_warp = qkp_warp_bytes(npl);
  const int by_smem = (smem_optin - blob_bytes - (int)attr.sharedSizeBytes - 64) / per_warp;
  if (by_smem < wpc) wpc = by_smem;
  if (wpc < 1) return cudaErrorInvalidConfiguration;
  e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, blob_bytes + wpc * per_warp);
  if (e != cudaSuccess) return e;
  *max_wpc = wpc;
  return cudaSuccess;
}

// Dynamic shared memory = blob + wpc * per-warp region (phi + WarpState).
// replay = true: the exact-replay kernel (saim_qkp.cuh RP) over the same grid.
cudaError_t qkp_launch(int npl, int qb, int pk, const RunArgs &a, int n_inst, int wpc, int blob_bytes, cudaStream_t st,
                       bool replay) {
  qkp_kernel_t k = replay ? qkp_replay_kernel_for(npl, qb, pk) : qkp_kernel_for(npl, qb, pk);
  if (!k) return cudaErrorInvalidValue;
  dim3 grid((a.R + wpc - 1) / wpc, n_inst);
  const int smem = blob_bytes + wpc * qkp_warp_bytes(npl);
  // The dynamic shared-memory limit is a per-function, process-wide attribute: a later
  // saim_create of a smaller instance with the same template may have lowered it, so every launch
  // sets it to exactly what it requests.
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  k<<<grid, wpc * 32, smem, st>>>(a);
  return cudaGetLastError();
}

}  // namespace saim

// ---------------------------------------------------------------------------------------------
// Self-tests (include/saim.h saim_selftest).
namespace saim {
__global__ void selftest_philox_kernel(const uint32_t *in, uint32_t *out, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t *p = in + 6 * i;
  const uint4 o = philox4x32_10(make_uint4(p[0], p[1], p[2], p[3]), make_uint2(p[4], p[5]));
  out[4 * i + 0] = o.x; out[4 * i + 1] = o.y; out[4 * i + 2] = o.z; out[4 * i + 3] = o.w;
}

__global__ void selftest_logit_kernel(unsigned long long *out) {
  // one thread per numerator 2m+1, m in [0, 2^23)
  const uint32_t m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= (1u << 23)) return;
  const uint32_t w = m << 9;                       // any word with floor(w / 2^9) = m
  const float lf = logit_f32(w);
  const double u = uniform_f64(w);
  const double l = log(u) - log1p(-u);
  const double err = fabs((double)lf - l);
  double rel = err / ((double)kLogitAbs + (double)kLogitRel * fabs(l));
  if ((double)uniform_f32(w) != u) rel = 1e30;     // the fp32 uniform must be the exact (2m + 1) 2^-24
  atomicMax(out + 0, (unsigned long long)__double_as_longlong(rel));   // non-negative doubles order as ints
  atomicMax(out + 1, (unsigned long long)__double_as_longlong(err));
}

// Record of selftest 2 (include/saim.h): the double-double decision on given exact components.
struct DdRecord {
  long long phi, pi, kappa, s_o, s_c;
  double P, eta, beta_max;
  int32_t tn, td;
  uint32_t w;
  int32_t pad;
};
static_assert(sizeof(DdRecord) == 80, "DdRecord layout is part of the ABI");

__global__ void selftest_dd_kernel(const DdRecord *in, uint32_t *out, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const DdRecord r = in[i];
  InstHdr h;
  memset(&h, 0, sizeof(h));
  h.s_o = r.s_o; h.s_c = r.s_c; h.P = r.P; h.eta = r.eta; h.beta_max = r.beta_max;
  out[i] = (uint32_t)decide_dd(r.phi, r.pi, r.kappa, r.tn, r.td, &h, r.w);
}

int selftest(int which, int n, const uint32_t *in_u32, uint32_t *out_u32, double *out_f64) {
  if (which == 0) {
    uint32_t *d_in = nullptr, *d_out = nullptr;
    if (cudaMalloc(&d_in, sizeof(uint32_t) * 6 * (size_t)n) != cudaSuccess) return -1;
    if (cudaMalloc(&d_out, sizeof(uint32_t) * 4 * (size_t)n) != cudaSuccess) { cudaFree(d_in); return -1; }
    cudaMemcpy(d_in, in_u32, sizeof(uint32_t) * 6 * (size_t)n, cudaMemcpyHostToDevice);
    selftest_philox_kernel<<<(n + 127) / 128, 128>>>(d_in, d_out, n);
    cudaError_t e = cudaMemcpy(out_u32, d_out, sizeof(uint32_t) * 4 * (size_t)n, cudaMemcpyDeviceToHost);
    cudaFree(d_in); cudaFree(d_out);
    return e == cudaSuccess ? 0 : -1;
  }
  if (which == 2) {
    DdRecord *d_in = nullptr;
    uint32_t *d_out = nullptr;
    if (cudaMalloc(&d_in, sizeof(DdRecord) * (size_t)n) != cudaSuccess) return -1;
    if (cudaMalloc(&d_out, sizeof(uint32_t) * (size_t)n) != cudaSuccess) { cudaFree(d_in); return -1; }
    cudaMemcpy(d_in, in_u32, sizeof(DdRecord) * (size_t)n, cudaMemcpyHostToDevice);
    selftest_dd_kernel<<<(n + 127) / 128, 128>>>(d_in, d_out, n);
    cudaError_t e = cudaMemcpy(out_u32, d_out, sizeof(uint32_t) * (size_t)n, cudaMemcpyDeviceToHost);
    cudaFree(d_in); cudaFree(d_out);
    return e == cudaSuccess ? 0 : -1;
  }
  if (which == 1) {
    unsigned long long *d = nullptr;
    if (cudaMalloc(&d, 16) != cudaSuccess) return -1;
    cudaMemset(d, 0, 16);
    selftest_logit_kernel<<<(1u << 23) / 256, 256>>>(d);
    unsigned long long h[2];
    cudaError_t e = cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    cudaFree(d);
    memcpy(&out_f64[0], &h[0], 8);
    memcpy(&out_f64[1], &h[1], 8);
    return e == cudaSuccess ? 0 : -1;
  }
  return -1;
}
}  // namespace saim
