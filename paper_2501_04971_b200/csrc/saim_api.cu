// saim_api.cu -- host side of libsaim (C ABI declared in include/saim.h).
//
// saim_create: validation, slack extension, normalisation scales,
// integer-range proofs (DESIGN.md Appendix B), and the HBM layout of saim_layout.h.
// saim_run: argument checks and the asynchronous launches (init + fused SAIM kernel) on the
// caller's stream.  No arithmetic of the sweep happens on the host.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include <mutex>

#include "../../include/saim.h"
#include "saim_dev.cuh"
#include "saim_layout.h"

namespace saim {
int qkp_npl_bucket(int npl);
cudaError_t qkp_configure(int npl, int qb, int pk, int blob_bytes, int smem_optin, int *max_wpc);
cudaError_t qkp_launch(int npl, int qb, int pk, const RunArgs &a, int n_inst, int wpc, int smem_bytes, cudaStream_t st,
                       bool replay);
int mkp_plan(int n, int M, int N_max, int smem_optin, int *MM_out, uint32_t *blob_bytes, uint32_t *per_warp,
             int *max_wpc, uint32_t *per_warp_prod, int *max_wpc_prod);
cudaError_t mkp_launch(const RunArgs &a, int n_inst, int MM, int wpc, uint32_t per_warp, cudaStream_t st, bool replay);
int mkpt_plan(int M, int N_max, int smem_optin, int MM, uint32_t blob_bytes, int L, uint32_t *per_warp, int *max_wpc);
cudaError_t mkpt_launch(const RunArgs &a, int n_inst, int MM, int L, int wpc, uint32_t per_warp, cudaStream_t st,
                        bool replay);
int mkps_plan(int M, int N_max, int smem_optin, int MM, uint32_t blob_bytes, uint32_t *per_warp, int *max_wpc);
cudaError_t mkps_launch(const RunArgs &a, int n_inst, int MM, int wpc, uint32_t per_warp, cudaStream_t st, bool replay);
int mkpx_plan(int M, int N_max, int smem_optin, int MM, uint32_t blob_bytes, int G, uint32_t *table_bytes,
              uint32_t *per_warp, int *max_wpc, int *regs);
cudaError_t mkpx_launch(const RunArgs &a, int n_inst, int MM, int G, int wpc, uint32_t per_warp, cudaStream_t st,
                        bool replay);
int selftest(int which, int n, const uint32_t *in_u32, uint32_t *out_u32, double *out_f64);
}  // namespace saim

using namespace saim;

static thread_local std::string g_err;

// The fp64 slow path's logit table (saim_dev.cuh logit_f64): one per device, built on first use
// and kept for the life of the process (64 MB).
__global__ void saim_logit_table_kernel(double *t) {
  const uint32_t m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m < (1u << 23)) t[m] = logit_f64_calc(m << 9);
}

static std::mutex g_tab_mu;
static double *g_tab[64] = {};

// saim_selftest(3): the table's entries (through the slow path's accessor) next to a direct
// computation, for given Philox words.
__global__ void saim_selftest_logit_table_kernel(const double *tab, const uint32_t *w, double *out, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  InstHdr h;
  memset(&h, 0, sizeof(h));
  h.logit_tab = tab;
  out[2 * i] = logit_f64(&h, w[i]);
  out[2 * i + 1] = logit_f64_calc(w[i]);
}

static cudaError_t logit_table(int dev, const double **out) {
  std::lock_guard<std::mutex> lk(g_tab_mu);
  if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  if (!g_tab[dev]) {
    double *p = nullptr;
    cudaError_t e = cudaMalloc(&p, sizeof(double) << 23);
    if (e != cudaSuccess) return e;
    saim_logit_table_kernel<<<(1u << 23) / 256, 256>>>(p);
    e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      cudaFree(p);
      return e;
    }
    g_tab[dev] = p;
  }
  *out = g_tab[dev];
  return cudaSuccess;
}

static int fail(int code, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

static int cuda_fail(cudaError_t e, const char *what) {
  return fail(SAIM_ECUDA, "%s: %s", what, cudaGetErrorString(e));
}

struct saim_ctx {
  int device = 0;
  int n_inst = 0, n = 0, M = 0;
  int kernel = 0;       // 1 = QKP, 2 = MKP
  int npl = 0, qb = 0, pk = 0;  // QKP (pk: phi packed as two int16 per word)
  int lanes = 32;       // lanes per replica (QKP: 32; MKP: 1 lockstep, L = 2 or 4 outcome tree)
  int mm = 0;           // MKP padded constraint count
  int mkp_kind = 0;     // MKP kernel: 0 lockstep, 1 outcome tree, 2 row split, 3 speculative sub-warp
  uint32_t per_warp = 0;
  uint32_t spec_fixed = 0;     // MKP speculative kernel: shared bytes per CTA besides the warps' (blob + spin table + static)
  int spec_regs = 0;           // ... registers per thread
  int smem_sm = 0;             // shared memory per SM
  uint32_t per_warp_prod = 0;  // MKP lockstep with producer warps: per-consumer region, max consumers per CTA
  int max_wpc_prod = 0;
  int N_max = 0, n_slack_max = 0;
  int smem_bytes = 0, max_wpc = 32, sm_count = 148;
  uint32_t blob_bytes = 0, a_off = 0, c_off = 0, x_off = 0;
  double beta_max = 0, eta = 0;
  int flags = 0;
  long long r_abs_max = 0;
  long long a_ext_max = 0;  // max A_ext entry (items and slack weights) over instances
  int r_tol = 0;        // QKP certificate tolerance D (min over instances)
  unsigned char *d_blob = nullptr;
  uint8_t *d_replay = nullptr;   // QKP exact-replay flags, [n_inst][R] (grown on demand)
  size_t replay_cap = 0;
  InstHdr *d_hdr = nullptr;
  std::vector<InstHdr> hdr;
  std::vector<std::vector<int32_t>> q;  // slack bits per row per instance
};

static int bit_length(long long v) {
  int q = 0;
  while (v > 0) { ++q; v >>= 1; }
  return q;
}

static uint32_t align16(uint32_t v) { return (v + 15u) & ~15u; }

__global__ void saim_init_outputs(int64_t *inst_best, int n_inst, uint64_t *counters) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (inst_best && i < n_inst) inst_best[i] = LLONG_MAX;
  if (counters && i < SAIM_NUM_COUNTERS) counters[i] = 0;
}

extern "C" const char *saim_last_error(void) { return g_err.c_str(); }

extern "C" int saim_create(const saim_problem *prob, const saim_params *par, saim_ctx **out) {
  g_err.clear();
  if (!prob || !par || !out) return fail(SAIM_EINVAL, "null argument");
  *out = nullptr;
  const int S = prob->n_inst, n = prob->n_items, M = prob->n_cons;
  if (S < 1 || S >= 4096) return fail(SAIM_EINVAL, "n_inst must be in [1, 4096) (RNG counter field), got %d", S);
  if (n < 1) return fail(SAIM_EINVAL, "n_items must be >= 1");
  if (M < 0 || M > 32) return fail(SAIM_EINVAL, "n_cons must be in [0, 32], got %d", M);
  if (!prob->c || (M > 0 && (!prob->A || !prob->b)) || !par->P)
    return fail(SAIM_EINVAL, "missing c/A/b/P array");
  if (!std::isfinite(par->eta) || par->eta < 0) return fail(SAIM_EINVAL, "eta must be finite and >= 0");
  if (!std::isfinite(par->beta_max) || par->beta_max <= 0) return fail(SAIM_EINVAL, "beta_max must be finite and > 0");
  const int xmask = SAIM_FLAG_MKP_SPEC2 | SAIM_FLAG_MKP_SPEC4 | SAIM_FLAG_MKP_SPEC8 | SAIM_FLAG_MKP_SPEC16 | SAIM_FLAG_MKP_SPEC32;
  const int kmask = SAIM_FLAG_MKP_LOCKSTEP | SAIM_FLAG_MKP_L2 | SAIM_FLAG_MKP_L4 | SAIM_FLAG_MKP_SPLIT2 | xmask;
  if ((par->flags & ~(SAIM_FLAG_NO_FREEZE_EXIT | SAIM_FLAG_QKP_NO_HOT_LOOP | SAIM_FLAG_MKP_NO_PRODUCER | SAIM_FLAG_TEST_REPLAY | kmask)) || __builtin_popcount(par->flags & kmask) > 1)
    return fail(SAIM_EINVAL, "unknown or conflicting flags 0x%x", par->flags);

  if (M > 1 && prob->Q)
    return fail(SAIM_EUNSUPPORTED, "quadratic objective with M = %d > 1 constraints has no kernel", M);

  saim_ctx *ctx = new saim_ctx();
  ctx->device = par->device;
  ctx->n_inst = S; ctx->n = n; ctx->M = M;
  ctx->beta_max = par->beta_max; ctx->eta = par->eta;
  ctx->flags = par->flags;
  ctx->hdr.resize(S);
  ctx->q.resize(S);

  // ---- per-instance validation, slack, scales, range proofs ----
  long long rmax_all = 0;
  long long phib_all = 0;   // max phi bound over instances (QKP packed-phi eligibility)
  int qmax_abs = 0;
  for (int s = 0; s < S; ++s) {
    const int32_t *Q = prob->Q ? prob->Q + (size_t)s * n * n : nullptr;
    const int32_t *c = prob->c + (size_t)s * n;
    const int32_t *A = M ? prob->A + (size_t)s * M * n : nullptr;
    const int64_t *b = M ? prob->b + (size_t)s * M : nullptr;
    const double P = par->P[s];
    if (!std::isfinite(P) || P < 0) { delete ctx; return fail(SAIM_EINVAL, "P[%d] must be finite and >= 0", s); }
    long long so = 0, sc = 0;
    long long phi_bound = 0;
    for (int i = 0; i < n; ++i) {
      long long rowsum = std::llabs((long long)c[i]);
      so = std::max(so, std::llabs((long long)c[i]));
      if (Q) {
        if (Q[(size_t)i * n + i] != 0) { delete ctx; return fail(SAIM_EINVAL, "Q[%d] has a nonzero diagonal at %d", s, i); }
        for (int j = 0; j < n; ++j) {
          const long long qij = Q[(size_t)i * n + j];
          if (qij != Q[(size_t)j * n + i]) { delete ctx; return fail(SAIM_EINVAL, "Q[%d] is not symmetric at (%d,%d)", s, i, j); }
          so = std::max(so, std::llabs(qij));
          rowsum += std::llabs(qij);
          qmax_abs = (int)std::max<long long>(qmax_abs, std::llabs(qij));
        }
      }
      phi_bound = std::max(phi_bound, rowsum);
    }
    int n_slack = 0;
    long long rmax = 0;
    for (int k = 0; k < M; ++k) {
      if (b[k] < 1) { delete ctx; return fail(SAIM_EINVAL, "b[%d][%d] must be >= 1", s, k); }
      if (b[k] >= (1LL << 30)) { delete ctx; return fail(SAIM_ERANGE, "b[%d][%d] >= 2^30", s, k); }
      sc = std::max(sc, (long long)b[k]);
      long long load = 0;
      for (int j = 0; j < n; ++j) {
        const long long v = A[(size_t)k * n + j];
        if (v < 0) { delete ctx; return fail(SAIM_EINVAL, "A[%d] has a negative entry", s); }
        sc = std::max(sc, v);
        load += v;
      }
      const int q = bit_length(b[k]);  // Q = floor(log2 b + 1)
      ctx->q[s].push_back(q);
      n_slack += q;
      const long long slack_max = (1LL << q) - 1;
      rmax = std::max(rmax, std::max((long long)b[k], load + slack_max - b[k]));
    }
    if (so == 0) so = 1;
    if (sc == 0) sc = 1;
    rmax_all = std::max(rmax_all, rmax);
    InstHdr &h = ctx->hdr[s];
    memset(&h, 0, sizeof(h));
    h.N = n + n_slack;
    h.n_slack = n_slack;
    h.b0 = M ? b[0] : 0;
    h.s_o = so; h.s_c = sc;
    h.c_o = 1.0 / (double)so;
    h.c_p = P / ((double)sc * (double)sc);
    h.c_l = par->eta / ((double)sc * (double)sc);
    h.phi_bound = (double)phi_bound;
    h.P = P; h.eta = par->eta; h.beta_max = par->beta_max;
    phib_all = std::max(phib_all, phi_bound);
    {
      long long amax = 0;
      for (int k = 0; k < M; ++k) {
        amax = std::max(amax, (1LL << (ctx->q[s][k] - 1)));
        for (int j = 0; j < n; ++j) amax = std::max(amax, (long long)A[(size_t)k * n + j]);
      }
      h.v_bound = 2.0 * (double)rmax + (double)amax;
      ctx->a_ext_max = std::max(ctx->a_ext_max, amax);
      h.r_bound = (double)rmax;
      // QKP quiet certificates hold for |r - r_cert| <= D: the tolerance widens the scan threshold
      // by 2 beta c_p D |A_i| <= 1 (of ln(2^24-1) = 16.6) for the heaviest item.
      long long aitem = 0;
      for (int k = 0; k < M; ++k)
        for (int j = 0; j < n; ++j) aitem = std::max(aitem, (long long)A[(size_t)k * n + j]);
      const double dt = (h.c_p > 0 && aitem > 0) ? std::floor(0.5 / (par->beta_max * h.c_p * (double)aitem)) : 0.0;
      const int rt = (int)std::min(dt, (double)(1 << 20));
      ctx->r_tol = (s == 0) ? rt : std::min(ctx->r_tol, rt);
    }
    ctx->N_max = std::max(ctx->N_max, h.N);
    ctx->n_slack_max = std::max(ctx->n_slack_max, n_slack);
    // exactness proofs (DESIGN.md Appendix B)
    if (phi_bound >= (1LL << 22))
      { delete ctx; return fail(SAIM_ERANGE, "instance %d: |phi| bound %lld >= 2^22", s, phi_bound); }
    if (rmax >= (1LL << 21))
      { delete ctx; return fail(SAIM_ERANGE, "instance %d: |r| bound %lld >= 2^21", s, rmax); }
    long long fb = 0;
    for (int i = 0; i < n; ++i) fb += std::llabs((long long)c[i]) + (Q ? phi_bound : 0);
    if (fb >= (1LL << 42)) { delete ctx; return fail(SAIM_ERANGE, "instance %d: |f| bound >= 2^42", s); }
  }
  ctx->r_abs_max = rmax_all;
  if (ctx->N_max > 2048) { delete ctx; return fail(SAIM_ESMEM, "N = %d spins > 2048", ctx->N_max); }

  cudaError_t e = cudaSetDevice(ctx->device);
  if (e != cudaSuccess) { delete ctx; return cuda_fail(e, "cudaSetDevice"); }
  {
    const double *tab = nullptr;
    if ((e = logit_table(ctx->device, &tab)) != cudaSuccess) { delete ctx; return cuda_fail(e, "logit table"); }
    for (int s = 0; s < S; ++s) ctx->hdr[s].logit_tab = tab;
  }
  int smem_optin = 0;
  cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->device);
  cudaDeviceGetAttribute(&ctx->sm_count, cudaDevAttrMultiProcessorCount, ctx->device);
  cudaDeviceGetAttribute(&ctx->smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, ctx->device);

  std::vector<unsigned char> blob;
  if (M <= 1) {
    // ---------------- QKP kernel layout ----------------
    ctx->kernel = 1;
    const int npl = (n + 31) / 32;
    ctx->npl = qkp_npl_bucket(npl);
    if (ctx->npl < 0) { delete ctx; return fail(SAIM_ESMEM, "n = %d items > 512 (Q does not fit shared memory)", n); }
    ctx->qb = qmax_abs <= 127 ? 1 : (qmax_abs <= 32767 ? 2 : 0);
    if (!ctx->qb) { delete ctx; return fail(SAIM_ERANGE, "|Q| entries > 32767 need wider storage"); }
    // int8 Q with |phi| <= 32767 in every state: phi held as biased int16 pairs, a Q-row update is
    // one packed integer add per two items (DESIGN.md 6.1 "Packed phi")
    ctx->pk = (ctx->qb == 1 && phib_all <= 32767) ? 1 : 0;
    const int E = 4 / ctx->qb;
    const int QW = (ctx->npl + E - 1) / E;
    const int NBP = ((ctx->npl + 2) + 3) & ~3;            // blocks incl. padding to a 4-block group
    // [A_ext | c | Q rows]: offsets fixed by the (NPL, QB) template, so the kernel addresses all
    // three from one register (saim_layout.h)
    const uint32_t q_bytes = align16((uint32_t)n * QW * 128u);
    ctx->a_off = 0;
    ctx->c_off = align16(NBP * 32 * 4);
    ctx->x_off = ctx->c_off + align16(ctx->npl * 32 * 4);   // Q rows
    ctx->blob_bytes = ctx->x_off + q_bytes;
    if ((int)ctx->blob_bytes + 64 > smem_optin) {
      delete ctx;
      return fail(SAIM_ESMEM, "QKP blob of %u bytes exceeds shared memory (%d)", ctx->blob_bytes, smem_optin);
    }
    ctx->smem_bytes = (int)ctx->blob_bytes;
    blob.assign((size_t)S * ctx->blob_bytes, 0);
    const uint32_t bias = 1u << (8 * ctx->qb - 1);
    for (int s = 0; s < S; ++s) {
      unsigned char *B = blob.data() + (size_t)s * ctx->blob_bytes;
      const int32_t *Q = prob->Q ? prob->Q + (size_t)s * n * n : nullptr;
      for (int j = 0; j < n; ++j) {
        uint32_t *row = reinterpret_cast<uint32_t *>(B + ctx->x_off + (size_t)j * QW * 128u);
        for (int w = 0; w < QW; ++w)
          for (int l = 0; l < 32; ++l) {
            uint32_t word = 0;
            for (int e2 = 0; e2 < E; ++e2) {
              const int m = E * w + e2, i = 32 * m + l;
              const long long qv = (Q && i < n) ? Q[(size_t)j * n + i] : 0;
              word |= ((uint32_t)(qv + bias) & ((1u << (8 * ctx->qb)) - 1u)) << (8 * ctx->qb * e2);
            }
            row[32 * w + l] = word;
          }
      }
      float *Aext = reinterpret_cast<float *>(B + ctx->a_off);
      const int Ns = ctx->hdr[s].N;
      for (int i = 0; i < NBP * 32; ++i) Aext[i] = i < Ns ? 0.0f : std::nanf("");   // NaN: no spin (scan: quiet)
      if (M == 1) {
        const int32_t *A = prob->A + (size_t)s * n;
        for (int i = 0; i < n; ++i) Aext[i] = (float)A[i];
        const int q = ctx->q[s][0];
        for (int bit = 0; bit < q; ++bit) Aext[n + bit] = (float)(1LL << bit);
      }
      int32_t *cc = reinterpret_cast<int32_t *>(B + ctx->c_off);
      for (int i = 0; i < n; ++i) cc[i] = prob->c[(size_t)s * n + i];
    }
    e = qkp_configure(ctx->npl, ctx->qb, ctx->pk, ctx->smem_bytes, smem_optin, &ctx->max_wpc);
    if (e == cudaErrorInvalidConfiguration) {
      delete ctx;
      return fail(SAIM_ESMEM, "QKP layout (%u bytes) leaves no room for one warp's state in shared memory", ctx->blob_bytes);
    }
    if (e != cudaSuccess) { delete ctx; return cuda_fail(e, "configure QKP kernel"); }
    ctx->lanes = 32;
  } else if (!prob->Q) {
    // ---------------- MKP kernel layout (saim_layout.h MkpLayout) ----------------
    ctx->kernel = 2;
    ctx->lanes = 1;
    if (mkp_plan(n, M, ctx->N_max, smem_optin, &ctx->mm, &ctx->blob_bytes, &ctx->per_warp, &ctx->max_wpc,
                 &ctx->per_warp_prod, &ctx->max_wpc_prod) != 0) {
      delete ctx;
      return fail(SAIM_ESMEM, "MKP instance (n=%d, M=%d, N=%d) does not fit shared memory", n, M, ctx->N_max);
    }
    const int MM = ctx->mm;
    const MkpLayout L = mkp_layout(n, MM);
    ctx->smem_bytes = (int)(L.bytes + ctx->per_warp);
    // Default (measured on B200): the speculative sub-warp kernel with G = 8
    // lanes per replica for M <= 8 (the outcome tree with L = 2 if it does not fit), the lockstep
    // kernel for M > 8; the row split (M > 8) only on request.
    const int xmask = SAIM_FLAG_MKP_SPEC2 | SAIM_FLAG_MKP_SPEC4 | SAIM_FLAG_MKP_SPEC8 | SAIM_FLAG_MKP_SPEC16 | SAIM_FLAG_MKP_SPEC32;
    const int kmask = SAIM_FLAG_MKP_LOCKSTEP | SAIM_FLAG_MKP_L2 | SAIM_FLAG_MKP_L4 | SAIM_FLAG_MKP_SPLIT2 | xmask;
    bool spec = (ctx->flags & xmask) != 0 || (!(ctx->flags & kmask) && M <= 8);
    if (spec) {   // speculative sub-warp kernel (saim_mkp_spec.cu)
      const int G = (ctx->flags & SAIM_FLAG_MKP_SPEC2) ? 2 : (ctx->flags & SAIM_FLAG_MKP_SPEC4) ? 4
                    : (ctx->flags & SAIM_FLAG_MKP_SPEC16) ? 16 : (ctx->flags & SAIM_FLAG_MKP_SPEC32) ? 32 : 8;
      uint32_t tb = 0, pw = 0;
      int wpc = 0;
      if (mkpx_plan(M, ctx->N_max, smem_optin, MM, L.bytes, G, &tb, &pw, &wpc, &ctx->spec_regs) == 0) {
        ctx->lanes = G;
        ctx->mkp_kind = 3;
        ctx->per_warp = pw;
        ctx->max_wpc = wpc;
        ctx->smem_bytes = (int)(L.bytes + tb + pw);
        ctx->spec_fixed = L.bytes + tb + 1024u + 256u;   // + the per-CTA reservation and static shared memory
      } else if (ctx->flags & xmask) {
        delete ctx;
        return fail(SAIM_ESMEM, "MKP speculative kernel (G=%d) has no instantiation for M=%d or does not fit shared memory", G, M);
      } else {
        spec = false;
      }
    }
    const bool tree = (ctx->flags & (SAIM_FLAG_MKP_L2 | SAIM_FLAG_MKP_L4)) ||
                      (!spec && !(ctx->flags & SAIM_FLAG_MKP_LOCKSTEP) && M <= 8);
    const bool split = !tree && !spec && MM >= 16 && (ctx->flags & SAIM_FLAG_MKP_SPLIT2);
    if (spec) {
      // (planned above)
    } else if (tree) {   // outcome-tree kernel (saim_mkp_tree.cu)
      const int lanes = (ctx->flags & SAIM_FLAG_MKP_L4) ? 4 : 2;
      uint32_t pw = 0;
      int wpc = 0;
      if (mkpt_plan(M, ctx->N_max, smem_optin, MM, L.bytes, lanes, &pw, &wpc) == 0) {
        ctx->lanes = lanes;
        ctx->mkp_kind = 1;
        ctx->per_warp = pw;
        ctx->max_wpc = wpc;
        ctx->smem_bytes = (int)(L.bytes + pw);
      } else if (ctx->flags & (SAIM_FLAG_MKP_L2 | SAIM_FLAG_MKP_L4)) {
        delete ctx;
        return fail(SAIM_ESMEM, "MKP outcome-tree kernel (L=%d) does not fit shared memory", lanes);
      }
    } else if (split) {   // row-split kernel (saim_mkp_split.cu)
      uint32_t pw = 0;
      int wpc = 0;
      if (mkps_plan(M, ctx->N_max, smem_optin, MM, L.bytes, &pw, &wpc) == 0) {
        ctx->lanes = 2;
        ctx->mkp_kind = 2;
        ctx->per_warp = pw;
        ctx->max_wpc = wpc;
        ctx->smem_bytes = (int)(L.bytes + pw);
      } else if (ctx->flags & SAIM_FLAG_MKP_SPLIT2) {
        delete ctx;
        return fail(SAIM_ESMEM, "MKP row-split kernel does not fit shared memory");
      }
    }
    blob.assign((size_t)S * ctx->blob_bytes, 0);
    for (int s = 0; s < S; ++s) {
      unsigned char *B = blob.data() + (size_t)s * ctx->blob_bytes;
      const InstHdr &h = ctx->hdr[s];
      float *acol = reinterpret_cast<float *>(B + L.acol);
      float *ic = reinterpret_cast<float *>(B + L.iconst);
      int32_t *cc = reinterpret_cast<int32_t *>(B + L.cint);
      int64_t *brow = reinterpret_cast<int64_t *>(B + L.brow);
      int32_t *qrow = reinterpret_cast<int32_t *>(B + L.qrow);
      for (int i = 0; i < n; ++i) {
        double a2 = 0.0, a1 = 0.0;
        for (int k = 0; k < M; ++k) {
          const double v = (double)prob->A[((size_t)s * M + k) * n + i];
          acol[(size_t)i * MM + k] = (float)v;
          a2 += v * v;
          a1 += v;
        }
        const int32_t ci = prob->c[(size_t)s * n + i];
        const float cphi = (float)(-h.c_o * (double)ci), cpa = (float)(h.c_p * a2);
        ic[4 * i + 0] = cphi;
        ic[4 * i + 1] = cpa;
        ic[4 * i + 2] = (float)a1;
        // E0_i = (2 (MM+6) 2^-24 + 1.01 2^-22) (|c_o c_i| + c_p a_i), DESIGN.md 6.2 (factor 2:
        // margin; the 2^-22 term bounds the final rounding of z through |z|'s static bound)
        ic[4 * i + 3] = (float)((2.0 * (MM + 6) * 0x1p-24 + 1.01 * 0x1p-22) * (fabs((double)cphi) + (double)cpa));
        cc[i] = ci;
      }
      for (int k = 0; k < M; ++k) {
        brow[k] = prob->b[(size_t)s * M + k];
        qrow[k] = ctx->q[s][k];
      }
      float *band = reinterpret_cast<float *>(B + L.band);
      const uint32_t bs = mkp_band_stride(n);
      for (int d = 1; d <= 3; ++d)
        for (int i = d; i < n; ++i) {
          double g = 0.0;
          for (int k = 0; k < M; ++k)
            g += (double)prob->A[((size_t)s * M + k) * n + i] * (double)prob->A[((size_t)s * M + k) * n + i - d];
          band[(d - 1) * bs + i] = (float)g;
        }
    }
  } else {
    delete ctx;
    return fail(SAIM_EUNSUPPORTED, "quadratic objective with M = %d > 1 constraints has no kernel", M);
  }

  e = cudaMalloc(&ctx->d_blob, blob.size());
  if (e != cudaSuccess) { delete ctx; return cuda_fail(e, "cudaMalloc blob"); }
  e = cudaMalloc(&ctx->d_hdr, sizeof(InstHdr) * S);
  if (e != cudaSuccess) { cudaFree(ctx->d_blob); delete ctx; return cuda_fail(e, "cudaMalloc hdr"); }
  e = cudaMemcpy(ctx->d_blob, blob.data(), blob.size(), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(ctx->d_hdr, ctx->hdr.data(), sizeof(InstHdr) * S, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) { saim_destroy(ctx); return cuda_fail(e, "upload"); }
  *out = ctx;
  return SAIM_OK;
}

extern "C" int saim_run(saim_ctx *ctx, uint64_t seed, int32_t rep0, int32_t R, int32_t K, int32_t T,
                        void *cuda_stream, const saim_outputs *out) {
  g_err.clear();
  if (!ctx || !out) return fail(SAIM_EINVAL, "null argument");
  if (R < 1 || rep0 < 0 || (long long)rep0 + R > (1LL << 20))
    return fail(SAIM_EINVAL, "replicas must satisfy 1 <= R and rep0 + R <= 2^20");
  if (K < 1 || T < 1) return fail(SAIM_EINVAL, "K and T must be >= 1");
  if (!out->best_f || !out->best_x || !out->best_k || !out->n_feasible)
    return fail(SAIM_EINVAL, "best_f, best_x, best_k and n_feasible are required");
  if ((double)K * (double)(ctx->r_abs_max + 1) >= 4.0e18)
    return fail(SAIM_ERANGE, "K * max|r| would overflow the int64 Lagrange accumulator");
  // kappa_i = sum_m Lambda_m A_mi in int64 on the double-double slow path (R18)
  if ((double)K * (double)(ctx->r_abs_max + 1) * (double)ctx->a_ext_max * (double)std::max(ctx->M, 1) >= 4.0e18)
    return fail(SAIM_ERANGE, "K * max|r| * max A * M would overflow the int64 field component kappa");
  cudaError_t e = cudaSetDevice(ctx->device);
  if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
  e = cudaGetLastError();  // surface earlier asynchronous faults
  if (e != cudaSuccess) return cuda_fail(e, "pending CUDA error");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(cuda_stream);

  RunArgs a;
  memset(&a, 0, sizeof(a));
  a.blob = ctx->d_blob; a.hdr = ctx->d_hdr; a.blob_bytes = ctx->blob_bytes;
  a.a_off = ctx->a_off; a.c_off = ctx->c_off; a.x_off = ctx->x_off;
  a.n = ctx->n; a.M = ctx->M;
  a.Wn = (ctx->n + 31) / 32; a.WN = (ctx->N_max + 31) / 32;
  a.R = R; a.rep0 = rep0; a.K = K; a.T = T;
  a.seed = seed; a.beta_max = ctx->beta_max;
  for (int r = 0; r < 10; ++r) {
    a.ks[2 * r] = (uint32_t)seed + (uint32_t)r * 0x9E3779B9u;
    a.ks[2 * r + 1] = (uint32_t)(seed >> 32) + (uint32_t)r * 0xBB67AE85u;
  }
  a.flags = ctx->flags;
  a.rtol2 = 2.0f * (float)ctx->r_tol;
  a.out = *out;
  saim_init_outputs<<<(ctx->n_inst + 255) / 256, 256, 0, st>>>(out->inst_best, ctx->n_inst, out->counters);
  if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "init launch");

  // Launch geometry (warps per CTA and the grid's x extent) of the selected kernel.
  int wpc = 1, gx = 1;
  bool prod = false;
  if (ctx->kernel == 1) {
    const long long warps = (long long)R * ctx->n_inst;
    wpc = (int)((warps + ctx->sm_count - 1) / ctx->sm_count);
    wpc = std::max(1, std::min(wpc, ctx->max_wpc));
    gx = (R + wpc - 1) / wpc;
  } else if (ctx->mkp_kind == 0) {
    const long long warps = (long long)((R + 31) / 32) * ctx->n_inst;   // 32 replicas per warp (lockstep)
    wpc = (int)((warps + ctx->sm_count - 1) / ctx->sm_count);
    // producer warps when the consumers still fit one wave with their partners
    prod = !(ctx->flags & SAIM_FLAG_MKP_NO_PRODUCER) && wpc <= ctx->max_wpc_prod;
    a.mkp_prod = prod ? 1 : 0;
    wpc = std::max(1, std::min(wpc, prod ? ctx->max_wpc_prod : ctx->max_wpc));
    gx = ((R + 31) / 32 + wpc - 1) / wpc;
  } else if (ctx->mkp_kind == 3) {
    // speculative sub-warp kernel: the whole grid resident in one wave if registers and shared
    // memory allow, with the fewest warps on the fullest SM (then the smallest CTAs: even spread);
    // otherwise one CTA per SM and the fewest waves x warps per CTA
    const int C = 32 / ctx->lanes;
    const int warps_inst = (R + C - 1) / C;
    long long best = -1;
    for (int w = 1; w <= ctx->max_wpc; ++w) {
      const long long ctas = (long long)((warps_inst + w - 1) / w) * ctx->n_inst;
      const long long per_sm = (ctas + ctx->sm_count - 1) / ctx->sm_count;
      const bool fit1 = (long long)ctx->spec_fixed + (long long)w * ctx->per_warp <= ctx->smem_sm &&
                        w * 32LL * std::max(ctx->spec_regs, 1) <= 65536;
      if (!fit1) break;
      const bool fits = per_sm * ((long long)ctx->spec_fixed + (long long)w * ctx->per_warp) <= ctx->smem_sm &&
                        per_sm * w * 32LL * std::max(ctx->spec_regs, 1) <= 65536 && per_sm * w <= 64 && per_sm <= 32;
      const long long cost = fits ? per_sm * w : 1000000LL + per_sm * w;   // (not resident: per_sm = waves)
      if (best < 0 || cost < best) { best = cost; wpc = w; }
    }
    gx = (warps_inst + wpc - 1) / wpc;
  } else {
    // one CTA per SM: spread each instance's warps over floor(SMs / n_inst) CTAs
    const int G = 32 / ctx->lanes;
    const int warps_inst = (R + G - 1) / G;
    const int ctas_inst = std::max(1, ctx->sm_count / ctx->n_inst);
    wpc = (warps_inst + ctas_inst - 1) / ctas_inst;
    wpc = std::max(1, std::min(wpc, ctx->max_wpc));
    gx = (warps_inst + wpc - 1) / wpc;
  }
  // Exact-replay flags: one byte per warp slot of the grid, zeroed every run.
  const size_t need = (size_t)ctx->n_inst * (size_t)gx * 32u;
  if (need > ctx->replay_cap) {
    if (ctx->d_replay) cudaFree(ctx->d_replay);
    ctx->d_replay = nullptr;
    ctx->replay_cap = 0;
    if ((e = cudaMalloc(&ctx->d_replay, need)) != cudaSuccess) return cuda_fail(e, "cudaMalloc replay flags");
    ctx->replay_cap = need;
  }
  a.replay = ctx->d_replay;
  if ((e = cudaMemsetAsync(ctx->d_replay, 0, need, st)) != cudaSuccess) return cuda_fail(e, "replay flags");

  // The main kernel, then the exact replay over the same grid: it re-runs only warps the main
  // kernel flagged (a decision its fp64 level could not certify) and its CTAs exit at once when
  // there are none -- the usual case.
  for (int pass = 0; pass < 2 && e == cudaSuccess; ++pass) {
    const bool replay = pass == 1;
    if (ctx->kernel == 1)
      e = qkp_launch(ctx->npl, ctx->qb, ctx->pk, a, ctx->n_inst, wpc, ctx->smem_bytes, st, replay);
    else if (ctx->mkp_kind == 0)
      e = mkp_launch(a, ctx->n_inst, ctx->mm, wpc, prod ? ctx->per_warp_prod : ctx->per_warp, st, replay);
    else if (ctx->mkp_kind == 1)
      e = mkpt_launch(a, ctx->n_inst, ctx->mm, ctx->lanes, wpc, ctx->per_warp, st, replay);
    else if (ctx->mkp_kind == 3)
      e = mkpx_launch(a, ctx->n_inst, ctx->mm, ctx->lanes, wpc, ctx->per_warp, st, replay);
    else
      e = mkps_launch(a, ctx->n_inst, ctx->mm, wpc, ctx->per_warp, st, replay);
  }
  if (e != cudaSuccess) return cuda_fail(e, "kernel launch");
  return SAIM_OK;
}

extern "C" int saim_get_info(const saim_ctx *ctx, saim_info *out) {
  if (!ctx || !out) return fail(SAIM_EINVAL, "null argument");
  out->n_inst = ctx->n_inst; out->n_items = ctx->n; out->n_cons = ctx->M;
  out->n_spins_max = ctx->N_max;
  out->words_items = (ctx->n + 31) / 32;
  out->words_full = (ctx->N_max + 31) / 32;
  out->kernel = ctx->kernel;
  out->smem_bytes = ctx->smem_bytes;
  out->q_bytes = ctx->kernel == 1 ? ctx->qb : 0;
  out->phi_packed = ctx->kernel == 1 ? ctx->pk : 0;
  out->lanes_per_replica = ctx->lanes;
  return SAIM_OK;
}

extern "C" int saim_get_instance(const saim_ctx *ctx, int32_t inst, int32_t *N, int64_t *s_o, int64_t *s_c, int32_t *q) {
  if (!ctx || inst < 0 || inst >= ctx->n_inst) return fail(SAIM_EINVAL, "bad instance index");
  const InstHdr &h = ctx->hdr[inst];
  if (N) *N = h.N;
  if (s_o) *s_o = h.s_o;
  if (s_c) *s_c = h.s_c;
  if (q) for (int k = 0; k < ctx->M; ++k) q[k] = ctx->q[inst][k];
  return SAIM_OK;
}

extern "C" void saim_destroy(saim_ctx *ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  if (ctx->d_blob) cudaFree(ctx->d_blob);
  if (ctx->d_hdr) cudaFree(ctx->d_hdr);
  if (ctx->d_replay) cudaFree(ctx->d_replay);
  delete ctx;
}

extern "C" int saim_selftest(int which, int device, int n, const uint32_t *in_u32, uint32_t *out_u32, double *out_f64) {
  g_err.clear();
  if (((which == 0 || which == 2) && (n < 1 || !in_u32 || !out_u32)) || (which == 1 && !out_f64) ||
      (which == 3 && (n < 1 || !in_u32 || !out_f64)) || which < 0 || which > 3)
    return fail(SAIM_EINVAL, "bad selftest arguments");
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
  if (which == 3) {
    const double *tab = nullptr;
    if ((e = logit_table(device, &tab)) != cudaSuccess) return cuda_fail(e, "logit table");
    uint32_t *d_w = nullptr;
    double *d_o = nullptr;
    if ((e = cudaMalloc(&d_w, sizeof(uint32_t) * (size_t)n)) != cudaSuccess) return cuda_fail(e, "cudaMalloc");
    if ((e = cudaMalloc(&d_o, sizeof(double) * 2 * (size_t)n)) != cudaSuccess) { cudaFree(d_w); return cuda_fail(e, "cudaMalloc"); }
    cudaMemcpy(d_w, in_u32, sizeof(uint32_t) * (size_t)n, cudaMemcpyHostToDevice);
    saim_selftest_logit_table_kernel<<<(n + 127) / 128, 128>>>(tab, d_w, d_o, n);
    e = cudaMemcpy(out_f64, d_o, sizeof(double) * 2 * (size_t)n, cudaMemcpyDeviceToHost);
    cudaFree(d_w);
    cudaFree(d_o);
    return e == cudaSuccess ? SAIM_OK : cuda_fail(e, "selftest 3");
  }
  if (selftest(which, n, in_u32, out_u32, out_f64) != 0) return fail(SAIM_ECUDA, "selftest failed");
  return SAIM_OK;
}
