// saim_mkp.cuh -- fused SAIM kernel for linear objectives with 2 <= M <= 32 constraints (MKP,
// PAPER.md:321-326; BASELINE.json configs 3-4).  sm_100a.
//
// Mapping: one LANE = one replica, one warp = 32 replicas of the same instance
// marching through the spins in lockstep.  Every lane makes every decision of its own chain in
// the exact sequential order of Algorithm 1 / Eq. 9-10 -- there is no speculation, so the ~25%
// flip rate of MKP anneals costs nothing extra -- while the instance data a step needs (the item
// column A_{.i}, its constants) is the same for all lanes: one shared-memory broadcast.
//
// Items are decided one after the other; the slack bits of different rows, whose fields involve
// their own row's residual only, are decided interleaved (the rows' sequences are independent once
// the items are done, so the decisions are those of the sequential sweep).
//
// Field of spin i (R1), with r = A_ext x - b, Lambda the Lagrange accumulator (R10):
//   item i:   F_i = -c_o c_i - c_p a_i (1 - 2x_i) - 2 c_p (A_{.i} . r) - c_l (A_{.i} . Lambda)
//   slack bit q of row m (A = 2^q):  F = -A (2 c_p r_m + c_l Lambda_m) - c_p A^2 (1 - 2x)
// r is kept as exact integers in fp32 registers (|r| < 2^21, host-proven); the dot products are
// fp32 with a rigorous error bound; c_l Lambda_m is rounded once per iteration.
// Decisions are certified exactly as in the QKP kernel: saturated test, fp32 logit band, fp64
// slow path (counted when even that is not certain).
#pragma once
#include <algorithm>
#include <climits>
#include <cstdint>
#include <cstdio>
#include <type_traits>

#include "saim_dev.cuh"

#ifndef SAIM_MKP_SLACKB
#define SAIM_MKP_SLACKB 4   // rows of slack bits taken interleaved at MM = 32
#endif
#ifndef SAIM_MKP_FILL_UNROLL
#define SAIM_MKP_FILL_UNROLL 4   // Philox calls in flight per lane when a group's logits are drawn
#endif
#ifndef SAIM_MKP_SLACKB_SMALL
#define SAIM_MKP_SLACKB_SMALL 2   // ... at MM <= 16 (128-register instantiations)
#endif

namespace saim {

namespace {

constexpr uint32_t kFull = 0xffffffffu;
constexpr int kFillUnroll = SAIM_MKP_FILL_UNROLL;

// fp64 tail of the slow path: z and its magnitude sum S are accurate to ~2^-50 S; returns
// (x | uncertified << 1).
__device__ __noinline__ int certify_fp64(double zz, double S, uint32_t w) {
  const double d = zz - logit_f64_calc(w);
  return (d > 0.0 ? 1 : 0) | (fabs(d) <= (S + 1.0 + fabs(zz)) * 0x1p-46 ? 2 : 0);
}

// Uniform word of spin i (R2) recomputed for the slow path.
__device__ __noinline__ uint32_t word_of(uint2 key, int i, int t, int k, uint32_t srho) {
  const uint4 w4 = philox_group(key, i >> 7, i & 31, t, k, srho);
  const int j = (i >> 5) & 3;
  return j == 0 ? w4.x : (j == 1 ? w4.y : (j == 2 ? w4.z : w4.w));
}

// logit(u) in fp32 with its sign made exact (sign(logit u) = sign(u - 1/2) <=> w >= 2^31).
__device__ __forceinline__ float logit_signed(uint32_t w) {
  const float l = fabsf(logit_f32(w));
  return (w >> 31) ? l : -l;
}

// mbarrier helpers for the consumer/producer pairs (shared::cta, one phase per buffer fill).
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
  }
}

// 16 bytes of read-only shared memory (item columns) by shared-window address
__device__ __forceinline__ float4 lds_f4(uint32_t a) {
  float4 v;
  asm("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}

template <int MM>
struct MkpCfg {
  static constexpr int kThreads = MM <= 16 ? 512 : 256;
};

}  // namespace

// MM: padded constraint count (layout); MA <= MM: rows the arithmetic loops cover (= M for the
// instantiated exact sizes, else MM with zero-padded rows).
template <int MM, int MA, bool PROD, bool RP>
__global__ void __launch_bounds__(MkpCfg<MM>::kThreads, 1) saim_mkp_kernel(const RunArgs a) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ uint64_t mbar;

  const int s = blockIdx.y;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // Producer warps (a.mkp_prod): the CTA's second half of warps draws the logits
  // of the first half's replicas -- state-independent -- into double-buffered groups, so the
  // consumers' instruction stream (one warp per SMSP: issue-limited per warp) is decisions only.
  constexpr bool prod = PROD;                          // (a.mkp_prod selects this instantiation)
  const int nc = prod ? (int)(blockDim.x >> 6) : (int)(blockDim.x >> 5);   // consumer warps per CTA
  const bool producer = prod && warp >= nc;
  const int cw = producer ? warp - nc : warp;          // consumer warp (own, or the partner's)
  unsigned char *wbase = smem + a.blob_bytes + cw * mkp_warp_bytes(a.WN, MM, prod ? 1 : 0);
  const uint32_t lbytes = (prod ? 2u : 1u) * 128u * 128u;
  uint64_t *mb = reinterpret_cast<uint64_t *>(wbase + align16u(a.WN * 128u) + lbytes + MM * 256u);  // full[2], empty[2]
  if constexpr (RP) {                                  // exact replay: only CTAs holding a flagged warp
    if (!__syncthreads_or(a.replay[replay_slot(cw)] != 0)) return;
  }
  if (prod && !producer && lane == 0) {
#pragma unroll
    for (int i = 0; i < 4; ++i) mbar_init(mb + i, 32);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  bulk_stage(smem, a.blob + (size_t)s * a.blob_bytes, a.blob_bytes, &mbar);   // (includes __syncthreads)

  const int ridx = (blockIdx.x * nc + cw) * 32 + lane;
  const int wfirst = (blockIdx.x * nc + cw) * 32;
  if (wfirst >= a.R) return;                         // whole warp beyond R (its partner too)
  const bool live = ridx < a.R;                        // lanes beyond R compute but never write
  const int rho = a.rep0 + (live ? ridx : a.R - 1);
  const InstHdr *Hp = a.hdr + s;
  const int n = a.n, M = a.M;
  const int N = Hp->N;
  const MkpLayout L = mkp_layout(n, MM);
  const float *sAcol = reinterpret_cast<const float *>(smem + L.acol);
  uint32_t acol_sa = smem_u32(sAcol);                  // the item columns as a shared-window address
  asm volatile("" : "+r"(acol_sa));
  const float4 *sIc = reinterpret_cast<const float4 *>(smem + L.iconst);
  const int32_t *sC = reinterpret_cast<const int32_t *>(smem + L.cint);
  const long long *sB = reinterpret_cast<const long long *>(smem + L.brow);
  const int32_t *sQ = reinterpret_cast<const int32_t *>(smem + L.qrow);
  uint32_t *xw = reinterpret_cast<uint32_t *>(wbase) + lane;                            // word w: xw[32 w]
  // logit of spin i of the current group: lt[loff + 32 (i & 127)] (with producers, successive
  // groups alternate between two buffers, loff = 0 or 4096)
  float *lt = reinterpret_cast<float *>(wbase + align16u(a.WN * 128u)) + lane;
  long long *Lam = reinterpret_cast<long long *>(wbase + align16u(a.WN * 128u) + lbytes) + lane;  // [m]
  // per-lane copies of r and c_l Lambda indexed by row (slack phase): rs[32 m], cLs[32 m]
  float *rs = reinterpret_cast<float *>(wbase + align16u(a.WN * 128u) + lbytes + MM * 256u + (prod ? 32u : 0u)) + lane;
  float *cLs = rs + MM * 32;

  if (producer) {
    // The consumer takes the groups g = 0 .. NG-1 of every sweep t of every iteration k in order
    // (fill f = running index): buffer f & 1, full[f & 1] completes its (f >> 1)-th phase when
    // filled, empty[f & 1] when the consumer has moved past it.
    const uint2 pkey = make_uint2((uint32_t)a.seed, (uint32_t)(a.seed >> 32));
    const uint32_t psrho = ((uint32_t)s << 20) | (uint32_t)rho;
    const int NG = (N + 127) >> 7;
    uint32_t f = 0;
    for (int k = 0; k < a.K; ++k)
      for (int t = 0; t < a.T; ++t)
        for (int g = 0; g < NG; ++g, ++f) {
          const uint32_t b = f & 1u;
          if (f >= 2) mbar_wait(mb + 2 + b, ((f >> 1) - 1u) & 1u);
          float *dst = lt + 32 * 128 * b;
          const int nw = min(4, (N - 128 * g + 31) >> 5);
#pragma unroll 4
          for (int j = 0; j < 32; ++j) {
            const uint4 w4 = philox_group(pkey, g, j, t, k, psrho);
            dst[32 * (j + 0)] = logit_signed(w4.x);
            if (nw > 1) dst[32 * (j + 32)] = logit_signed(w4.y);
            if (nw > 2) dst[32 * (j + 64)] = logit_signed(w4.z);
            if (nw > 3) dst[32 * (j + 96)] = logit_signed(w4.w);
          }
          mbar_arrive(mb + b);
        }
    return;
  }

  const double c_o = Hp->c_o, c_p = Hp->c_p, c_l = Hp->c_l;
  const float twocp = (float)(2.0 * c_p), cpf = (float)c_p;
  const float rbound = (float)Hp->r_bound;
  const float amax = (float)(Hp->v_bound - 2.0 * Hp->r_bound);   // max A_ext entry
  const float *sBand = reinterpret_cast<const float *>(smem + L.band);

  float r[MM], cL[MM];
#pragma unroll
  for (int m = 0; m < MM; ++m) {
    r[m] = m < M ? (float)(-sB[m]) : 0.0f;             // x = 0: r = -b
    cL[m] = 0.0f;
    Lam[32 * m] = 0;
  }
  for (int w = 0; w < a.WN; ++w) xw[32 * w] = 0u;
  long long best_f = LLONG_MAX;
  int best_k = -1, nfeas = 0;
  uint32_t c_flips = 0, c_unif = 0, c_fp64 = 0, c_unc = 0, c_philox = 0;
  const uint2 key = make_uint2((uint32_t)a.seed, (uint32_t)(a.seed >> 32));
  const uint32_t srho = ((uint32_t)s << 20) | (uint32_t)rho;
  const double bstep = (a.T >= 2) ? a.beta_max / (double)(a.T - 1) : a.beta_max;
  const int Wn = (n + 31) >> 5;
  uint32_t pf = 0;                                     // groups taken from the producer so far
  int loff = 0;                                        // buffer of the current group (0 without producers)

  for (int k = 0; k < a.K; ++k) {
    // ---- per-iteration constants: c_l Lambda_m (rounded once), error-bound slope E1 ----
    float cLmax = 0.0f;
#pragma unroll
    for (int m = 0; m < MM; ++m) {
      cL[m] = (float)(c_l * (double)Lam[32 * m]);
      cLs[32 * m] = cL[m];
      cLmax = fmaxf(cLmax, fabsf(cL[m]));
    }
    // |z_f32 - z| <= beta (E1 |A_i|_1 + E0_i) + 2^-23 |z|, E = (MM+8) 2^-24 (...):
    // the lookahead's band value adds |A_i . A_{i-1}| <= |A_i|_1 max A; factor 2: safety margin.
    // + 2^-22 |z| folded in with |z| <= beta (|c_o c_i| + c_p a_i + |A_i|_1 (2 c_p r_max + max|c_l Lambda|))
    const double Wk = 2.0 * c_p * ((double)rbound + (double)amax) + (double)cLmax;
    const float E1 = (float)((MM + 8) * 0x1p-24 * Wk * 2.0 + 0x1p-22 * Wk * 1.01);

    for (int t = 0; t < a.T; ++t) {
      const bool bz = (a.T >= 2) && (t == 0);          // beta_0 = 0: x_i = [u < 1/2]
      const double beta = (a.T >= 2) ? bstep * (double)t : a.beta_max;
      const float bf = (float)beta;
      uint32_t xcur = 0;

      // Logits of the uniforms of spins 128g .. 128g+127 (R2: the Philox call of counter
      // (32g + j, t, k, s<<20|rho) yields the words of spins 128g + 32w + j, w = 0..3).  They do
      // not depend on the state, so they are drawn in one ILP-friendly burst per group, off the
      // sequential dependency chain of the decisions.
      // Software-pipelined by one step of 4 calls: the logits (two MUFU each, XU pipe) of the
      // previous 4 calls are taken next to the Philox rounds (IMAD/LOP3) of the next 4, so a warp
      // alone on its SMSP has both pipes busy instead of one after the other.
      auto fill_words = [&](int g, auto NW) {              // NW = words of the group holding spins
        auto put = [&](int j, const uint4 &w4) {
          lt[32 * (j + 0)] = logit_signed(w4.x);
          if (NW.value > 1) lt[32 * (j + 32)] = logit_signed(w4.y);
          if (NW.value > 2) lt[32 * (j + 64)] = logit_signed(w4.z);
          if (NW.value > 3) lt[32 * (j + 96)] = logit_signed(w4.w);
        };
        uint4 wq[kFillUnroll];
#pragma unroll
        for (int b = 0; b < kFillUnroll; ++b) wq[b] = philox_group(key, g, b, t, k, srho);
#pragma unroll 1
        for (int j0 = kFillUnroll; j0 < 32; j0 += kFillUnroll) {
          uint4 wn[kFillUnroll];
#pragma unroll
          for (int b = 0; b < kFillUnroll; ++b) wn[b] = philox_group(key, g, j0 + b, t, k, srho);
#pragma unroll
          for (int b = 0; b < kFillUnroll; ++b) put(j0 - kFillUnroll + b, wq[b]);
#pragma unroll
          for (int b = 0; b < kFillUnroll; ++b) wq[b] = wn[b];
        }
#pragma unroll
        for (int b = 0; b < kFillUnroll; ++b) put(32 - kFillUnroll + b, wq[b]);
      };
      auto fill_group = [&](int g) {
        if (prod) {                                        // the producer's buffer (g & 1)
          if (pf >= 1) mbar_arrive(mb + 2 + ((pf - 1u) & 1u));   // done with the previous group
          mbar_wait(mb + (pf & 1u), (pf >> 1) & 1u);
          loff = (int)(pf & 1u) * (32 * 128);
          ++pf;
        } else {
          const int nw = min(4, (N - 128 * g + 31) >> 5);
          if (nw >= 4) fill_words(g, std::integral_constant<int, 4>{});
          else if (nw == 3) fill_words(g, std::integral_constant<int, 3>{});
          else if (nw == 2) fill_words(g, std::integral_constant<int, 2>{});
          else fill_words(g, std::integral_constant<int, 1>{});
        }
        c_philox += 32;
      };
      // Certified decision [u < sigma(z)] (R18, R19) from z, its error bound e and l = logit(u)
      // (exact sign), evaluated branch-free; only the rare fp64 re-evaluation (slow(): returns
      // x | uncertified << 1) sits behind a warp vote.
      auto decide = [&](float z, float e, float l, auto slow) -> int {
        // e bounds |z_f32 - z| for every reachable state and does not depend on z, so both
        // thresholds are ready before z: the dependency chain is z -> d -> compare.
        const float satT = e + kSatThr;
        const float certT = (e + kLogitAbs + kLogitRel * fabsf(l)) * 1.0001f;
        const float d = z - l;
        const bool sat = fabsf(z) > satT;
        int nx = sat ? (z > 0.0f) : (d > 0.0f);
        if (bz) nx = (int)(__float_as_uint(l) >> 31);     // beta_0 = 0: u < 1/2 (sign bit, -0 included)
        c_unif += (!bz && !sat) ? 1u : 0u;
        const bool need = !bz && !sat && !(fabsf(d) > certT);
        // (the whole warp takes the slow path when some lane needs it -- its result is used by those
        // lanes only: a warp-uniform branch, so the common path carries no reconvergence barrier)
        if (__any_sync(kFull, need)) {
          const int rs = slow();
          if (need) {
            ++c_fp64;
            if (rs & 2) ++c_unc;
            nx = rs & 1;
          }
        }
        return nx;
      };

      // ---- items i = 0..n-1, with a one-spin lookahead ----
      // pre = A_i . r evaluated with r as it was BEFORE the decision of spin i-1 (so it is computed
      // off the sequential dependency chain, during step i-1); the exact dot follows from one fma
      // with the band value G_i = A_i . A_{i-1}:  A_i . r_now = pre + delta_{i-1} G_i.
      // A column is read from shared memory once: the lookahead of step i loads column i + 1 into
      // registers for its dot products, and step i + 1 updates r from the same registers (two
      // columns live, the item loop unrolled by two so they alternate without moves).  The loads go
      // through a 32-bit shared-window address (through the generic pointer the compiler rebuilt
      // the window base -- S2R SR_CgaCtaId, MOV, LEA -- in every step).
      constexpr int NC4 = (MA + 3) / 4;
      auto ldcol = [&](int i, float4 (&c)[NC4]) {
        const uint32_t ca = acol_sa + (uint32_t)i * (MM * 4u);
#pragma unroll
        for (int m4 = 0; m4 < NC4; ++m4) c[m4] = lds_f4(ca + 16u * m4);
      };
      auto dots = [&](const float4 (&c)[NC4], float &pr, float &dlv) {
        // four partial sums per dot product (short dependency chains; each term still passes at
        // most MA/4 + 2 roundings, inside the (MM + 8) 2^-24 bound of E1)
        float dr0 = 0.f, dr1 = 0.f, dr2 = 0.f, dr3 = 0.f, dl0 = 0.f, dl1 = 0.f, dl2 = 0.f, dl3 = 0.f;
#pragma unroll
        for (int m4 = 0; m4 < NC4; ++m4) {
          const float4 av = c[m4];
          dr0 = fmaf(av.x, r[4 * m4 + 0], dr0);
          dl0 = fmaf(av.x, cL[4 * m4 + 0], dl0);
          if (4 * m4 + 1 < MA) { dr1 = fmaf(av.y, r[4 * m4 + 1], dr1); dl1 = fmaf(av.y, cL[4 * m4 + 1], dl1); }
          if (4 * m4 + 2 < MA) { dr2 = fmaf(av.z, r[4 * m4 + 2], dr2); dl2 = fmaf(av.z, cL[4 * m4 + 2], dl2); }
          if (4 * m4 + 3 < MA) { dr3 = fmaf(av.w, r[4 * m4 + 3], dr3); dl3 = fmaf(av.w, cL[4 * m4 + 3], dl3); }
        }
        pr = (dr0 + dr1) + (dr2 + dr3);
        dlv = (dl0 + dl1) + (dl2 + dl3);
      };
      float pre = 0.f, dlc = 0.f, dprev = 0.f, Gc = 0.f;
      float4 colA[NC4], colB[NC4];
      ldcol(0, colA);
      dots(colA, pre, dlc);                               // (column n is zero: the lookahead past n-1 is harmless)
      float l = 0.f, G_n = 0.f;
      float4 ic = make_float4(0.f, 0.f, 0.f, 0.f);
      // one item step: decision of spin i = 32 w + ii with column i in cur; the lookahead fills nxt
      auto item_step = [&](int i, int ii, const float4 (&cur)[NC4], float4 (&nxt)[NC4]) {
        const float l_n = lt[loff + 32 * ((i + 1) & 127)];       // valid for ii + 1 < iend (same group)
        const float4 ic_n = sIc[i + 1];                   // padded entry n
        const float G_nn = sBand[i + 2 <= n ? i + 2 : n];
        const int xb = (xcur >> ii) & 1u;
        const float dr = fmaf(dprev, Gc, pre);            // A_i . r (current state)
        float pre_n, dl_n;
        ldcol(i + 1, nxt);
        dots(nxt, pre_n, dl_n);                           // lookahead (independent of this decision)
#ifndef SAIM_MKP_NO_PIN
        // keep the lookahead's FMAs ahead of the slow-path branch, next to the decision chain they
        // are meant to overlap (in one of the two unrolled steps the compiler sank them behind it)
        asm volatile("" : "+f"(pre_n), "+f"(dl_n));
#endif
        const float sg = xb ? -1.0f : 1.0f;               // 1 - 2 x_i
        const float F = fmaf(-twocp, dr, fmaf(-ic.y, sg, ic.x)) - dlc;
        const float z = bf * F;
        const float e = bf * fmaf(E1, ic.z, ic.w);
        const int nx = decide(z, e, l, [&]() -> int {
          const uint32_t wd = word_of(key, i, t, k, srho);
          double drd = 0.0, dld = 0.0, a2 = 0.0;
#pragma unroll
          for (int m = 0; m < MM; ++m) {
            const double Am = (double)sAcol[i * MM + m];
            drd += Am * (double)r[m];
            dld += Am * (double)Lam[32 * m];
            a2 += Am * Am;
          }
          const double t1 = c_o * (double)sC[i], t2 = c_p * a2, t3 = 2.0 * c_p * drd, t4 = c_l * dld;
          const double zz = beta * (-t1 - t2 * (1.0 - 2.0 * xb) - t3 - t4);
          const int rs = certify_fp64(zz, beta * (fabs(t1) + fabs(t2) + fabs(t3) + fabs(t4)), wd);
          if constexpr (RP) {                            // double-double level: replay kernel only
            if ((rs & 2) || (a.flags & SAIM_FLAG_TEST_REPLAY)) {
              // double-double level on the exact integers (drd, a2 exact in fp64; kappa in int64)
              long long kap = 0;
              for (int m = 0; m < MA; ++m) kap += (long long)sAcol[i * MM + m] * Lam[32 * m];
              return decide_dd(-(long long)sC[i], 2 * (long long)drd + (long long)a2 * (1 - 2 * xb), kap, a.T >= 2 ? t : 1, a.T >= 2 ? a.T - 1 : 1, Hp, wd);
            }
          }
          return rs;
        });
        const float dl = (nx != xb) ? sg : 0.0f;          // delta in {-1, 0, +1}; fma(0, A, r) == r
#pragma unroll
        for (int m4 = 0; m4 < NC4; ++m4) {
          const float4 av = cur[m4];
          r[4 * m4 + 0] = fmaf(dl, av.x, r[4 * m4 + 0]);
          if (4 * m4 + 1 < MA) r[4 * m4 + 1] = fmaf(dl, av.y, r[4 * m4 + 1]);
          if (4 * m4 + 2 < MA) r[4 * m4 + 2] = fmaf(dl, av.z, r[4 * m4 + 2]);
          if (4 * m4 + 3 < MA) r[4 * m4 + 3] = fmaf(dl, av.w, r[4 * m4 + 3]);
        }
        xcur ^= (uint32_t)(nx != xb) << ii;
        c_flips += (nx != xb) ? 1u : 0u;
        pre = pre_n; dlc = dl_n; Gc = G_n; dprev = dl;
        l = l_n; ic = ic_n; G_n = G_nn;
      };
      for (int w = 0; 32 * w < n; ++w) {
        xcur = xw[32 * w];
        if ((w & 3) == 0) fill_group(w >> 2);
        const int iend = min(32, n - 32 * w);
        // state-independent operands of the current step, prefetched one step ahead
        l = lt[loff + 32 * ((32 * w) & 127)];
        ic = sIc[32 * w];                                 // (-c_o c_i, c_p a_i, |A_i|_1, E0_i)
        G_n = sBand[32 * w + 1];
        int ii = 0;
        for (; ii + 1 < iend; ii += 2) {
          item_step(32 * w + ii, ii, colA, colB);
          item_step(32 * w + ii + 1, ii + 1, colB, colA);
        }
        if (ii < iend) {                                  // odd tail: one step, then the next column becomes colA
          item_step(32 * w + ii, ii, colA, colB);
#pragma unroll
          for (int m4 = 0; m4 < NC4; ++m4) colA[m4] = colB[m4];
        }
        xw[32 * w] = xcur;
      }
      // ---- slack bits: row m, bit q, spin i = n + sum_{m'<m} q_m' + q (R4) ----
      // The field of a slack bit of row m involves r_m only, and after the items r_m is moved by
      // row m's own slack bits alone: the rows' decision sequences are independent of each other, so
      // taking them interleaved -- SB rows at a time, bit by bit, each row's bits in order -- gives
      // exactly the decisions of the sequential sweep (same state seen, same counter-based
      // uniforms), with SB independent dependency chains in flight instead of one.  The rows are
      // indexed dynamically, so r moves to per-lane shared memory for this phase (rs) and each
      // row's slack bits are held as one register (sv).  The logits stay in the one-group buffer:
      // a pass per 128-spin group takes the bits of every row that lie inside the group.
#pragma unroll
      for (int m = 0; m < MA; ++m) rs[32 * m] = r[m];
      // One batch step takes bit q of every row of the batch (a row is "on" while q is inside its
      // bit range of this pass), so everything that depends on q alone -- A = 2^q and the
      // products beta A, beta c_p A^2, the error-bound factors, the bit mask -- is shared by the
      // rows and doubled from step to step (exact scalings).  z = fma(-beta A, fma(2c_p, r, c_l
      // Lambda), -+ beta c_p A^2): 4 roundings' worth against the 12 the bound e allows (DESIGN 6.2).
      auto slack_phase = [&](auto BZ) {
        constexpr bool kBz = decltype(BZ)::value;          // sweep 0 (beta = 0): x = [u < 1/2], the logit's sign
        constexpr int SB = MM >= 32 ? SAIM_MKP_SLACKB : SAIM_MKP_SLACKB_SMALL;
        constexpr float kC = 8.0f * 0x1p-24f + 1.01f * 0x1p-22f;
        constexpr float kLA1 = kLogitAbs * 1.0001f, kLR1 = kLogitRel * 1.0001f;
        const float bfcp = bf * cpf, bfC = bf * kC, bfCcp = bfC * cpf;
        int mrow = 0, srow = n;                            // first unfinished row and its first spin
        for (int g = n >> 7; 128 * g < N; ++g) {
          if (128 * g >= n) fill_group(g);                 // (a group the items began is already filled)
          const int glo = max(n, 128 * g), ghi = min(N, 128 * g + 128);
          const float *ltg = lt + loff - 32 * 128 * g;     // logit of spin i of this group: ltg[32 i]
          while (mrow < M && srow < ghi) {
            float rr[SB], cl[SB];
            uint32_t sv[SB], sv0[SB], onm[SB];
            int S[SB], qq[SB];
            int q0 = 32, q1 = 0, sj = srow;
#pragma unroll
            for (int j = 0; j < SB; ++j) {
              const int m = min(mrow + j, M - 1);
              const bool act = mrow + j < M && sj < ghi;
              const int qm = sQ[m];
              S[j] = sj;
              qq[j] = qm;
              const int qa = act ? max(0, glo - sj) : 0;
              const int qb = act ? min(qm, ghi - sj) : 0;
              onm[j] = ((1u << qb) - 1u) & ~((1u << qa) - 1u);     // bits of the row taken in this pass (q < 32)
              rr[j] = rs[32 * m];
              cl[j] = cLs[32 * m];
              const int w0 = min(sj >> 5, a.WN - 1), o = sj & 31;
              const uint32_t lo = xw[32 * w0], hi = xw[32 * min(w0 + 1, a.WN - 1)];
              sv[j] = sv0[j] = __funnelshift_r(lo, hi, o) & ((1u << qm) - 1u);     // (qm <= 21)
              if (qb > qa) { q0 = min(q0, qa); q1 = max(q1, qb); }
              if (mrow + j < M) sj += qm;
            }
            float A = __int_as_float((127 + min(q0, 31)) << 23);      // 2^q
            float bA = bf * A, bcA2 = bfcp * A * A, eA = bfC * A, eA2 = bfCcp * A * A;
            uint32_t bit = 1u << min(q0, 31);
            for (int q = q0; q < q1; ++q) {
              bool needv[SB], flipv[SB];
              bool anyneed = false;
#pragma unroll
              for (int j = 0; j < SB; ++j) {
                const bool on = (onm[j] & bit) != 0u;
                const float l = on ? ltg[32 * (S[j] + q)] : 1.0f;
                const bool xb = (sv[j] & bit) != 0u;
                if constexpr (kBz) {
                  needv[j] = false;
                  flipv[j] = on && ((__float_as_uint(l) >> 31) != 0u) != xb;
                } else {
                  const float s1 = fabsf(twocp * rr[j]) + fabsf(cl[j]);
                  const float inner = fmaf(twocp, rr[j], cl[j]);
                  const float z = fmaf(-bA, inner, xb ? bcA2 : -bcA2);
                  // |z_f32 - z| <= beta (8 2^-24 + 1.01 2^-22) (A (|2 c_p r_m| + |c_l Lambda_m|) + c_p A^2)
                  const float e = fmaf(eA, s1, eA2);
                  const float satT = e + kSatThr;
                  const float certT = fmaf(1.0001f, e, fmaf(kLR1, fabsf(l), kLA1));
                  const float d = z - l;
                  const bool sat = fabsf(z) > satT;
                  const bool nx = (sat ? z : d) > 0.0f;
                  c_unif += (on && !sat) ? 1u : 0u;
                  needv[j] = on && !sat && !(fabsf(d) > certT);
                  anyneed |= needv[j];
                  flipv[j] = on && nx != xb;
                }
              }
              if constexpr (!kBz) {
                // the rare fp64 level, one vote for the SB rows
                if (__any_sync(kFull, anyneed)) {
#pragma unroll
                  for (int j = 0; j < SB; ++j) {
                    if (__any_sync(kFull, needv[j])) {       // (warp-uniform, as in decide())
                      const int i = S[j] + q, m = min(mrow + j, M - 1);
                      const int xb = (sv[j] >> q) & 1u;
                      const uint32_t w = word_of(key, i, t, k, srho);
                      const double Ad = (double)(1u << q);
                      const double t1 = Ad * 2.0 * c_p * (double)rr[j], t2 = Ad * c_l * (double)Lam[32 * m];
                      const double t3 = c_p * Ad * Ad;
                      const double zz = beta * (-t1 - t2 - t3 * (1.0 - 2.0 * xb));
                      int rs2 = certify_fp64(zz, beta * (fabs(t1) + fabs(t2) + fabs(t3)), w);
                      if constexpr (RP) {                  // double-double level: replay kernel only
                        if ((rs2 & 2) || (a.flags & SAIM_FLAG_TEST_REPLAY)) {
                          const long long Ai = 1LL << q;
                          rs2 = decide_dd(0, 2 * Ai * (long long)rr[j] + Ai * Ai * (1 - 2 * xb), Ai * Lam[32 * m],
                                          a.T >= 2 ? t : 1, a.T >= 2 ? a.T - 1 : 1, Hp, w);
                        }
                      }
                      if (needv[j]) {
                        ++c_fp64;
                        if (rs2 & 2) ++c_unc;
                        flipv[j] = (rs2 & 1) != xb;
                      }
                    }
                  }
                }
              }
#pragma unroll
              for (int j = 0; j < SB; ++j) {
                if (flipv[j]) {                            // r_m += delta 2^q, delta = 1 - 2 x
                  rr[j] += (sv[j] & bit) ? -A : A;
                  sv[j] ^= bit;
                }
              }
              A += A; bA += bA; eA += eA;
              bcA2 *= 4.0f; eA2 *= 4.0f;
              bit += bit;
            }
            // write back the rows of the batch that took decisions (every bit is decided once per
            // sweep, so the flips are the changed bits); rows completed leave the queue
#pragma unroll
            for (int j = 0; j < SB; ++j) {
              if (onm[j]) {
                c_flips += __popc(sv[j] ^ sv0[j]);
                rs[32 * (mrow + j)] = rr[j];
                const int w0 = S[j] >> 5, o = S[j] & 31;
                const uint32_t mask = (1u << qq[j]) - 1u;
                xw[32 * w0] = (xw[32 * w0] & ~(mask << o)) | (sv[j] << o);
                if (o + qq[j] > 32) xw[32 * (w0 + 1)] = (xw[32 * (w0 + 1)] & ~(mask >> (32 - o))) | (sv[j] >> (32 - o));
              }
            }
            // advance past the rows whose last bit lies inside this group
            int adv = 0, snext = srow;
#pragma unroll
            for (int j = 0; j < SB; ++j) {
              if (mrow + j < M && S[j] + qq[j] <= ghi && adv == j) { ++adv; snext = S[j] + qq[j]; }
            }
            mrow += adv;
            srow = snext;
            if (adv < SB) break;                           // row mrow (if any) continues in the next group
          }
        }
      };
      if (bz) slack_phase(std::true_type{});
      else slack_phase(std::false_type{});
#pragma unroll
      for (int m = 0; m < MA; ++m) r[m] = rs[32 * m];
    }

    // ---- readout of x_k: f, feasibility, trace, best, Lagrange step ----
    long long f = 0;
    for (int w = 0; w < Wn; ++w) {
      uint32_t bits = xw[32 * w];
      if (32 * w + 32 > n) bits &= (1u << (n - 32 * w)) - 1u;
      while (bits) {
        const int b = __ffs(bits) - 1;
        bits &= bits - 1u;
        f += sC[32 * w + b];
      }
    }
    // feasible <=> A x_items <= b  <=>  r_m <= (slack value of row m) for every row (R12)
    bool feas = true;
    {
      int i0 = n;
#pragma unroll
      for (int m = 0; m < MM; ++m) {
        const int qm = (m < M) ? sQ[m] : 0;
        if (qm > 0) {
          long long sv = 0;
          for (int q = 0; q < qm; ++q) {
            const int i = i0 + q;
            sv += (long long)((xw[32 * (i >> 5)] >> (i & 31)) & 1u) << q;
          }
          if ((long long)r[m] > sv) feas = false;
        }
        i0 += qm;
      }
    }
    const size_t row = ((size_t)s * a.R + ridx) * a.K + k;
    if (live) {
      if (a.out.tr_f) a.out.tr_f[row] = f;
      if (a.out.tr_feas) a.out.tr_feas[row] = (uint8_t)feas;
      for (int m = 0; m < M; ++m) {
        if (a.out.tr_lam) a.out.tr_lam[row * M + m] = Lam[32 * m];
      }
      if (a.out.tr_x)
        for (int w = 0; w < a.WN; ++w) a.out.tr_x[row * a.WN + w] = xw[32 * w];
    }
#pragma unroll
    for (int m = 0; m < MM; ++m) {
      if (m < M) {
        const long long rl = (long long)r[m];
        if (live && a.out.tr_r) a.out.tr_r[row * M + m] = rl;
        Lam[32 * m] += rl;                                 // lambda_{k+1} = lambda_k + eta g(x_k) (R10)
      }
    }
    if (feas) {
      ++nfeas;
      if (f < best_f) {
        best_f = f;
        best_k = k;
        if (live) {
          const size_t ri = (size_t)s * a.R + ridx;
          for (int w = 0; w < Wn; ++w) {
            uint32_t bits = xw[32 * w];
            if (32 * w + 32 > n) bits &= (1u << (n - 32 * w)) - 1u;
            a.out.best_x[ri * a.Wn + w] = bits;
          }
        }
      }
    }
  }

  // ---- outputs ----
  const size_t ri = (size_t)s * a.R + ridx;
  if (live) {
    a.out.best_f[ri] = best_f;
    a.out.best_k[ri] = best_k;
    a.out.n_feasible[ri] = nfeas;
    if (best_k < 0)
      for (int w = 0; w < Wn; ++w) a.out.best_x[ri * a.Wn + w] = 0u;
    if (a.out.final_x)
      for (int w = 0; w < a.WN; ++w) a.out.final_x[ri * a.WN + w] = xw[32 * w];
    if (a.out.final_lam)
      for (int m = 0; m < M; ++m) a.out.final_lam[ri * M + m] = Lam[32 * m];
    if (a.out.rep_flips) a.out.rep_flips[ri] = c_flips;
  }
  // per-instance best (f << 20 | rho): warp min, one atomic
  // Exact replay: the main kernel defers a warp in which some decision was not
  // certified by the fp64 level (SAIM_FLAG_TEST_REPLAY: any fp64-level decision) -- the replay
  // kernel re-runs its CTA with the double-double level and only the flagged warps contribute
  // their instance-best candidates and counters (the others did in the main kernel).
  const size_t rslot = replay_slot(cw);
  const bool defer = !RP && __any_sync(kFull, live && (c_unc != 0 || ((a.flags & SAIM_FLAG_TEST_REPLAY) && c_fp64 != 0)));
  const bool contribute = RP ? a.replay[rslot] != 0 : !defer;
  if (defer) {
    const uint32_t nrep = __popc(__ballot_sync(kFull, live));
    if (lane == 0) {
      a.replay[rslot] = 1;
      if (a.out.counters) atomicAdd(reinterpret_cast<unsigned long long *>(a.out.counters) + SAIM_CNT_REPLAYED, (unsigned long long)nrep);
    }
  }
  long long key_best = (live && best_k >= 0) ? ((best_f << 20) | (long long)rho) : LLONG_MAX;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const long long other = __shfl_xor_sync(kFull, key_best, o);
    key_best = other < key_best ? other : key_best;
  }
  if (contribute && lane == 0 && key_best != LLONG_MAX && a.out.inst_best)
    atomicMin(reinterpret_cast<long long *>(a.out.inst_best) + s, key_best);
  if (a.out.counters && contribute) {
    const unsigned long long nl = live ? 1ull : 0ull;
    const unsigned long long fl = warp_sum_u64(nl * c_flips), un = warp_sum_u64(nl * c_unif);
    const unsigned long long fp = warp_sum_u64(nl * c_fp64), uc = warp_sum_u64(nl * c_unc);
    const unsigned long long ph = warp_sum_u64(nl * c_philox), nf = warp_sum_u64(nl * (unsigned long long)nfeas);
    const unsigned long long lv = warp_sum_u64(nl);
    if (lane == 0) {
      unsigned long long *c = reinterpret_cast<unsigned long long *>(a.out.counters);
      atomicAdd(c + SAIM_CNT_DECISIONS, lv * (unsigned long long)a.K * a.T * N);
      atomicAdd(c + SAIM_CNT_FLIPS, fl);
      atomicAdd(c + SAIM_CNT_SWEEPS, lv * (unsigned long long)a.K * a.T);
      atomicAdd(c + SAIM_CNT_UNIFORMS, un);
      atomicAdd(c + SAIM_CNT_FP64, fp);
      atomicAdd(c + SAIM_CNT_UNCERTIFIED, uc);
      atomicAdd(c + SAIM_CNT_FEASIBLE, nf);
      atomicAdd(c + SAIM_CNT_PHILOX, ph);
    }
  }
}

// ---------------------------------------------------------------------------------------------
typedef void (*mkp_kernel_t)(const RunArgs);
// (MM, M) -> kernel (RPV: the exact-replay instantiation).
// Producer-warp instantiations exist for M <= 8 (where one consumer warp per SMSP is the norm).
template <bool RPV>
static mkp_kernel_t mkp_kernel_for_t(int MM, int M, bool prod) {
  if (prod) {
    if (MM == 8 && M == 5) return saim_mkp_kernel<8, 5, true, RPV>;
    if (MM == 4) return saim_mkp_kernel<4, 4, true, RPV>;
    if (MM == 8) return saim_mkp_kernel<8, 8, true, RPV>;
    return nullptr;
  }
  if (MM == 8 && M == 5) return saim_mkp_kernel<8, 5, false, RPV>;
  if (MM == 16 && M == 10) return saim_mkp_kernel<16, 10, false, RPV>;
  if (MM == 32 && M == 30) return saim_mkp_kernel<32, 30, false, RPV>;
  switch (MM) {
    case 4: return saim_mkp_kernel<4, 4, false, RPV>;
    case 8: return saim_mkp_kernel<8, 8, false, RPV>;
    case 16: return saim_mkp_kernel<16, 16, false, RPV>;
    case 32: return saim_mkp_kernel<32, 32, false, RPV>;
    default: return nullptr;
  }
}


}  // namespace saim
