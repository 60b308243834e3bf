// saim_mkp_spec.cuh -- speculative sub-warp SAIM kernel for linear objectives with few constraints
// (MKP; BASELINE.json config 3).  sm_100a.
//
// Mapping: G = 2..32 adjacent LANES = one replica (chain), C = 32/G chains per
// warp.  The chain's lanes form a sliding window over the sweep: they always hold its next G spins
// that are not final yet (spin i belongs to lane G-1 - i mod G; items and slack bits alike: a slack
// bit q of row m is the column 2^q e_m, built into a per-CTA spin table).  One ROUND evaluates, for
// every lane, the decision of its spin on the chain's current state; the first lane in spin order
// whose decision flips is the chain's next state change: the lanes up to it are final and move on
// to their next spins, the flip is applied to r (replicated in the chain's lanes), and the lanes
// after it are evaluated again in the next round with the same counter-based uniforms -- the
// sequential sweep of Eq. 9-10, bit for bit.  A round without a flip finalises
// all G lanes.  The chains of a warp are NOT synchronised: each has its own window position and
// sweep index, so a chain takes exactly (flips + flip-free runs of G spins) rounds per sweep
// whatever its neighbours do; they meet again at the end of the anneal (readout, Lagrange step).
// The logits of a chain's sweep are drawn by all 32 lanes of the warp together when that chain
// enters the sweep.
//
// Why: config 3 has 6,144 chains.  Lane-per-chain (lockstep) makes 192 warps -- one per SMSP on a
// third of the GPU -- and a chain's decision then costs its ~100 warp-instructions at the IPC of
// a lone warp; the outcome trees (L lanes per chain) pay 2^l combinations.  Here a round of ~105
// warp-instructions is shared by C chains and finalises ~4 spins of each.
//
// Arithmetic and certification are those of the lockstep kernel (saim_mkp.cuh): r exact integers
// in fp32, the field F_i = -c_o c_i - c_p a_i (1 - 2x_i) - 2 c_p (A_i . r) - (A_i . c_l Lambda)
// in fp32 with the rigorous bound beta (E1 |A_i|_1 + E0_i) (no lookahead term here), saturation
// test, fp32 logit band, fp64 second level, double-double third level in the replay instantiation.
#pragma once
#include <algorithm>
#include <climits>
#include <cstdint>
#include <cstdio>

#include "saim_dev.cuh"

namespace saim {

namespace {

constexpr uint32_t kFullX = 0xffffffffu;

// fp64 tail of the slow path (as in saim_mkp.cuh): returns (x | uncertified << 1).
__device__ __noinline__ int certify_fp64_x(double zz, double S, uint32_t w) {
  const double d = zz - logit_f64_calc(w);
  return (d > 0.0 ? 1 : 0) | (fabs(d) <= (S + 1.0 + fabs(zz)) * 0x1p-46 ? 2 : 0);
}

// Uniform word of spin i (R2) recomputed for the slow path.
__device__ __noinline__ uint32_t word_of_x(uint2 key, int i, int t, int k, uint32_t srho) {
  const uint4 w4 = philox_group(key, i >> 7, i & 31, t, k, srho);
  const int j = (i >> 5) & 3;
  return j == 0 ? w4.x : (j == 1 ? w4.y : (j == 2 ? w4.z : w4.w));
}

// logit(u) in fp32 with its sign made exact (sign(logit u) = sign(u - 1/2) <=> w >= 2^31).
__device__ __forceinline__ float logit_signed_x(uint32_t w) {
  const float l = fabsf(logit_f32(w));
  return (w >> 31) ? l : -l;
}

// Shared-memory accesses by 32-bit shared-window address (the hot loop keeps such addresses in
// registers; generic pointers made the compiler rebuild the window base in every block load).
__device__ __forceinline__ float4 lds128(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ float lds32f(uint32_t a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t lds32u(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void sts32u(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}

}  // namespace

// MM: padded constraint count (layout); MA <= MM: rows the arithmetic covers; G lanes per chain.
template <int MM, int MA, int G, bool RP>
__global__ void __launch_bounds__((G == 32 ? 672 : (G == 16 ? 352 : 512)), (G == 16 ? 2 : 1)) saim_mkp_spec_kernel(const RunArgs a) {
  static_assert(G == 2 || G == 4 || G == 8 || G == 16 || G == 32, "G must divide 32");
  constexpr int C = 32 / G;
  constexpr uint32_t GM = G == 32 ? 0xffffffffu : ((1u << (G & 31)) - 1u);
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ uint64_t mbar;

  const int s = blockIdx.y;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if constexpr (RP) {                                  // exact replay: only CTAs holding a flagged warp
    if (!__syncthreads_or(a.replay[replay_slot(warp)] != 0)) return;
  }
  bulk_stage(smem, a.blob + (size_t)s * a.blob_bytes, a.blob_bytes, &mbar);

  const InstHdr *Hp = a.hdr + s;
  const int n = a.n, M = a.M;
  const int N = Hp->N;
  const MkpLayout Ly = mkp_layout(n, MM);
  const float *sAcol = reinterpret_cast<const float *>(smem + Ly.acol);
  const float4 *sIc = reinterpret_cast<const float4 *>(smem + Ly.iconst);
  const int32_t *sC = reinterpret_cast<const int32_t *>(smem + Ly.cint);
  const long long *sB = reinterpret_cast<const long long *>(smem + Ly.brow);
  const int32_t *sQ = reinterpret_cast<const int32_t *>(smem + Ly.qrow);
  const double c_o = Hp->c_o, c_p = Hp->c_p, c_l = Hp->c_l;
  const float twocp = (float)(2.0 * c_p), cpf = (float)c_p;

  // ---- spin table (all N spins, padded to NS = 32 WN rows of RS floats): column A_{.i} in slots
  // 0..MM-1 and (c_p a_i, -c_o c_i, |A_i|_1, E0_i); slack bit q of row m: column 2^q e_m, c = 0,
  // a = 4^q.  c_p a_i sits in the first unused column slot when MA is not a multiple of 4 (it then
  // arrives with the column's last 16-byte load), else in slot MM. ----
  constexpr int RS = MM + 4;
  constexpr int CPA = (MA % 4 != 0) ? MA : MM;
  const int NS = a.WN * 32;
  float *trow = reinterpret_cast<float *>(smem + a.blob_bytes);
  for (int i = threadIdx.x; i < NS; i += blockDim.x) {
    float4 sc = make_float4(0.f, 0.f, 0.f, 0.f);       // (-c_o c_i, c_p a_i, |A_i|_1, E0_i)
    float *row = trow + i * RS;
#pragma unroll
    for (int m = 0; m < MM; ++m) row[m] = i < n ? sAcol[i * MM + m] : 0.0f;
    if (i < n) {
      sc = sIc[i];
    } else if (i < N) {
      int q = i - n, m = 0;
      while (m < M - 1 && q >= sQ[m]) { q -= sQ[m]; ++m; }
      const float A = (float)(1u << q);
      row[m] = A;
      const float cpa = (cpf * A) * A;
      sc = make_float4(0.f, cpa, A, (float)((2.0 * (MM + 6) * 0x1p-24 + 1.01 * 0x1p-22) * (double)cpa));
    }
    row[MM] = 0.0f;
    row[CPA] = sc.y;
    row[MM + 1] = sc.x;
    row[MM + 2] = sc.z;
    row[MM + 3] = sc.w;
  }
  __syncthreads();

  const int gi = lane / G, ell = lane % G, gbase = gi * G;
  const int sl = G - 1 - ell;                          // this lane's spins are i = sl (mod G)
  uint32_t gmsh = GM << gbase;                         // this chain's lanes
  // (opaque to the compiler: kept in a register instead of being recomputed in every round)
  asm volatile("" : "+r"(gmsh));
  const int wglob = blockIdx.x * (blockDim.x >> 5) + warp;
  if (wglob * C >= a.R) return;       // whole warp beyond R
  const int ridx = wglob * C + gi;
  const bool live = ridx < a.R;       // chains beyond R compute but never write
  const int rho = a.rep0 + (live ? ridx : a.R - 1);
  const uint32_t cbytes = mkpx_chain_bytes(a.WN, MM);
  unsigned char *wbase = smem + a.blob_bytes + mkpx_table_bytes(a.WN, MM) + (size_t)warp * C * cbytes;
  const uint32_t lam_off = align16u((uint32_t)a.WN * 4u), kt_off = lam_off + MM * 8u;
  uint32_t *xw = reinterpret_cast<uint32_t *>(wbase + gi * cbytes);               // [WN]
  long long *Lam = reinterpret_cast<long long *>(wbase + gi * cbytes + lam_off);  // [MM]
  // per spin of this chain: (T_i, error slope) of this iteration, (logit, logit tolerance) of this sweep
  const float4 *kt = reinterpret_cast<const float4 *>(wbase + gi * cbytes + kt_off);   // [NS]

  const float rbound = (float)Hp->r_bound;
  const float amax = (float)(Hp->v_bound - 2.0 * Hp->r_bound);   // max A_ext entry

  float r[MA];
#pragma unroll
  for (int m = 0; m < MA; ++m) r[m] = m < M ? (float)(-sB[m]) : 0.0f;   // x = 0: r = -b
  for (int m = ell; m < MM; m += G) Lam[m] = 0;
  for (int w = ell; w < a.WN; w += G) xw[w] = 0u;
  __syncwarp();
  long long best_f = LLONG_MAX;
  int best_k = -1, nfeas = 0;
  uint32_t c_flips = 0, c_unif = 0, c_fp64 = 0, c_unc = 0;
  const uint2 key = make_uint2((uint32_t)a.seed, (uint32_t)(a.seed >> 32));
  const uint32_t srho = ((uint32_t)s << 20) | (uint32_t)rho;
  const double bstep = (a.T >= 2) ? a.beta_max / (double)(a.T - 1) : a.beta_max;
  const int Wn = (n + 31) >> 5;
  const int WNi = (N + 31) >> 5, NG = (N + 127) >> 7;  // words / 128-spin Philox groups of this instance
  // shared-window byte addresses: the spin table, this chain's per-spin table and x words
  uint32_t rowbase = (uint32_t)__cvta_generic_to_shared(trow);
  uint32_t ktbase = (uint32_t)__cvta_generic_to_shared(kt);
  uint32_t xwbase = (uint32_t)__cvta_generic_to_shared(xw);
  asm volatile("" : "+r"(rowbase), "+r"(ktbase), "+r"(xwbase));

  for (int k = 0; k < a.K; ++k) {
    // Logits of chain c's sweep tt (R2: the Philox call of counter (32g + j, t, k, s<<20|rho)
    // yields the words of spins 128g + 32w + j, w = 0..3), drawn by the whole warp (lane = j) into
    // the chain's table together with the logit tolerance of the certificate.  The beta = 0 sweep
    // (T >= 2, t = 0) decides x_i = [u < 1/2]: the exact sign bit of the logit, stored as +-1.
    auto fill = [&](int c, int tt, uint32_t sr) {
      float4 *dst = reinterpret_cast<float4 *>(wbase + c * cbytes + kt_off) + lane;
      const bool bz = a.T >= 2 && tt == 0;
      auto put = [&](float4 *q, uint32_t w) {
        float lv = logit_signed_x(w);
        if (bz) lv = (w >> 31) ? 1.0f : -1.0f;
        *reinterpret_cast<float2 *>(&q->z) = make_float2(lv, (kLogitAbs + kLogitRel * fabsf(lv)) * 1.0001f);
      };
      for (int g = 0; g < NG; ++g) {
        const uint4 w4 = philox_group(key, g, lane, tt, k, sr);
        const int nw = WNi - 4 * g;
        put(dst + 128 * g, w4.x);
        if (nw > 1) put(dst + 128 * g + 32, w4.y);
        if (nw > 2) put(dst + 128 * g + 64, w4.z);
        if (nw > 3) put(dst + 128 * g + 96, w4.w);
      }
    };

    // ---- per-iteration tables of every chain of the warp (all 32 lanes): c_l Lambda_m rounded
    // once; T_i = -c_o c_i - A_i . (c_l Lambda); error slope E1 |A_i|_1 + E0_i with
    // |z_f32 - z| <= beta (E1 |A_i|_1 + E0_i) as in the lockstep kernel;
    // then the logits of sweep 0 ----
#pragma unroll 1
    for (int c = 0; c < C; ++c) {
      const long long *Lc = reinterpret_cast<const long long *>(wbase + c * cbytes + lam_off);
      float cLc[MA], cLmax = 0.0f;
#pragma unroll
      for (int m = 0; m < MA; ++m) {
        cLc[m] = (float)(c_l * (double)Lc[m]);
        cLmax = fmaxf(cLmax, fabsf(cLc[m]));
      }
      const double Wk = 2.0 * c_p * ((double)rbound + (double)amax) + (double)cLmax;
      const float E1 = (float)((MM + 8) * 0x1p-24 * Wk * 2.0 + 0x1p-22 * Wk * 1.01);
      float4 *ktc = reinterpret_cast<float4 *>(wbase + c * cbytes + kt_off);
      for (int i = lane; i < NS; i += 32) {
        const float *row = trow + i * RS;
        float q0 = 0.f, q1 = 0.f;
#pragma unroll
        for (int m = 0; m < MA; m += 2) {
          q0 = fmaf(row[m], cLc[m], q0);
          if (m + 1 < MA) q1 = fmaf(row[m + 1], cLc[m + 1], q1);
        }
        *reinterpret_cast<float2 *>(&ktc[i].x) = make_float2(row[MM + 1] - (q0 + q1), fmaf(E1, row[MM + 2], row[MM + 3]));
      }
      fill(c, 0, __shfl_sync(kFullX, srho, c * G));
    }
    __syncwarp();

    // ---- chain state (identical in the chain's lanes) and this lane's current spin ----
    // Sliding window: the chain's G lanes always hold its next G spins that are not final yet;
    // spin i belongs to lane G-1 - i mod G, so a lane whose spin became final moves on to spin i + G.
    int t = 0, w0 = 0;                                 // sweep, first spin that is not final
    bool done = false, wrapf = false;                  // wrapf: sweep finished, the next one not yet entered
    double beta = (a.T >= 2) ? 0.0 : a.beta_max;
    float bf = (float)beta, tb = -bf * twocp;
    int ime = sl - G;                                  // this lane's spin (>= N: none left in this sweep)
    bool open = false;                                 // ... exists and is not final
    float a_[MA];
    // signed by sg = 1 - 2 x_i (x_i the spin's value when the lane took it): zs = sg z, ls = sg logit
    float tbs = 0.f, zbs = 0.f, ls = 0.f, satT = 0.f, certT = 0.f, sg = 1.0f;

    // this lane takes spin ime + G (if the sweep has one)
    auto next_spin = [&]() {
      ime += G;
      open = ime < N && !done;
      const int il = open ? ime : 0;                   // (a lane without a spin loads row 0, unused)
      const uint32_t rowp = rowbase + (uint32_t)(il * (RS * 4));
      float cpa;
#pragma unroll
      for (int m4 = 0; m4 < (MA + 3) / 4; ++m4) {
        const float4 av = lds128(rowp + 16u * m4);
        a_[4 * m4 + 0] = av.x;
        if (4 * m4 + 1 < MA) a_[4 * m4 + 1] = av.y;
        if (4 * m4 + 2 < MA) a_[4 * m4 + 2] = av.z;
        if (4 * m4 + 3 < MA) a_[4 * m4 + 3] = av.w;
        if (CPA / 4 == m4) cpa = (CPA % 4 == 1) ? av.y : ((CPA % 4 == 2) ? av.z : av.w);
      }
      if (CPA == MM) cpa = lds32f(rowp + 4u * MM);
      const float4 kv = lds128(ktbase + (uint32_t)(il * 16));
      const uint32_t xb = (lds32u(xwbase + (uint32_t)((il >> 5) * 4)) >> (il & 31)) & 1u;
      sg = xb ? -1.0f : 1.0f;
      // F = T_i - c_p a_i sg - 2 c_p (A_i . r);  zs = sg beta F = fma(sg tb, A_i . r, bf (sg T_i - c_p a_i))
      zbs = bf * fmaf(sg, kv.x, -cpa);
      tbs = sg * tb;
      ls = sg * kv.z;
      const float e = bf * kv.y;
      satT = e + kSatThr;
      certT = fmaf(e, 1.0001f, kv.w);
      if (!open) {                                     // no spin: certified "saturated, no flip" in every round
        tbs = 0.0f;
        zbs = -3.0e38f;
      }
    };

    // fp64 second level (and, in the replay instantiation, the double-double third level) for
    // this lane's spin in the current state: returns x | uncertified << 1.
    auto slow = [&]() -> int {
      const int i = ime;
      const uint32_t wd = word_of_x(key, i, t, k, srho);
      double drd = 0.0, dld = 0.0, a2 = 0.0;
#pragma unroll
      for (int m = 0; m < MA; ++m) {
        const double Am = (double)a_[m];
        drd += Am * (double)r[m];
        dld += Am * (double)Lam[m];
        a2 += Am * Am;
      }
      const int ci = i < n ? sC[i] : 0;
      const int xi = sg < 0.0f ? 1 : 0;
      const double t1 = c_o * (double)ci, t2 = c_p * a2, t3 = 2.0 * c_p * drd, t4 = c_l * dld;
      const double zz = beta * (-t1 - t2 * (1.0 - 2.0 * xi) - t3 - t4);
      const int rs = certify_fp64_x(zz, beta * (fabs(t1) + fabs(t2) + fabs(t3) + fabs(t4)), wd);
      if constexpr (RP) {                              // double-double level: replay kernel only
        if ((rs & 2) || (a.flags & SAIM_FLAG_TEST_REPLAY)) {
          long long kap = 0;
          for (int m = 0; m < MA; ++m) kap += (long long)a_[m] * Lam[m];
          return decide_dd(-(long long)ci, 2 * (long long)drd + (long long)a2 * (1 - 2 * xi), kap,
                           a.T >= 2 ? t : 1, a.T >= 2 ? a.T - 1 : 1, Hp, wd);
        }
      }
      return rs;
    };

    // spin iev of the chain flips (doit) from x = xold: r += delta A_iev, x bit toggled in the
    // chain's x words (called by all lanes of the chain; all store the same word)
    auto apply_flip = [&](int iev, bool xold, bool doit) {
      const uint32_t cj = rowbase + (uint32_t)(iev * (RS * 4));
      const float dl = doit ? (xold ? -1.0f : 1.0f) : 0.0f;       // delta = 1 - 2 x_j (0: fma(0, a, r) = r)
#pragma unroll
      for (int m4 = 0; m4 < (MA + 3) / 4; ++m4) {
        const float4 av = lds128(cj + 16u * m4);
        r[4 * m4 + 0] = fmaf(dl, av.x, r[4 * m4 + 0]);
        if (4 * m4 + 1 < MA) r[4 * m4 + 1] = fmaf(dl, av.y, r[4 * m4 + 1]);
        if (4 * m4 + 2 < MA) r[4 * m4 + 2] = fmaf(dl, av.z, r[4 * m4 + 2]);
        if (4 * m4 + 3 < MA) r[4 * m4 + 3] = fmaf(dl, av.w, r[4 * m4 + 3]);
      }
      const uint32_t xa = xwbase + (uint32_t)((iev >> 5) * 4);
      sts32u(xa, lds32u(xa) ^ (doit ? (1u << (iev & 31)) : 0u));
      c_flips += doit ? 1u : 0u;
    };

    next_spin();

    // ---- rounds ----
#pragma unroll 1
    for (;;) {
      float p0 = 0.f, p1 = 0.f;
#pragma unroll
      for (int m = 0; m < MA; m += 2) {
        p0 = fmaf(a_[m], r[m], p0);
        if (m + 1 < MA) p1 = fmaf(a_[m + 1], r[m + 1], p1);
      }
      const float zs = fmaf(tbs, p0 + p1, zbs);
      const float ds = zs - ls;
      // Certified decision, signed (sg z, sg (z - logit)): the spin flips <=> sg z > 0 if
      // saturated, sg (z - logit) > 0 otherwise.  cf: a certified flip (saturated towards the
      // flip, or unsaturated with sg (z - logit) beyond the fp32 band); need: unsaturated and
      // inside the band (ties z = 0, d = 0 included): not certified in fp32.  A lane without a
      // spin has zs = -3e38: saturated, no flip.
      const bool sat = fabsf(zs) > satT;
      const bool cf = zs > satT || (ds > certT && !sat);
      const bool need = !sat && !(fabsf(ds) > certT);
      // The chain's first event in spin order.  Spin i belongs to the chain's lane G-1 - i mod G
      // (descending), the window starts at spin w0 and wraps around the lanes: the chain's ballot
      // bits rotated left by w0 mod G have the window's k-th spin at bit G-1-k, so the first event
      // is the highest set bit (one FLO).  Returns the event's spin (0 if none: row 0 is then read
      // and unused) and lane.
      auto first_event = [&](uint32_t evw, bool &hasev, int &iev, int &jl) {
        const uint32_t e = (evw >> gbase) & GM;
        hasev = e != 0u;
        const int s0 = w0 & (G - 1);
        uint32_t rot;
        if constexpr (G == 32) rot = __funnelshift_l(e, e, s0);
        else rot = ((e | (e << G)) >> (G - s0)) & GM;
        const int kk = __clz(rot) - (32 - G);
        iev = hasev ? w0 + kk : 0;
        jl = gbase + G - 1 - ((s0 + kk) & (G - 1));
      };
      const uint32_t cfw = __ballot_sync(kFullX, cf);                        // certified flips
      bool hasev, fin;
      int iev, jl;
      if (!__any_sync(kFullX, need || wrapf)) {
        // ---- common round: every open decision of the warp is certified ----
        first_event(cfw, hasev, iev, jl);
        // final: the open lanes up to the flip (all of them if there is none)
        fin = open && (!hasev || ime <= iev);
        c_unif += (fin && !sat) ? 1u : 0u;             // (this lane's spin drew u)
        const float dlj = __shfl_sync(kFullX, sg, jl);  // delta = 1 - 2 x of the flipping spin
        apply_flip(iev, dlj < 0.0f, hasev);
        w0 = hasev ? iev + 1 : w0 + G;
      } else {
        // ---- rare round: some open decision is not certified in fp32 (it is an event too: if it
        // is its chain's first, it is settled on the slow path), or a chain finished its sweep in
        // the previous round (it idles this round) ----
        first_event(__ballot_sync(kFullX, cf || need), hasev, iev, jl);
        const uint32_t ndw = __ballot_sync(kFullX, need);
        const bool nfirst = hasev && ((ndw >> jl) & 1u) != 0u;
        const bool xold = __shfl_sync(kFullX, sg, jl) < 0.0f;
        fin = open && (!hasev || ime < iev + (nfirst ? 0 : 1));
        c_unif += (fin && !sat) ? 1u : 0u;
        bool sflip = false;
        if (nfirst && ime == iev && open) {
          ++c_fp64;
          const int rs = slow();
          if (rs & 2) ++c_unc;
          sflip = (rs & 1) != (sg < 0.0f ? 1 : 0);
          ++c_unif;                                    // (not saturated: it drew u)
          fin = true;                                  // settled now
        }
        const bool gflip = (__ballot_sync(kFullX, sflip) & gmsh) != 0u;
        apply_flip(iev, xold, hasev && (!nfirst || gflip));
        w0 = hasev ? iev + 1 : w0 + G;
        if (__any_sync(kFullX, wrapf)) {
          if (wrapf) {
            ++t;
            done = t == a.T;
          }
          uint32_t fw = __ballot_sync(kFullX, wrapf && !done);
          while (fw) {
            const int src = __ffs(fw) - 1;
            const int c = src / G;
            fill(c, __shfl_sync(kFullX, t, src), __shfl_sync(kFullX, srho, src));
            fw &= ~(GM << (c * G));
          }
          __syncwarp();
          if (wrapf) {
            wrapf = false;
            beta = bstep * (double)t;                  // (T >= 2 here: T = 1 is done after sweep 0)
            bf = (float)beta;
            tb = -bf * twocp;
            w0 = 0;
            ime = sl - G;                              // (takes spin sl just below)
            fin = true;
          }
          if (__all_sync(kFullX, done)) break;
        }
      }
      if (fin) next_spin();
      if (w0 >= N && !done) wrapf = true;              // sweep finished (every lane has open = false)
    }
    __syncwarp();

    // ---- readout of x_k: f, feasibility, trace, best, Lagrange step ----
    long long fpart = 0;
    for (int w = ell; w < Wn; w += G) {
      uint32_t bits = xw[w];
      if (32 * w + 32 > n) bits &= (1u << (n - 32 * w)) - 1u;
      while (bits) {
        const int bb = __ffs(bits) - 1;
        bits &= bits - 1u;
        fpart += sC[32 * w + bb];
      }
    }
#pragma unroll
    for (int o = 1; o < G; o <<= 1) fpart += __shfl_xor_sync(kFullX, fpart, o);
    const long long f = fpart;
    // feasible <=> A x_items <= b <=> r_m <= (slack value of row m) for every row (R12)
    bool feas = true;
    {
      int i0 = n;
#pragma unroll
      for (int m = 0; m < MA; ++m) {
        const int qm = (m < M) ? sQ[m] : 0;
        long long sv = 0;
        for (int q = 0; q < qm; ++q) {
          const int i = i0 + q;
          sv += (long long)((xw[i >> 5] >> (i & 31)) & 1u) << q;
        }
        if (m < M && (long long)r[m] > sv) feas = false;
        i0 += qm;
      }
    }
    const size_t row = ((size_t)s * a.R + ridx) * a.K + k;
    if (live) {
      if (ell == 0) {
        if (a.out.tr_f) a.out.tr_f[row] = f;
        if (a.out.tr_feas) a.out.tr_feas[row] = (uint8_t)feas;
      }
      if (a.out.tr_x)
        for (int w = ell; w < a.WN; w += G) a.out.tr_x[row * a.WN + w] = xw[w];
    }
    // trace rows of r and Lambda (before the update), then Lambda += g(x_k) (R10)
#pragma unroll
    for (int m = 0; m < MA; ++m) {
      if (m < M && (m % G) == ell) {
        const long long rl = (long long)r[m];
        const long long lm = Lam[m];
        if (live) {
          if (a.out.tr_r) a.out.tr_r[row * M + m] = rl;
          if (a.out.tr_lam) a.out.tr_lam[row * M + m] = lm;
        }
        Lam[m] = lm + rl;
      }
    }
    if (feas) {
      ++nfeas;
      if (f < best_f) {
        best_f = f;
        best_k = k;
        if (live) {
          const size_t ri = (size_t)s * a.R + ridx;
          for (int w = ell; w < Wn; w += G) {
            uint32_t bits = xw[w];
            if (32 * w + 32 > n) bits &= (1u << (n - 32 * w)) - 1u;
            a.out.best_x[ri * a.Wn + w] = bits;
          }
        }
      }
    }
    __syncwarp();
  }

  // ---- outputs ----
  const size_t ri = (size_t)s * a.R + ridx;
  if (live) {
    if (ell == 0) {
      a.out.best_f[ri] = best_f;
      a.out.best_k[ri] = best_k;
      a.out.n_feasible[ri] = nfeas;
      if (a.out.rep_flips) a.out.rep_flips[ri] = c_flips;     // every lane of the chain counts all its flips
    }
    if (best_k < 0)
      for (int w = ell; w < Wn; w += G) a.out.best_x[ri * a.Wn + w] = 0u;
    if (a.out.final_x)
      for (int w = ell; w < a.WN; w += G) a.out.final_x[ri * a.WN + w] = xw[w];
    if (a.out.final_lam)
      for (int m = ell; m < M; m += G) a.out.final_lam[ri * M + m] = Lam[m];
  }
  // Exact replay: the main kernel defers a warp in which some decision was not
  // certified by the fp64 level (SAIM_FLAG_TEST_REPLAY: any fp64-level decision) -- the replay
  // kernel re-runs its CTA with the double-double level and only the flagged warps contribute
  // their instance-best candidates and counters (the others did in the main kernel).
  const size_t rslot = replay_slot(warp);
  const bool defer = !RP && __any_sync(kFullX, live && (c_unc != 0 || ((a.flags & SAIM_FLAG_TEST_REPLAY) && c_fp64 != 0)));
  const bool contribute = RP ? a.replay[rslot] != 0 : !defer;
  if (defer) {
    const uint32_t nrep = __popc(__ballot_sync(kFullX, live && ell == 0));
    if (lane == 0) {
      a.replay[rslot] = 1;
      if (a.out.counters) atomicAdd(reinterpret_cast<unsigned long long *>(a.out.counters) + SAIM_CNT_REPLAYED, (unsigned long long)nrep);
    }
  }
  long long kb = (live && ell == 0 && best_k >= 0) ? ((best_f << 20) | (long long)rho) : LLONG_MAX;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const long long other = __shfl_xor_sync(kFullX, kb, o);
    kb = other < kb ? other : kb;
  }
  if (contribute && lane == 0 && kb != LLONG_MAX && a.out.inst_best)
    atomicMin(reinterpret_cast<long long *>(a.out.inst_best) + s, kb);
  if (a.out.counters && contribute) {
    const unsigned long long nl = live ? 1ull : 0ull;
    const unsigned long long g0 = (live && ell == 0) ? 1ull : 0ull;
    // c_unif: per lane (its own spins); the beta = 0 sweep (T >= 2) has z = 0, never saturated, so
    // it added exactly N per chain and iteration, which do not count (no u is "drawn" there, R19)
    const unsigned long long fl = warp_sum_u64(g0 * c_flips);
    const unsigned long long un = warp_sum_u64(nl * c_unif) - (a.T >= 2 ? warp_sum_u64(g0) * (unsigned long long)a.K * N : 0ull);
    const unsigned long long fp = warp_sum_u64(nl * c_fp64), uc = warp_sum_u64(nl * c_unc);
    const unsigned long long nf = warp_sum_u64(g0 * (unsigned long long)nfeas);
    const unsigned long long lv = warp_sum_u64(g0);
    if (lane == 0) {
      unsigned long long *c = reinterpret_cast<unsigned long long *>(a.out.counters);
      atomicAdd(c + SAIM_CNT_DECISIONS, lv * (unsigned long long)a.K * a.T * N);
      atomicAdd(c + SAIM_CNT_FLIPS, fl);
      atomicAdd(c + SAIM_CNT_SWEEPS, lv * (unsigned long long)a.K * a.T);
      atomicAdd(c + SAIM_CNT_UNIFORMS, un);
      atomicAdd(c + SAIM_CNT_FP64, fp);
      atomicAdd(c + SAIM_CNT_UNCERTIFIED, uc);
      atomicAdd(c + SAIM_CNT_FEASIBLE, nf);
      atomicAdd(c + SAIM_CNT_PHILOX, lv * (unsigned long long)a.K * a.T * NG * 32ull);   // 32 calls per 128-spin group
    }
  }
}

// ---------------------------------------------------------------------------------------------
typedef void (*mkpx_kernel_t)(const RunArgs);

template <int G, bool RPV>
static mkpx_kernel_t mkpx_pick(int MM, int M) {
  if (MM == 8 && M == 5) return saim_mkp_spec_kernel<8, 5, G, RPV>;
  switch (MM) {
    case 4: return saim_mkp_spec_kernel<4, 4, G, RPV>;
    case 8: return saim_mkp_spec_kernel<8, 8, G, RPV>;
    default: return nullptr;
  }
}

// Instantiated for M <= 8 (MM = 4, 8) and G = 2, 4, 8, 16, 32 lanes per chain.
template <bool RPV>
static mkpx_kernel_t mkpx_kernel_for_t(int MM, int M, int G) {
  switch (G) {
    case 2: return mkpx_pick<2, RPV>(MM, M);
    case 4: return mkpx_pick<4, RPV>(MM, M);
    case 8: return mkpx_pick<8, RPV>(MM, M);
    case 16: return mkpx_pick<16, RPV>(MM, M);
    case 32: return mkpx_pick<32, RPV>(MM, M);
    default: return nullptr;
  }
}

}  // namespace saim
