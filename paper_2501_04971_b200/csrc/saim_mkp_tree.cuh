// saim_mkp_tree.cuh -- MKP kernel with outcome-tree blocks (linear objective, 2 <= M <= 32;
// PAPER.md:321-326, BASELINE.json configs 3-4).  sm_100a.
//
// Mapping: L lanes (L = 2 or 4) cooperate on one replica; a warp holds G = 32/L
// replicas of one instance, all at the same spin position.  Spins are processed in blocks of up
// to L consecutive spins (never crossing a slack row or a 32-spin word), lane l owning spin
// i0 + l.  The sequential Gibbs order (R4) makes lane l's decision depend on the flips of lanes
// j < l of the same block, but only through the residuals r: flipping spin j by delta_j moves
// lane l's field by  -2 c_p delta_j (A_l . A_j)  (difference of Eq. 3 / R1; A_l . A_j from an
// O(3n) band of nearby-column products for items, 2^q 2^q' for slack bits of one row).  So lane
// l evaluates its decision for all 2^l combinations of earlier flips -- an "outcome tree" -- and
// one OR-reduction over the L lanes (log2 L shuffles) gives every lane all the tables, from which
// the flips that actually happen follow in L local steps.  The decisions are exactly those of
// the sequential sweep (nothing is ever rolled back), the dependency chain per spin is ~L times
// shorter than in the lane-per-replica kernel, and a replica needs only 1/G of a warp.
//
// Every lane keeps the replica's full residual vector r (exact integers in fp32 registers) and
// c_l Lambda (fp32, rounded once per iteration); decisions are certified as in the other kernels
// (saturation test, fp32 logit band, fp64 re-evaluation of the combination that occurred).
#pragma once
#include <climits>
#include <cstdint>
#include <cstdio>

#include "saim_dev.cuh"

namespace saim {

namespace {

constexpr uint32_t kFull = 0xffffffffu;

// logit(u) in fp32 with its sign made exact (sign(logit u) = sign(u - 1/2) <=> w >= 2^31).
__device__ __forceinline__ float logit_signed_t(uint32_t w) {
  const float l = fabsf(logit_f32(w));
  return (w >> 31) ? l : -l;
}

// Uniform word of spin i (R2) recomputed for the slow path.
__device__ __noinline__ uint32_t word_of_t(uint2 key, int i, int t, int k, uint32_t srho) {
  const uint4 w4 = philox_group(key, i >> 7, i & 31, t, k, srho);
  const int j = (i >> 5) & 3;
  return j == 0 ? w4.x : (j == 1 ? w4.y : (j == 2 ? w4.z : w4.w));
}

// fp64 tail of the slow path: z and its magnitude sum S are accurate to ~2^-50 S; returns
// (x | uncertified << 1).
__device__ __noinline__ int certify_fp64_t(double zz, double S, uint32_t w) {
  const double d = zz - logit_f64_calc(w);
  return (d > 0.0 ? 1 : 0) | (fabs(d) <= (S + 1.0 + fabs(zz)) * 0x1p-46 ? 2 : 0);
}

constexpr int kTreeThreads = 512;

}  // namespace

// MM: padded constraint count (layout); MA <= MM: rows the arithmetic covers; L: lanes/replica.
template <int MM, int MA, int L, bool RP>
__global__ void __launch_bounds__(kTreeThreads, 1) saim_mkp_tree_kernel(const RunArgs a) {
  constexpr int G = 32 / L;           // replicas per warp
  constexpr int NC = 1 << (L - 1);    // combinations of earlier flips (lane L-1 needs them all)
  constexpr int B = 32 / L;           // bits per lane in the packed tables (>= NC)
  static_assert(NC <= B, "packed outcome tables must fit 32 bits");
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ uint64_t mbar;

  const int s = blockIdx.y;
  if constexpr (RP) {                                  // exact replay: only CTAs holding a flagged warp
    if (!__syncthreads_or(a.replay[replay_slot((int)(threadIdx.x >> 5))] != 0)) return;
  }
  bulk_stage(smem, a.blob + (size_t)s * a.blob_bytes, a.blob_bytes, &mbar);

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gi = lane / L;            // replica group within the warp
  const int ell = lane % L;           // position within a block
  const int wglob = blockIdx.x * (blockDim.x >> 5) + warp;
  if (wglob * G >= a.R) return;       // whole warp beyond R
  const int ridx = wglob * G + gi;
  const bool live = ridx < a.R;       // groups beyond R compute but never write
  const int rho = a.rep0 + (live ? ridx : a.R - 1);
  const InstHdr *Hp = a.hdr + s;
  const int n = a.n, M = a.M;
  const int N = Hp->N;
  const MkpLayout Ly = mkp_layout(n, MM);
  const float *sAcol = reinterpret_cast<const float *>(smem + Ly.acol);
  const float4 *sIc = reinterpret_cast<const float4 *>(smem + Ly.iconst);
  const int32_t *sC = reinterpret_cast<const int32_t *>(smem + Ly.cint);
  const long long *sB = reinterpret_cast<const long long *>(smem + Ly.brow);
  const int32_t *sQ = reinterpret_cast<const int32_t *>(smem + Ly.qrow);
  const float *sBand = reinterpret_cast<const float *>(smem + Ly.band);
  const int bstr = (int)mkp_band_stride(n);
  unsigned char *wbase = smem + a.blob_bytes + warp * mkpt_warp_bytes(a.WN, L, MM);
  uint32_t *xw = reinterpret_cast<uint32_t *>(wbase) + gi;                         // word w: xw[G w]
  float *lt = reinterpret_cast<float *>(wbase + align16u(a.WN * G * 4u)) + gi;      // spin 128g+j: lt[G j]
  long long *Lam = reinterpret_cast<long long *>(wbase + align16u(a.WN * G * 4u) + 128u * G * 4u) + gi;  // [G m]

  const double c_o = Hp->c_o, c_p = Hp->c_p, c_l = Hp->c_l;
  const float twocp = (float)(2.0 * c_p), cpf = (float)c_p;
  const float rbound = (float)Hp->r_bound;
  const float amax = (float)(Hp->v_bound - 2.0 * Hp->r_bound);   // max A_ext entry

  float r[MA], cL[MA];
#pragma unroll
  for (int m = 0; m < MA; ++m) {
    r[m] = m < M ? (float)(-sB[m]) : 0.0f;           // x = 0: r = -b
    cL[m] = 0.0f;
  }
  for (int m = ell; m < MM; m += L) Lam[G * m] = 0;
  for (int w = ell; w < a.WN; w += L) xw[G * w] = 0u;
  __syncwarp();
  long long best_f = LLONG_MAX;
  int best_k = -1, nfeas = 0;
  uint32_t c_flips = 0, c_unif = 0, c_fp64 = 0, c_unc = 0, c_philox = 0;
  const uint2 key = make_uint2((uint32_t)a.seed, (uint32_t)(a.seed >> 32));
  const uint32_t srho = ((uint32_t)s << 20) | (uint32_t)rho;
  const double bstep = (a.T >= 2) ? a.beta_max / (double)(a.T - 1) : a.beta_max;
  const int Wn = (n + 31) >> 5;

  for (int k = 0; k < a.K; ++k) {
    float cLmax = 0.0f;
#pragma unroll
    for (int m = 0; m < MA; ++m) {
      cL[m] = (float)(c_l * (double)Lam[G * m]);
      cLmax = fmaxf(cLmax, fabsf(cL[m]));
    }
    // Error slope of the lockstep kernel with the final-rounding term doubled
    // for the up to L-1 extra additions of the outcome-tree corrections.
    const double Wk = 2.0 * c_p * ((double)rbound + (double)amax) + (double)cLmax;
    const float E1 = (float)((MM + 8) * 0x1p-24 * Wk * 2.0 + 0x1p-21 * Wk * 1.01);

    for (int t = 0; t < a.T; ++t) {
      const bool bz = (a.T >= 2) && (t == 0);          // beta_0 = 0: x_i = [u < 1/2]
      const double beta = (a.T >= 2) ? bstep * (double)t : a.beta_max;
      const float bf = (float)beta;
      const float corr_c = -2.0f * bf * cpf;           // dz per unit of delta_j (A_l . A_j)
      int filled = -1, curw = -1;
      uint32_t xcur = 0;                               // x word curw (identical in the L lanes)

      // Logits of the 128 spins of group g (R2: call (32g + j, t, k, s<<20|rho) -> spins
      // 128g + 32w + j), drawn by the L lanes of each replica (calls j = ell, ell + L, ...)
      // off the decision chain.  Blocks never cross a word, so one group is live at a time.
      auto ensure = [&](int g) {
        if (g == filled) return;
        filled = g;
        __syncwarp();
#pragma unroll 2
        for (int j = ell; j < 32; j += L) {
          const uint4 w4 = philox_group(key, g, j, t, k, srho);
          lt[G * (j + 0)] = logit_signed_t(w4.x);
          lt[G * (j + 32)] = logit_signed_t(w4.y);
          lt[G * (j + 64)] = logit_signed_t(w4.z);
          lt[G * (j + 96)] = logit_signed_t(w4.w);
        }
        c_philox += 32 / L;
        __syncwarp();
      };
      auto flush = [&]() {
        if (curw >= 0 && ell == 0) xw[G * curw] = xcur;
        __syncwarp();
      };
      auto word = [&](int w) {
        if (w == curw) return;
        flush();
        curw = w;
        xcur = xw[G * w];
      };

      // Outcome tree of one block: z0 = this lane's z in the block-start state, dcorr[j] = dz if
      // the spin of lane j < ell flips, e = error bound, act = lane owns a spin, xblk = x bits of
      // the block.  slow(c) re-decides combination c in fp64.  Returns the block's flip mask.
      auto decide_block = [&](bool act, uint32_t xblk, int ibit, float z0, const float(&dcorr)[L], float e,
                              auto slow) -> uint32_t {
        const int xb = (xblk >> ell) & 1u;
        const float l = act ? lt[G * (ibit & 127)] : 0.0f;
        const float satT = e + kSatThr;
        const float certT = (e + kLogitAbs + kLogitRel * fabsf(l)) * 1.0001f;
        float zc[NC];
        uint32_t fb = 0, nb = 0, ub = 0;               // per combination: flips, needs fp64, drew u
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          int jl = 0;                                   // lowest set bit of c (folds after unrolling)
#pragma unroll
          for (int j = L - 1; j >= 0; --j)
            if ((c >> j) & 1) jl = j;
          zc[c] = c == 0 ? z0 : zc[c & (c - 1)] + dcorr[jl];
          const float z = zc[c];
          const float d = z - l;
          const bool sat = fabsf(z) > satT;
          int nx = sat ? (z > 0.0f) : (d > 0.0f);
          if (bz) nx = (int)(__float_as_uint(l) >> 31);
          fb |= (uint32_t)(nx != xb) << c;
          nb |= (uint32_t)(!bz && !sat && !(fabsf(d) > certT)) << c;
          ub |= (uint32_t)(!bz && !sat) << c;
        }
        if (!act) fb = nb = 0;
        uint32_t mask;
        for (;;) {
          uint32_t P = fb << (B * ell), Nn = nb << (B * ell);
#pragma unroll
          for (int o = 1; o < L; o <<= 1) {
            P |= __shfl_xor_sync(kFull, P, o);
            Nn |= __shfl_xor_sync(kFull, Nn, o);
          }
          mask = 0;
          int jn = -1;                                  // first lane of the chain needing fp64
#pragma unroll
          for (int j = 0; j < L; ++j) {
            const int c = (int)(mask & ((1u << j) - 1u));
            if (jn < 0 && ((Nn >> (B * j + c)) & 1u)) jn = j;
            mask |= ((P >> (B * j + c)) & 1u) << j;
          }
          if (!__any_sync(kFull, jn >= 0)) break;
          if (jn == ell) {                              // the flips before it are final
            const uint32_t c = mask & ((1u << ell) - 1u);
            ++c_fp64;
            const int rs = slow(c);
            if (rs & 2) ++c_unc;
            fb = (fb & ~(1u << c)) | ((uint32_t)((rs & 1) != xb) << c);
            nb &= ~(1u << c);
          }
        }
        if (act && ((ub >> (mask & ((1u << ell) - 1u))) & 1u)) ++c_unif;
        return mask;
      };

      // ---- items: blocks i0 = 0, L, 2L, ... (L | 32: a block never crosses a word) ----
      for (int i0 = 0; i0 < n; i0 += L) {
        ensure(i0 >> 7);
        word(i0 >> 5);
        const int i = i0 + ell;
        const bool act = i < n;
        const int ic_i = act ? i : n;                   // padded zero column n
        const uint32_t xblk = (xcur >> (i0 & 31)) & ((1u << L) - 1u);
        const int xb = (xblk >> ell) & 1u;
        const float4 *Ac = reinterpret_cast<const float4 *>(sAcol + ic_i * MM);
        float dr0 = 0.f, dr1 = 0.f, dl0 = 0.f, dl1 = 0.f;
#pragma unroll
        for (int m4 = 0; m4 < (MA + 3) / 4; ++m4) {
          const float4 av = Ac[m4];
          dr0 = fmaf(av.x, r[4 * m4 + 0], dr0);
          dl0 = fmaf(av.x, cL[4 * m4 + 0], dl0);
          if (4 * m4 + 1 < MA) { dr1 = fmaf(av.y, r[4 * m4 + 1], dr1); dl1 = fmaf(av.y, cL[4 * m4 + 1], dl1); }
          if (4 * m4 + 2 < MA) { dr0 = fmaf(av.z, r[4 * m4 + 2], dr0); dl0 = fmaf(av.z, cL[4 * m4 + 2], dl0); }
          if (4 * m4 + 3 < MA) { dr1 = fmaf(av.w, r[4 * m4 + 3], dr1); dl1 = fmaf(av.w, cL[4 * m4 + 3], dl1); }
        }
        const float4 ic = sIc[ic_i];                    // (-c_o c_i, c_p a_i, |A_i|_1, E0_i)
        const float sg = xb ? -1.0f : 1.0f;             // 1 - 2 x_i
        const float F = fmaf(-twocp, dr0 + dr1, fmaf(-ic.y, sg, ic.x)) - (dl0 + dl1);
        const float z0 = bf * F;
        float dcorr[L];
        float gsum = 0.0f;
#pragma unroll
        for (int j = 0; j < L; ++j) {
          float g = 0.0f;
          if (j < ell) g = sBand[(ell - j - 1) * bstr + ic_i];   // A_i . A_{i0+j}
          dcorr[j] = corr_c * (((xblk >> j) & 1u) ? -g : g);
          gsum += fabsf(g);
        }
        // |z_f32 - z| <= beta (E1 |A_i|_1 + E0_i + 2^-21 2 c_p sum|g|) for every combination
        const float e = bf * fmaf(E1, ic.z, fmaf(twocp * 0x1p-21f, gsum, ic.w));
        const uint32_t fm = decide_block(act, xblk, i, z0, dcorr, e, [&](uint32_t cstar) -> int {
          const uint32_t wd = word_of_t(key, i, t, k, srho);
          double drd = 0.0, dld = 0.0, a2 = 0.0;
#pragma unroll
          for (int m = 0; m < MA; ++m) {
            const double Am = (double)sAcol[i * MM + m];
            double rm = (double)r[m];
#pragma unroll
            for (int j = 0; j < L - 1; ++j)
              if (j < ell && ((cstar >> j) & 1u))
                rm += (((xblk >> j) & 1u) ? -1.0 : 1.0) * (double)sAcol[(i0 + j) * MM + m];
            drd += Am * rm;
            dld += Am * (double)Lam[G * m];
            a2 += Am * Am;
          }
          const double t1 = c_o * (double)sC[i], t2 = c_p * a2, t3 = 2.0 * c_p * drd, t4 = c_l * dld;
          const double zz = beta * (-t1 - t2 * (1.0 - 2.0 * xb) - t3 - t4);
          const int rs = certify_fp64_t(zz, beta * (fabs(t1) + fabs(t2) + fabs(t3) + fabs(t4)), wd);
          if constexpr (RP) {                          // double-double level: replay kernel only
            if ((rs & 2) || (a.flags & SAIM_FLAG_TEST_REPLAY)) {
              // double-double level on the exact integers (drd, a2 exact in fp64; kappa in int64)
              long long kap = 0;
              for (int m = 0; m < MA; ++m) kap += (long long)sAcol[i * MM + m] * Lam[G * m];
              return decide_dd(-(long long)sC[i], 2 * (long long)drd + (long long)a2 * (1 - 2 * xb), kap, a.T >= 2 ? t : 1, a.T >= 2 ? a.T - 1 : 1, Hp, wd);
            }
          }
          return rs;
        });
        // r += sum_j delta_j A_{i0+j} over the flipped spins (every lane keeps the full r)
#pragma unroll
        for (int j = 0; j < L; ++j) {
          const float dj = ((fm >> j) & 1u) ? (((xblk >> j) & 1u) ? -1.0f : 1.0f) : 0.0f;
          const float4 *Aj = reinterpret_cast<const float4 *>(sAcol + min(i0 + j, n) * MM);
#pragma unroll
          for (int m4 = 0; m4 < (MA + 3) / 4; ++m4) {
            const float4 av = Aj[m4];
            r[4 * m4 + 0] = fmaf(dj, av.x, r[4 * m4 + 0]);
            if (4 * m4 + 1 < MA) r[4 * m4 + 1] = fmaf(dj, av.y, r[4 * m4 + 1]);
            if (4 * m4 + 2 < MA) r[4 * m4 + 2] = fmaf(dj, av.z, r[4 * m4 + 2]);
            if (4 * m4 + 3 < MA) r[4 * m4 + 3] = fmaf(dj, av.w, r[4 * m4 + 3]);
          }
        }
        if (ell == 0) c_flips += __popc(fm);
        xcur ^= fm << (i0 & 31);
      }

      // ---- slack bits: row m, bits q0..; blocks end at the row end or a word boundary ----
      int ibase = n;
#pragma unroll 1
      for (int m = 0; m < M; ++m) {
        const int qm = sQ[m];
        const int iend = ibase + qm;
        float rm = 0.0f, cLm = 0.0f;
#pragma unroll
        for (int mm = 0; mm < MA; ++mm)
          if (mm == m) { rm = r[mm]; cLm = cL[mm]; }
        for (int i0 = ibase; i0 < iend;) {
          const int bend = min(min(i0 + L, iend), (i0 | 31) + 1);
          ensure(i0 >> 7);
          word(i0 >> 5);
          const int i = i0 + ell;
          const bool act = i < bend;
          const int q0 = i0 - ibase;
          const uint32_t xblk = (xcur >> (i0 & 31)) & ((1u << L) - 1u);
          const int xb = (xblk >> ell) & 1u;
          const float A = act ? (float)(1u << (q0 + ell)) : 0.0f;
          const float sg = xb ? -1.0f : 1.0f;
          const float inner = fmaf(twocp, rm, cLm);                  // 2 c_p r_m + c_l Lambda_m
          const float z0 = bf * (-(A * inner) - (cpf * A) * A * sg);
          float dcorr[L];
          float gsum = 0.0f;
#pragma unroll
          for (int j = 0; j < L; ++j) {
            const float g = j < ell ? A * (float)(1u << (q0 + j)) : 0.0f;   // A_q . A_{q0+j}, same row
            dcorr[j] = corr_c * (((xblk >> j) & 1u) ? -g : g);
            gsum += g;
          }
          // |z_f32 - z| <= beta (8 2^-24 + 2.02 2^-22) (A (|2 c_p r_m| + |c_l Lambda_m|) + c_p A^2 + 2 c_p sum g)
          const float e = bf * (8.0f * 0x1p-24f + 2.02f * 0x1p-22f) *
                          (fmaf(A, fabsf(twocp * rm) + fabsf(cLm), cpf * A * A) + twocp * gsum);
          const uint32_t fm = decide_block(act, xblk, i, z0, dcorr, e, [&](uint32_t cstar) -> int {
            const uint32_t wd = word_of_t(key, i, t, k, srho);
            double rr = (double)rm;
            for (int j = 0; j < ell; ++j)
              if ((cstar >> j) & 1u) rr += (((xblk >> j) & 1u) ? -1.0 : 1.0) * (double)(1u << (q0 + j));
            const double Ad = (double)A;
            const double t1 = Ad * 2.0 * c_p * rr, t2 = Ad * c_l * (double)Lam[G * m], t3 = c_p * Ad * Ad;
            const double zz = beta * (-t1 - t2 - t3 * (1.0 - 2.0 * xb));
            const int rs = certify_fp64_t(zz, beta * (fabs(t1) + fabs(t2) + fabs(t3)), wd);
            if constexpr (RP) {                          // double-double level: replay kernel only
              if ((rs & 2) || (a.flags & SAIM_FLAG_TEST_REPLAY)) {
                const long long Ai = (long long)A;
                return decide_dd(0, 2 * Ai * (long long)rr + Ai * Ai * (1 - 2 * xb), Ai * Lam[G * m], a.T >= 2 ? t : 1, a.T >= 2 ? a.T - 1 : 1, Hp, wd);
              }
            }
            return rs;
          });
          float dsum = 0.0f;
#pragma unroll
          for (int j = 0; j < L; ++j)
            if ((fm >> j) & 1u) dsum += (((xblk >> j) & 1u) ? -1.0f : 1.0f) * (float)(1u << (q0 + j));
          rm += dsum;                                    // exact: integers < 2^21
          if (ell == 0) c_flips += __popc(fm);
          xcur ^= fm << (i0 & 31);
          i0 = bend;
        }
#pragma unroll
        for (int mm = 0; mm < MA; ++mm)
          if (mm == m) r[mm] = rm;
        ibase = iend;
      }
      flush();
    }

    // ---- readout of x_k: f, feasibility, trace, best, Lagrange step ----
    long long fpart = 0;
    for (int w = ell; w < Wn; w += L) {
      uint32_t bits = xw[G * w];
      if (32 * w + 32 > n) bits &= (1u << (n - 32 * w)) - 1u;
      while (bits) {
        const int b = __ffs(bits) - 1;
        bits &= bits - 1u;
        fpart += sC[32 * w + b];
      }
    }
#pragma unroll
    for (int o = 1; o < L; o <<= 1) fpart += __shfl_xor_sync(kFull, fpart, o);
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
          sv += (long long)((xw[G * (i >> 5)] >> (i & 31)) & 1u) << q;
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
        for (int w = ell; w < a.WN; w += L) a.out.tr_x[row * a.WN + w] = xw[G * w];
    }
    // trace rows of r and Lambda (before the update), then Lambda += g(x_k) (R10)
#pragma unroll
    for (int m = 0; m < MA; ++m) {
      if (m < M && (m % L) == ell) {
        const long long rl = (long long)r[m];
        const long long lm = Lam[G * m];
        if (live) {
          if (a.out.tr_r) a.out.tr_r[row * M + m] = rl;
          if (a.out.tr_lam) a.out.tr_lam[row * M + m] = lm;
        }
        Lam[G * m] = lm + rl;
      }
    }
    if (feas) {
      ++nfeas;
      if (f < best_f) {
        best_f = f;
        best_k = k;
        if (live) {
          const size_t ri = (size_t)s * a.R + ridx;
          for (int w = ell; w < Wn; w += L) {
            uint32_t bits = xw[G * w];
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
      if (a.out.rep_flips) a.out.rep_flips[ri] = c_flips;     // lane 0 counts the whole replica's flips
    }
    if (best_k < 0)
      for (int w = ell; w < Wn; w += L) a.out.best_x[ri * a.Wn + w] = 0u;
    if (a.out.final_x)
      for (int w = ell; w < a.WN; w += L) a.out.final_x[ri * a.WN + w] = xw[G * w];
    if (a.out.final_lam)
      for (int m = ell; m < M; m += L) a.out.final_lam[ri * M + m] = Lam[G * m];
  }
  // Exact replay: the main kernel defers a warp in which some decision was not
  // certified by the fp64 level (SAIM_FLAG_TEST_REPLAY: any fp64-level decision) -- the replay
  // kernel re-runs its CTA with the double-double level and only the flagged warps contribute
  // their instance-best candidates and counters (the others did in the main kernel).
  const size_t rslot = replay_slot((int)(threadIdx.x >> 5));
  const bool defer = !RP && __any_sync(kFull, live && (c_unc != 0 || ((a.flags & SAIM_FLAG_TEST_REPLAY) && c_fp64 != 0)));
  const bool contribute = RP ? a.replay[rslot] != 0 : !defer;
  if (defer) {
    const uint32_t nrep = __popc(__ballot_sync(kFull, live && ell == 0));
    if (lane == 0) {
      a.replay[rslot] = 1;
      if (a.out.counters) atomicAdd(reinterpret_cast<unsigned long long *>(a.out.counters) + SAIM_CNT_REPLAYED, (unsigned long long)nrep);
    }
  }
  long long kb = (live && ell == 0 && best_k >= 0) ? ((best_f << 20) | (long long)rho) : LLONG_MAX;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const long long other = __shfl_xor_sync(kFull, kb, o);
    kb = other < kb ? other : kb;
  }
  if (contribute && lane == 0 && kb != LLONG_MAX && a.out.inst_best)
    atomicMin(reinterpret_cast<long long *>(a.out.inst_best) + s, kb);
  if (a.out.counters && contribute) {
    const unsigned long long nl = live ? 1ull : 0ull;
    const unsigned long long g0 = (live && ell == 0) ? 1ull : 0ull;
    const unsigned long long fl = warp_sum_u64(nl * c_flips), un = warp_sum_u64(nl * c_unif);
    const unsigned long long fp = warp_sum_u64(nl * c_fp64), uc = warp_sum_u64(nl * c_unc);
    const unsigned long long ph = warp_sum_u64(nl * c_philox), nf = warp_sum_u64(g0 * (unsigned long long)nfeas);
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
      atomicAdd(c + SAIM_CNT_PHILOX, ph);
    }
  }
}

// ---------------------------------------------------------------------------------------------
typedef void (*mkpt_kernel_t)(const RunArgs);

template <int L, bool RPV>
static mkpt_kernel_t mkpt_pick(int MM, int M) {
  if (MM == 8 && M == 5) return saim_mkp_tree_kernel<8, 5, L, RPV>;
  if (MM == 16 && M == 10) return saim_mkp_tree_kernel<16, 10, L, RPV>;
  if (MM == 32 && M == 30) return saim_mkp_tree_kernel<32, 30, L, RPV>;
  switch (MM) {
    case 4: return saim_mkp_tree_kernel<4, 4, L, RPV>;
    case 8: return saim_mkp_tree_kernel<8, 8, L, RPV>;
    case 16: return saim_mkp_tree_kernel<16, 16, L, RPV>;
    case 32: return saim_mkp_tree_kernel<32, 32, L, RPV>;
    default: return nullptr;
  }
}

template <bool RPV>
static mkpt_kernel_t mkpt_kernel_for_t(int MM, int M, int L) {
  return L == 4 ? mkpt_pick<4, RPV>(MM, M) : (L == 2 ? mkpt_pick<2, RPV>(MM, M) : nullptr);
}

}  // namespace saim
