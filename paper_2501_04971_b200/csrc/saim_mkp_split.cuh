// saim_mkp_split.cuh -- MKP kernel with the constraint rows of each replica split over S lanes
// (linear objective, 9 <= M <= 32, BASELINE.json config 4).  sm_100a.
//
// Mapping: the lockstep kernel of saim_mkp.cu (a warp marches its replicas through
// the spins in exact sequential order) with each replica held by S = 2 adjacent lanes, lane s
// owning the constraint rows s*MR .. s*MR+MR-1 (MR = MM/S): its residuals r_m, c_l Lambda_m and
// Lambda_m.  An item decision needs the full dot products A_i . r and A_i . c_l Lambda: each lane
// forms the partial sum over its rows and one shuffle adds the other lane's (a + b == b + a, so
// both lanes hold the same bits and take the same certified decision); the flip updates each
// lane's own rows.  A slack bit of row m concerns r_m only: its owner lane decides it, and the
// lanes merge their flip masks once per 32-spin word.  Halving the per-lane arithmetic and
// doubling the warps gives the SM twice as many independent dependency chains (config 4 has
// only 512 lane-per-replica warps, about one per SMSP) -- measured on B200 this does not pay:
// the duplicated per-decision logic costs 1.67x the instructions of the lockstep kernel and
// config 4 runs 1.2x slower, so this kernel is opt-in (SAIM_FLAG_MKP_SPLIT2).
#pragma once
#include <climits>
#include <cstdint>
#include <cstdio>
#include <type_traits>

#include "saim_dev.cuh"

namespace saim {

namespace {

constexpr uint32_t kFull = 0xffffffffu;
constexpr int kSplitThreads = 512;

__device__ __forceinline__ int certify_fp64_s(double zz, double S, uint32_t w) {
  const double d = zz - logit_f64_calc(w);
  return (d > 0.0 ? 1 : 0) | (fabs(d) <= (S + 1.0 + fabs(zz)) * 0x1p-46 ? 2 : 0);
}

__device__ __forceinline__ uint32_t word_of_s(uint2 key, int i, int t, int k, uint32_t srho) {
  const uint4 w4 = philox_group(key, i >> 7, i & 31, t, k, srho);
  const int j = (i >> 5) & 3;
  return j == 0 ? w4.x : (j == 1 ? w4.y : (j == 2 ? w4.z : w4.w));
}

__device__ __forceinline__ float logit_signed_s(uint32_t w) {
  const float l = fabsf(logit_f32(w));
  return (w >> 31) ? l : -l;
}

}  // namespace

// MM: padded constraint count (layout); MA: rows with data (<= MM); S: lanes per replica.
template <int MM, int MA, int S, bool RP>
__global__ void __launch_bounds__(kSplitThreads, 1) saim_mkp_split_kernel(const RunArgs a) {
  constexpr int G = 32 / S;                 // replicas per warp
  constexpr int MR = MM / S;                // rows per lane
  static_assert(S == 2, "row split implemented for S = 2");
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ uint64_t mbar;

  const int s = blockIdx.y;
  if constexpr (RP) {                                  // exact replay: only CTAs holding a flagged warp
    if (!__syncthreads_or(a.replay[replay_slot((int)(threadIdx.x >> 5))] != 0)) return;
  }
  bulk_stage(smem, a.blob + (size_t)s * a.blob_bytes, a.blob_bytes, &mbar);

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gi = lane / S, sl = lane % S;   // replica group, row slice
  const int wglob = blockIdx.x * (blockDim.x >> 5) + warp;
  if (wglob * G >= a.R) return;             // whole warp beyond R
  const int ridx = wglob * G + gi;
  const bool live = ridx < a.R;             // groups beyond R compute but never write
  const bool lead = sl == 0;                // writes the replica's outputs
  const int rho = a.rep0 + (live ? ridx : a.R - 1);
  const InstHdr *Hp = a.hdr + s;
  const int n = a.n, M = a.M;
  const int N = Hp->N;
  const MkpLayout Ly = mkp_layout(n, MM);
  const float *sAcol = reinterpret_cast<const float *>(smem + Ly.acol);
  const float *sArow = sAcol + sl * MR;     // this lane's rows of column i: sArow[i * MM + k]
  const float4 *sIc = reinterpret_cast<const float4 *>(smem + Ly.iconst);
  const int32_t *sC = reinterpret_cast<const int32_t *>(smem + Ly.cint);
  const long long *sB = reinterpret_cast<const long long *>(smem + Ly.brow);
  const int32_t *sQ = reinterpret_cast<const int32_t *>(smem + Ly.qrow);
  const float *sBand = reinterpret_cast<const float *>(smem + Ly.band);
  unsigned char *wbase = smem + a.blob_bytes + warp * mkps_warp_bytes(a.WN, S, MM);
  uint32_t *xw = reinterpret_cast<uint32_t *>(wbase) + gi;                         // word w: xw[G w]
  float *lt = reinterpret_cast<float *>(wbase + align16u(a.WN * G * 4u)) + gi;      // spin 128g+j: lt[G j]
  long long *Lam = reinterpret_cast<long long *>(wbase + align16u(a.WN * G * 4u) + 128u * G * 4u) + lane;  // [32 k]

  const double c_o = Hp->c_o, c_p = Hp->c_p, c_l = Hp->c_l;
  const float twocp = (float)(2.0 * c_p), cpf = (float)c_p;
  const float rbound = (float)Hp->r_bound;
  const float amax = (float)(Hp->v_bound - 2.0 * Hp->r_bound);   // max A_ext entry

  float r[MR], cL[MR];
#pragma unroll
  for (int k = 0; k < MR; ++k) {
    const int m = sl * MR + k;
    r[k] = m < M ? (float)(-sB[m]) : 0.0f;             // x = 0: r = -b
    cL[k] = 0.0f;
    Lam[32 * k] = 0;
  }
  for (int w = sl; w < a.WN; w += S) xw[G * w] = 0u;
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
    for (int kk = 0; kk < MR; ++kk) {
      cL[kk] = (float)(c_l * (double)Lam[32 * kk]);
      cLmax = fmaxf(cLmax, fabsf(cL[kk]));
    }
    cLmax = fmaxf(cLmax, __shfl_xor_sync(kFull, cLmax, 1));
    // error slope of the lockstep kernel; the partial sums change only the order
    const double Wk = 2.0 * c_p * ((double)rbound + (double)amax) + (double)cLmax;
    const float E1 = (float)((MM + 8) * 0x1p-24 * Wk * 2.0 + 0x1p-22 * Wk * 1.01);

    for (int t = 0; t < a.T; ++t) {
      const bool bz = (a.T >= 2) && (t == 0);          // beta_0 = 0: x_i = [u < 1/2]
      const double beta = (a.T >= 2) ? bstep * (double)t : a.beta_max;
      const float bf = (float)beta;
      uint32_t xcur = 0;

      // Logits of spins 128g .. 128g+127 (R2), one burst per group; the S lanes of a replica
      // share the 32 Philox calls.
      auto fill_group = [&](int g) {
        __syncwarp();
#pragma unroll 2
        for (int j = sl; j < 32; j += S) {
          const uint4 w4 = philox_group(key, g, j, t, k, srho);
          lt[G * (j + 0)] = logit_signed_s(w4.x);
          lt[G * (j + 32)] = logit_signed_s(w4.y);
          lt[G * (j + 64)] = logit_signed_s(w4.z);
          lt[G * (j + 96)] = logit_signed_s(w4.w);
        }
        c_philox += 32 / S;
        __syncwarp();
      };
      // Certified decision (as in saim_mkp.cu); `mine` marks the lanes whose decision counts
      // (the lead lane for items, the owner lane for slack bits); slow() runs where needed.
      auto decide = [&](float z, float e, float l, bool mine, auto slow) -> int {
        const float satT = e + kSatThr;
        const float certT = (e + kLogitAbs + kLogitRel * fabsf(l)) * 1.0001f;
        const float d = z - l;
        const bool sat = fabsf(z) > satT;
        int nx = sat ? (z > 0.0f) : (d > 0.0f);
        if (bz) nx = (int)(__float_as_uint(l) >> 31);
        if (mine && !bz && !sat) ++c_unif;
        const bool need = !bz && !sat && !(fabsf(d) > certT);
        if (__any_sync(kFull, need)) {
          const int rs = slow();                          // all lanes: the item path shuffles
          if (need) {
            if (mine) {
              ++c_fp64;
              if (rs & 2) ++c_unc;
            }
            nx = rs & 1;
          }
        }
        return nx;
      };

      // ---- items i = 0..n-1, one-spin lookahead (saim_mkp.cu) on split dot products ----
      auto dots = [&](int i, float &pr, float &dlv) {
        const float4 *Ac = reinterpret_cast<const float4 *>(sArow + i * MM);
        float dr0 = 0.f, dr1 = 0.f, dl0 = 0.f, dl1 = 0.f;
#pragma unroll
        for (int m4 = 0; m4 < MR / 4; ++m4) {
          const float4 av = Ac[m4];
          dr0 = fmaf(av.x, r[4 * m4 + 0], dr0);
          dl0 = fmaf(av.x, cL[4 * m4 + 0], dl0);
          dr1 = fmaf(av.y, r[4 * m4 + 1], dr1);
          dl1 = fmaf(av.y, cL[4 * m4 + 1], dl1);
          dr0 = fmaf(av.z, r[4 * m4 + 2], dr0);
          dl0 = fmaf(av.z, cL[4 * m4 + 2], dl0);
          dr1 = fmaf(av.w, r[4 * m4 + 3], dr1);
          dl1 = fmaf(av.w, cL[4 * m4 + 3], dl1);
        }
        const float p = dr0 + dr1, q = dl0 + dl1;
        pr = p + __shfl_xor_sync(kFull, p, 1);            // identical bits in both lanes
        dlv = q + __shfl_xor_sync(kFull, q, 1);
      };
      float pre = 0.f, dlc = 0.f, dprev = 0.f, Gc = 0.f;
      dots(0, pre, dlc);
      for (int w = 0; 32 * w < n; ++w) {
        xcur = xw[G * w];
        if ((w & 3) == 0) fill_group(w >> 2);
        const int iend = min(32, n - 32 * w);
        float l = lt[G * ((32 * w) & 127)];
        float4 ic = sIc[32 * w];
        float G_n = sBand[32 * w + 1];
        for (int ii = 0; ii < iend; ++ii) {
          const int i = 32 * w + ii;
          const float l_n = lt[G * ((i + 1) & 127)];
          const float4 ic_n = sIc[i + 1];
          const float G_nn = sBand[i + 2 <= n ? i + 2 : n];
          const int xb = (xcur >> ii) & 1u;
          const float dr = fmaf(dprev, Gc, pre);
          float pre_n, dl_n;
          dots(i + 1, pre_n, dl_n);
          const float sg = xb ? -1.0f : 1.0f;
          const float F = fmaf(-twocp, dr, fmaf(-ic.y, sg, ic.x)) - dlc;
          const float z = bf * F;
          const float e = bf * fmaf(E1, ic.z, ic.w);
          const int nx = decide(z, e, l, lead, [&]() -> int {
            const uint32_t wd = word_of_s(key, i, t, k, srho);
            double drd = 0.0, dld = 0.0, a2 = 0.0;
#pragma unroll
            for (int kk = 0; kk < MR; ++kk) {
              const double Am = (double)sArow[i * MM + kk];
              drd += Am * (double)r[kk];
              dld += Am * (double)Lam[32 * kk];
              a2 += Am * Am;
            }
            long long kap = 0;                              // exact kappa for the double-double level
#pragma unroll
            for (int kk = 0; kk < MR; ++kk) kap += (long long)sArow[i * MM + kk] * Lam[32 * kk];
            drd += __shfl_xor_sync(kFull, drd, 1);
            dld += __shfl_xor_sync(kFull, dld, 1);
            a2 += __shfl_xor_sync(kFull, a2, 1);
            kap += __shfl_xor_sync(kFull, kap, 1);
            const double t1 = c_o * (double)sC[i], t2 = c_p * a2, t3 = 2.0 * c_p * drd, t4 = c_l * dld;
            const double zz = beta * (-t1 - t2 * (1.0 - 2.0 * xb) - t3 - t4);
            const int rs = certify_fp64_s(zz, beta * (fabs(t1) + fabs(t2) + fabs(t3) + fabs(t4)), wd);
            if constexpr (RP) {                          // double-double level: replay kernel only
              if ((rs & 2) || (a.flags & SAIM_FLAG_TEST_REPLAY)) {
                return decide_dd(-(long long)sC[i], 2 * (long long)drd + (long long)a2 * (1 - 2 * xb), kap, a.T >= 2 ? t : 1, a.T >= 2 ? a.T - 1 : 1, Hp, wd);
              }
            }
            return rs;
          });
          const float dl = (float)(nx - xb);
          const float4 *Ac = reinterpret_cast<const float4 *>(sArow + i * MM);
#pragma unroll
          for (int m4 = 0; m4 < MR / 4; ++m4) {
            const float4 av = Ac[m4];
            r[4 * m4 + 0] = fmaf(dl, av.x, r[4 * m4 + 0]);
            r[4 * m4 + 1] = fmaf(dl, av.y, r[4 * m4 + 1]);
            r[4 * m4 + 2] = fmaf(dl, av.z, r[4 * m4 + 2]);
            r[4 * m4 + 3] = fmaf(dl, av.w, r[4 * m4 + 3]);
          }
          xcur ^= (uint32_t)(nx != xb) << ii;
          c_flips += (lead && nx != xb) ? 1u : 0u;
          pre = pre_n; dlc = dl_n; Gc = G_n; dprev = dl;
          l = l_n; ic = ic_n; G_n = G_nn;
        }
        __syncwarp();
        if (lead) xw[G * w] = xcur;
      }
      __syncwarp();
      // ---- slack bits: row m (owner lane m / MR, local row m % MR), bit q (R4) ----
      // Slack bits of different rows do not interact (a bit's field depends on its own row's
      // r_m only), so the owner decides its rows' bits alone; the lanes' flip masks are merged
      // once per 32-spin word.
      int i = n;
      xcur = xw[G * (n >> 5)];
      uint32_t fl = 0;                                      // this lane's flips in the current word
#pragma unroll
      for (int m = 0; m < MA; ++m) {
        constexpr int kMR = MR;
        const int own = m / kMR, kk = m % kMR;
        const bool mine = sl == own;
        const int qm = (m < M) ? sQ[m] : 0;
        for (int q = 0; q < qm; ++q, ++i) {
          if ((i & 31) == 0) xcur = xw[G * (i >> 5)];
          if ((i & 127) == 0) fill_group(i >> 7);
          const float l = lt[G * (i & 127)];
          const int xb = (xcur >> (i & 31)) & 1u;
          const float A = (float)(1u << q);
          const float sg = xb ? -1.0f : 1.0f;
          const float inner = fmaf(twocp, r[kk], cL[kk]);
          const float F = -(A * inner) - (cpf * A) * A * sg;
          const float z = bf * F;
          const float e = bf * (8.0f * 0x1p-24f + 1.01f * 0x1p-22f) *
                          fmaf(A, fabsf(twocp * r[kk]) + fabsf(cL[kk]), cpf * A * A);
          const int nx = decide(z, e, l, mine, [&]() -> int {
            if (!mine) return 0;                            // only the owner's decision is used
            const uint32_t wd = word_of_s(key, i, t, k, srho);
            const double Ad = (double)A;
            const double t1 = Ad * 2.0 * c_p * (double)r[kk], t2 = Ad * c_l * (double)Lam[32 * kk];
            const double t3 = c_p * Ad * Ad;
            const double zz = beta * (-t1 - t2 - t3 * (1.0 - 2.0 * xb));
            const int rs = certify_fp64_s(zz, beta * (fabs(t1) + fabs(t2) + fabs(t3)), wd);
            if constexpr (RP) {                          // double-double level: replay kernel only
              if ((rs & 2) || (a.flags & SAIM_FLAG_TEST_REPLAY)) {
                const long long Ai = (long long)A;
                return decide_dd(0, 2 * Ai * (long long)r[kk] + Ai * Ai * (1 - 2 * xb), Ai * Lam[32 * kk], a.T >= 2 ? t : 1, a.T >= 2 ? a.T - 1 : 1, Hp, wd);
              }
            }
            return rs;
          });
          if (mine) {
            r[kk] = fmaf((float)(nx - xb), A, r[kk]);
            fl |= (uint32_t)(nx != xb) << (i & 31);
            c_flips += (nx != xb) ? 1u : 0u;
          }
          if ((i & 31) == 31 || i == N - 1) {
            xcur ^= fl | __shfl_xor_sync(kFull, fl, 1);
            fl = 0;
            __syncwarp();
            if (lead) xw[G * (i >> 5)] = xcur;
          }
        }
      }
      __syncwarp();
    }

    // ---- readout of x_k: f, feasibility, trace, best, Lagrange step ----
    long long f = 0;
    for (int w = 0; w < Wn; ++w) {
      uint32_t bits = xw[G * w];
      if (32 * w + 32 > n) bits &= (1u << (n - 32 * w)) - 1u;
      while (bits) {
        const int b = __ffs(bits) - 1;
        bits &= bits - 1u;
        f += sC[32 * w + b];
      }
    }
    // feasible <=> r_m <= (slack value of row m) for every row (R12); each lane checks its rows
    bool feas = true;
    {
      int i0 = n;
#pragma unroll
      for (int m = 0; m < MA; ++m) {
        const int qm = (m < M) ? sQ[m] : 0;
        if (qm > 0 && sl == m / MR) {
          long long sv = 0;
          for (int q = 0; q < qm; ++q) {
            const int i = i0 + q;
            sv += (long long)((xw[G * (i >> 5)] >> (i & 31)) & 1u) << q;
          }
          if ((long long)r[m % MR] > sv) feas = false;
        }
        i0 += qm;
      }
      const int feas_other = __shfl_xor_sync(kFull, (int)feas, 1);   // (not inside &&: every lane shuffles)
      feas = feas && feas_other;
    }
    const size_t row = ((size_t)s * a.R + ridx) * a.K + k;
    if (live) {
      if (lead) {
        if (a.out.tr_f) a.out.tr_f[row] = f;
        if (a.out.tr_feas) a.out.tr_feas[row] = (uint8_t)feas;
        if (a.out.tr_x)
          for (int w = 0; w < a.WN; ++w) a.out.tr_x[row * a.WN + w] = xw[G * w];
      }
    }
#pragma unroll
    for (int kk = 0; kk < MR; ++kk) {
      const int m = sl * MR + kk;
      if (m < M) {
        const long long rl = (long long)r[kk];
        if (live && a.out.tr_r) a.out.tr_r[row * M + m] = rl;
        if (live && a.out.tr_lam) a.out.tr_lam[row * M + m] = Lam[32 * kk];
        Lam[32 * kk] += rl;                               // lambda_{k+1} = lambda_k + eta g(x_k) (R10)
      }
    }
    if (feas) {
      ++nfeas;
      if (f < best_f) {
        best_f = f;
        best_k = k;
        if (live && lead) {
          const size_t ri = (size_t)s * a.R + ridx;
          for (int w = 0; w < Wn; ++w) {
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
  const uint32_t rflips = c_flips + __shfl_xor_sync(kFull, c_flips, 1);   // items (lead) + own slack rows
  if (live) {
    if (lead) {
      if (a.out.rep_flips) a.out.rep_flips[ri] = rflips;
      a.out.best_f[ri] = best_f;
      a.out.best_k[ri] = best_k;
      a.out.n_feasible[ri] = nfeas;
      if (best_k < 0)
        for (int w = 0; w < Wn; ++w) a.out.best_x[ri * a.Wn + w] = 0u;
      if (a.out.final_x)
        for (int w = 0; w < a.WN; ++w) a.out.final_x[ri * a.WN + w] = xw[G * w];
    }
    if (a.out.final_lam)
#pragma unroll
      for (int kk = 0; kk < MR; ++kk)
        if (sl * MR + kk < M) a.out.final_lam[ri * M + sl * MR + kk] = Lam[32 * kk];
  }
  // Exact replay: the main kernel defers a warp in which some decision was not
  // certified by the fp64 level (SAIM_FLAG_TEST_REPLAY: any fp64-level decision) -- the replay
  // kernel re-runs its CTA with the double-double level and only the flagged warps contribute
  // their instance-best candidates and counters (the others did in the main kernel).
  const size_t rslot = replay_slot((int)(threadIdx.x >> 5));
  const bool defer = !RP && __any_sync(kFull, live && (c_unc != 0 || ((a.flags & SAIM_FLAG_TEST_REPLAY) && c_fp64 != 0)));
  const bool contribute = RP ? a.replay[rslot] != 0 : !defer;
  if (defer) {
    const uint32_t nrep = __popc(__ballot_sync(kFull, live && lead));
    if (lane == 0) {
      a.replay[rslot] = 1;
      if (a.out.counters) atomicAdd(reinterpret_cast<unsigned long long *>(a.out.counters) + SAIM_CNT_REPLAYED, (unsigned long long)nrep);
    }
  }
  long long key_best = (live && lead && best_k >= 0) ? ((best_f << 20) | (long long)rho) : LLONG_MAX;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const long long other = __shfl_xor_sync(kFull, key_best, o);
    key_best = other < key_best ? other : key_best;
  }
  if (contribute && lane == 0 && key_best != LLONG_MAX && a.out.inst_best)
    atomicMin(reinterpret_cast<long long *>(a.out.inst_best) + s, key_best);
  if (a.out.counters && contribute) {
    const unsigned long long nl = live ? 1ull : 0ull;
    const unsigned long long g0 = (live && lead) ? 1ull : 0ull;
    const unsigned long long fl = warp_sum_u64(nl * c_flips), un = warp_sum_u64(nl * c_unif);
    const unsigned long long fp = warp_sum_u64(nl * c_fp64), uc = warp_sum_u64(nl * c_unc);
    const unsigned long long ph = warp_sum_u64(nl * c_philox), nf = warp_sum_u64(g0 * (unsigned long long)nfeas);
    const unsigned long long lv = warp_sum_u64(g0);
#ifdef SAIM_DEBUG_SPLIT
    if (blockIdx.x == 0 && blockIdx.y == 0 && warp == 0)
      printf("lane %d live %d lead %d g0 %llu c_philox %u c_flips %u lv %llu ph %llu N %d\n", lane, (int)live, (int)lead, g0,
             c_philox, c_flips, lv, ph, N);
#endif
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
typedef void (*mkps_kernel_t)(const RunArgs);

template <bool RPV>
static mkps_kernel_t mkps_kernel_for_t(int MM, int M) {
  if (MM == 16 && M == 10) return saim_mkp_split_kernel<16, 10, 2, RPV>;
  if (MM == 32 && M == 30) return saim_mkp_split_kernel<32, 30, 2, RPV>;
  switch (MM) {
    case 16: return saim_mkp_split_kernel<16, 16, 2, RPV>;
    case 32: return saim_mkp_split_kernel<32, 32, 2, RPV>;
    default: return nullptr;
  }
}

}  // namespace saim
