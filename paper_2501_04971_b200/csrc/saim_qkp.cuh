// saim_qkp.cuh -- fused SAIM kernel template for problems with a quadratic objective and M <= 1
// constraint (QKP; BASELINE.json configs 0-2).  sm_100a.
//
// One warp = one replica (an independent SAIM chain, R22); one CTA = up to 32 replicas of the
// same instance sharing that instance's Q, A_ext and c in shared memory (TMA bulk-staged once).
// The whole of Algorithm 1 runs inside the kernel: K anneals of T sweeps of
// N sequential p-bit decisions (Eq. 9-10), per-anneal readout, best
// tracking and the Lagrange step.  Nothing crosses the host boundary between iterations.
//
// Exact sequential semantics with 32 lanes: lane l owns the
// spins i = 32b + l.  For block b every pending lane evaluates its decision against the current
// state; a ballot finds the first lane whose decision flips its spin; decisions of the lanes
// before it (and its own) are final -- they were taken on exactly the state the sequential sweep
// would have seen.  The flip is applied (phi_j -= delta Q_ij for every item j, r += delta A_i) and
// the lanes after it re-evaluate with the SAME uniforms (counter-based Philox, R2).  A block
// costs 1 + (#flips in it) rounds.
//
// Field of spin i in binary form (R1): F_i = c_o phi_i - A_i (c_p v_i + c_l Lambda), with
// v_i = 2 r0 + A_i = 2r + A_i (1 - 2 x_i) (Eq. 3 and Eq. 5 differences, M = 1), z = beta_t F_i.
// phi_i, r, v_i are exact integers held in fp32 (|.| < 2^22, proved on the host).  The decision
// [u < sigma(z)] <=> [z > logit(u)] is taken in fp32 with a rigorous error bound e: saturated
// when |z| - e > ln(2^24-1) (no uniform needed, R19), else compared with logit(u) evaluated with
// MUFU lg2; inside the combined error band it is re-done in fp64 (R18).
#pragma once
#include <climits>
#include <cstdint>
#include <cstdio>
#include <cstring>

#include "saim_dev.cuh"

#ifdef SAIM_PROF
__device__ unsigned long long saim_prof[48];  // profiling build only (read by saim_prof_read, saim_qkp.cu)
#endif

namespace saim {

namespace {

constexpr uint32_t kFull = 0xffffffffu;
// fp32 field: |z_f32 - z| <= 2^-20 * S with S = |K1 phi| + |A|(|K2 v| + |K3|).  The true bound
// is ~3 * 2^-24 (three roundings plus fp32-rounded constants): a 5x margin.  The saturation test
// |z| - 2^-20 S > ln(2^24-1) is evaluated as fl(z * (+-2^20) - S) > 2^20 * kSatThr (one FFMA with
// an immediate; its single rounding costs < 1e-6 of the 7.7e-6 margin built into kSatThr).
constexpr float kZScale = 1048576.0f;                 // 2^20 = 1 / kZRel
constexpr float kSatThr20 = kSatThr * 1048576.0f;     // exact (power-of-two scaling)
// 28 warps x 32 lanes: one CTA of 28 replicas per SM covers 4096 replicas in one wave (<= 72 regs).
constexpr int kQkpMaxThreads = 896;

// kDivMagic[p] = ceil(2^16 / p): (x * kDivMagic[p]) >> 16 == x / p for all x <= 32, p in [1, 32]
// (checked exhaustively; tests/test_abi.py)
__constant__ uint32_t kDivMagic[33] = {
    0,     65536, 32768, 21846, 16384, 13108, 10923, 9363, 8192, 7282, 6554, 5958, 5462, 5042, 4682, 4370, 4096,
    3856,  3641,  3450,  3277,  3121,  2979,  2850,  2731, 2622, 2521, 2428, 2341, 2260, 2185, 2115, 2048};

// Shared-memory word by 32-bit shared-window address (apply_flip keeps the Q base as such an
// address: through a generic pointer the compiler rebuilt the window base -- S2UR/UMOV/UIADD3/ULEA
// -- on every flip).
__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}

__device__ __forceinline__ uint32_t sel4(const uint4 &u, int i) {
  return i == 0 ? u.x : (i == 1 ? u.y : (i == 2 ? u.z : u.w));
}


// Per-warp cold state in shared memory (kept out of the register file: the hot loop runs at
// 28 warps/SM, i.e. <= 72 registers per thread).
struct WarpState {
  float k1s, k2s, k3s;             // per unit t: K1 = t*bstep*c_o, K2 = t*bstep*c_p, K3 = t*bstep*c_l*Lambda
  float e0s, e1s;                  // scan error bound per unit t: e(A) = t*(e0s + e1s*A)
  int tden;                        // T - 1 (1 when T == 1): beta_t = beta_max t / tden exactly
  int force_dd;                    // SAIM_FLAG_TEST_REPLAY: treat every fp64-band decision as uncertified
  double bstep;                    // beta_max / (T-1)   (or beta_max with t := 1 when T == 1)
  long long Lam;                   // Lambda_k (Lambda_0 = 0)
  long long best_f;
  int best_k, nfeas;
  uint32_t cnt[6];                 // flips, uniforms, fp64, uncertified, philox, sweeps evaluated
  uint32_t best_word[32];
  uint2 key;                        // Philox key (lo32 seed, hi32 seed)
  uint32_t srho;                    // (s << 20) | rho
  uint32_t uw[4][32];               // lazily drawn words of the current group, per lane
#ifdef SAIM_PROF
  uint32_t prof[48];               // per 1/16 of the anneal: cycles, sweep-loop iterations, flips
#endif
};
enum { kCntFlips = 0, kCntUnif, kCntFp64, kCntUncert, kCntPhilox, kCntSweeps };

__device__ __forceinline__ void cnt_add(WarpState *ws, int i, uint32_t v) {
  if ((threadIdx.x & 31) == 0) ws->cnt[i] += v;      // warp-uniform events, counted once
}

// fp64 re-evaluation of one decision (R18 slow path).  Constants are re-derived in
// fp64 from the instance header; the bound 2^-47 (S + 1 + |l|) covers their few-ulp roundings.
// A decision inside that bound is certified by the double-double level (decide_dd, saim_dev.cuh)
// -- but only in the replay kernel (RP): a call to it from the main kernel would widen the
// registers this call clobbers and cost the hot loop ~10% (measured), so the main kernel returns
// the fp64 guess flagged uncertified and the replica is re-run exactly by the replay launch
// (DESIGN.md 6.1 "Exact replay").
template <bool RP>
__device__ __noinline__ int decide_fp64(float phib, float v, float A, int t, const InstHdr *H, const WarpState *ws,
                                        uint32_t w) {
  const double beta = ws->bstep * (double)t;
  const double K1d = beta * H->c_o, K2d = beta * H->c_p, K3d = beta * (H->c_l * (double)ws->Lam);
  const double Ad = (double)A, vd = (double)v, pd = (double)phib;
  const double z = fma(K1d, pd, -(Ad * fma(K2d, vd, K3d)));
  const double S = fabs(K1d * pd) + fabs(Ad) * (fabs(K2d * vd) + fabs(K3d));
  const double d = z - logit_f64(H, w);
  const double e = (S + 1.0 + fabs(z)) * 0x1p-47;
  if constexpr (!RP) {
    return (d > 0.0 ? 1 : 0) | (fabs(d) <= e ? 2 : 0);
  } else {
    if (fabs(d) > e && !ws->force_dd) return d > 0.0 ? 1 : 0;
    // third level: double-double on the exact integers (pi = A v, kappa = A Lambda)
    const long long Ai = (long long)A;
    return decide_dd((long long)phib, Ai * (long long)v, Ai * ws->Lam, t, ws->tden, H, w);
  }
}

// Lazily drawn uniforms of a group (key schedule from the kernel-parameter bank, RunArgs::ks):
// the empty volatile asm is a side effect, so the compiler cannot speculatively hoist the
// 10-round Philox into the common (saturated) path.
__device__ __forceinline__ uint4 philox_group_lazy_ks(const uint32_t (&ks)[20], int g, int lane, int t, int k,
                                                      uint32_t srho) {
  uint32_t x = 32u * (uint32_t)g + (uint32_t)lane;
  asm volatile("" : "+r"(x));
  return philox4x32_10_ks(make_uint4(x, (uint32_t)t, (uint32_t)k, srho), ks);
}

}  // namespace

// Blocks of the padded spin range: NPL item blocks + up to 2 slack blocks, rounded up to a whole
// 4-block group (spins >= N carry A = NaN, which the scan treats as quiet).
template <int NPL>
__host__ __device__ constexpr int qkp_nbp() {
  return ((NPL + 2) + 3) & ~3;
}
template <int NPL>
__host__ __device__ constexpr int qkp_warp_smem_bytes() {
  return (2 * qkp_nbp<NPL>() * 32 * 4 + (int)sizeof(WarpState) + 15) & ~15;
}

// Shared memory: [instance blob: Q rows | A_ext (NaN-padded) | c]
//                [per warp: phs = (2x-1) phi | asg = (2x-1) A, each NBP*32 floats | WarpState]
// PK (packed phi, int8 Q with |phi| <= 32767 in every state, host-proven): the phs region holds
// instead phw[p][lane] = (phi_{32(2p)+lane} + 2^15) | (phi_{32(2p+1)+lane} + 2^15) << 16, the
// unsigned phi of two blocks per word.  A Q-row update is then one packed integer add per two
// items: both 16-bit halves stay in [1, 65535], so no carry crosses between them.
//
// RP (replay kernel, DESIGN.md 6.1 "Exact replay"): launched after the main kernel over the same
// grid; only the replicas the main kernel flagged (a decision its fp64 level could not certify)
// run again, from the start, with the double-double level enabled, and their outputs replace the
// main kernel's.  A CTA with no flagged replica exits before staging anything.
template <int NPL, int QB, bool PK, bool RP>
__global__ void __launch_bounds__(kQkpMaxThreads, 1) saim_qkp_kernel(const RunArgs a) {
  constexpr int E = 4 / QB;                          // Q entries per 32-bit word
  constexpr int QW = (NPL + E - 1) / E;              // words per lane per Q row
  constexpr int NBP = qkp_nbp<NPL>();
  constexpr float kQBias = (float)(1 << (8 * QB - 1));
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ uint64_t mbar;

  const int s = blockIdx.y;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int ridx = blockIdx.x * (blockDim.x >> 5) + warp;
  if constexpr (RP) {
    const bool flagged = ridx < a.R && a.replay[replay_slot(warp)];
    if (!__syncthreads_or(flagged)) return;           // nothing to replay in this CTA
  }
  bulk_stage(smem, a.blob + (size_t)s * a.blob_bytes, a.blob_bytes, &mbar);

  if (ridx >= a.R) return;
  if constexpr (RP) {
    if (!a.replay[replay_slot(warp)]) return;
  }
  const InstHdr *Hp = a.hdr + s;
  // blob layout [A_ext | c | Q rows] (saim_layout.h): compile-time offsets from one base
  constexpr uint32_t kCOff = (NBP * 32 * 4 + 15) & ~15u, kQOff = kCOff + ((NPL * 32 * 4 + 15) & ~15u);
  const float *sAl = reinterpret_cast<const float *>(smem) + lane;              // A_ext[32b + lane] (NaN-padded)
  const int32_t *sC = reinterpret_cast<const int32_t *>(smem + kCOff);
  const uint32_t *sQl = reinterpret_cast<const uint32_t *>(smem + kQOff) + lane;  // Q word (row 0, w 0) of this lane
  // ... as a shared-window address: the Q row of a flip is read through it when NPL > 4 (config 2
  // 96.7 -> 94.3 ms; at NPL <= 4 the generic pointer measured 2.6% faster, config 1)
  constexpr bool kQAddr = NPL > 4;
  uint32_t sQa = kQAddr ? (uint32_t)__cvta_generic_to_shared(sQl) : 0u;
  if constexpr (kQAddr) asm volatile("" : "+r"(sQa));
  // word w of this lane in the Q row of spin j
  auto qword = [&](const uint32_t *rowp, uint32_t rowa, int w) -> uint32_t {
    if constexpr (kQAddr) return lds_u32(rowa + 128u * (uint32_t)w);
    else return rowp[32 * w];
  };
  unsigned char *wbase = smem + a.blob_bytes + warp * qkp_warp_smem_bytes<NPL>();
  float *phs = reinterpret_cast<float *>(wbase) + lane;                        // (2x_i - 1) phi_i, i = 32b + lane
  uint32_t *phw = reinterpret_cast<uint32_t *>(wbase) + lane;                  // PK: packed phi pairs
  float *asg = reinterpret_cast<float *>(wbase) + NBP * 32 + lane;             // (2x_i - 1) A_i
  WarpState *ws = reinterpret_cast<WarpState *>(wbase + 2 * NBP * 32 * 4);
  const int n = a.n;
  const int N = Hp->N;
  const int NB = (N + 31) >> 5;                      // NB <= NPL + 2
  const int NG = (NB + 3) >> 2;
  const uint32_t allb = (1u << NB) - 1u;             // NB <= 18 (padding blocks are never visited)
  const bool has_con = a.M > 0;

  // x = 0: phi_i = -c_i, so (2x-1) phi = c_i; (2x-1) A = -A.
#pragma unroll
  for (int m = 0; m < NBP; ++m) {
    if constexpr (PK) {
      const uint32_t h = 32768u - (uint32_t)((32 * m + lane < n) ? sC[32 * m + lane] : 0);
      if (m & 1) phw[32 * (m >> 1)] |= h << 16; else phw[32 * (m >> 1)] = h;
    } else {
      phs[32 * m] = (32 * m + lane < n) ? (float)sC[32 * m + lane] : 0.0f;
    }
    asg[32 * m] = -sAl[32 * m];
  }
  // phi_i of this lane's spin in block b (PK: exact via the 2^23 magic-number conversion)
  auto phi_pk = [&](int b) -> float {
    return __uint_as_float(__byte_perm(phw[32 * (b >> 1)], 0x4B000000u, (b & 1) ? 0x7632u : 0x7610u)) -
           (8388608.0f + 32768.0f);
  };
  if (lane == 0) {
    const double bstep = (a.T >= 2) ? a.beta_max / (double)(a.T - 1) : a.beta_max;
    ws->bstep = bstep;
    ws->tden = (a.T >= 2) ? a.T - 1 : 1;
    ws->force_dd = (a.flags & SAIM_FLAG_TEST_REPLAY) ? 1 : 0;
    ws->k1s = (float)(bstep * Hp->c_o);
    ws->k2s = (float)(bstep * Hp->c_p);
    ws->k3s = 0.0f;
    ws->e0s = (float)(bstep * Hp->c_o * Hp->phi_bound * 0x1p-20);
    // 2^-20 S error bound, plus the certificate tolerance: |2r - 2r_cert| <= 2D moves (2x-1) z by
    // at most 2 K2 D |A| (margin 1.001 over the fp32 rounding of K2)
    ws->e1s = (float)(bstep * Hp->c_p * (Hp->v_bound * 0x1p-20 + 1.001 * (double)a.rtol2));
    ws->Lam = 0;
    ws->best_f = LLONG_MAX;
    ws->best_k = -1;
    ws->nfeas = 0;
#ifdef SAIM_PROF
    for (int i = 0; i < 48; ++i) ws->prof[i] = 0;
#endif
#pragma unroll
    for (int i = 0; i < 6; ++i) ws->cnt[i] = 0;
  }
  ws->best_word[lane] = 0;
  __syncwarp();
  uint32_t xm = 0;                                  // bit b = x_{32b + lane}
  uint32_t nflip = 0;                               // flips so far (warp-uniform)
  uint32_t qmask = 0;                               // blocks certified quiet since the last flip
  uint32_t dense = 0;                               // groups processed without scans (bit g)
  uint32_t nunif = 0, nphil = 0;                    // uniforms drawn, lazy Philox calls x 32 (sweeps t >= 1)
  float r2 = has_con ? (float)(-2 * Hp->b0) : 0.0f; // 2r, r = A_ext x - b (exact integer)

  if (lane == 0) {
    ws->key = make_uint2((uint32_t)a.seed, (uint32_t)(a.seed >> 32));
    ws->srho = ((uint32_t)s << 20) | (uint32_t)(a.rep0 + ridx);
  }
  __syncwarp();

  // Flip of spin j = 32b + L by delta = dl (+1/-1): Eq. 9 in incremental form.
  //   own lane: x_j, and the signs of its (2x-1) phi, (2x-1) A;  all lanes: phi_i -= delta Q_ij
  //   (stored as (2x_i - 1) phi_i), r += delta A_j.
  auto apply_flip = [&](int b, int L, float AL, float dl) {
    r2 = fmaf(dl + dl, AL, r2);
    if (lane == L) {
      xm ^= (1u << b);
      if constexpr (!PK) phs[32 * b] = -phs[32 * b];
      asg[32 * b] = -asg[32 * b];
    }
    const int j = 32 * b + L;
    if (j < n) {                                    // an item flip moves phi: certificates void
      qmask = 0u;
      const uint32_t *row = sQl + j * (QW * 32);
      const uint32_t rowa = sQa + (uint32_t)(j * (QW * 128));
      if constexpr (PK) {
        // phi_i -= delta Q_ij on two items per word: pq = biased bytes (Q + 128) of entries
        // (2p, 2p+1) as 16-bit halves, phi - delta (pq - 0x00800080)
        if (dl > 0.0f) {
#pragma unroll
          for (int w = 0; w < QW; ++w) {
            const uint32_t word = qword(row, rowa, w);
#pragma unroll
            for (int h = 0; h < 2; ++h)
              if (4 * w + 2 * h < NPL)
                phw[32 * (2 * w + h)] = phw[32 * (2 * w + h)] - __byte_perm(word, 0u, h ? 0x4342u : 0x4140u) + 0x00800080u;
          }
        } else {
#pragma unroll
          for (int w = 0; w < QW; ++w) {
            const uint32_t word = qword(row, rowa, w);
#pragma unroll
            for (int h = 0; h < 2; ++h)
              if (4 * w + 2 * h < NPL)
                phw[32 * (2 * w + h)] = phw[32 * (2 * w + h)] + __byte_perm(word, 0u, h ? 0x4342u : 0x4140u) - 0x00800080u;
          }
        }
      } else {
#pragma unroll
        for (int w = 0; w < QW; ++w) {
          const uint32_t word = qword(row, rowa, w);
#pragma unroll
          for (int e = 0; e < E; ++e) {
            const int m = E * w + e;
            if (m < NPL) {
              const uint32_t selr = (QB == 1) ? (0x7650u | (uint32_t)e) : (0x7600u | ((2u * e + 1u) << 4) | (2u * e));
              const float q = __uint_as_float(__byte_perm(word, 0x4B000000u, selr)) - (8388608.0f + kQBias);
              const float sdl = ((xm >> m) & 1u) ? dl : -dl;           // (2x_i - 1) delta
              phs[32 * m] = fmaf(-sdl, q, phs[32 * m]);
            }
          }
        }
      }
    }
    ++nflip;
  };
  // Quiet certificates are made with margin for any 2r within
  // +-rtol2 of r2c, the value of 2r when they were made: blocks found quiet at another r replace
  // the current certificates (the others are scanned again next sweep).
  float r2c = 0.0f;
  auto certify = [&](uint32_t bits) {
    if (!qmask || r2 != r2c) { r2c = r2; qmask = bits; } else { qmask |= bits; }
  };

  for (int k = 0; k < a.K; ++k) {
    int t0 = 0;
    if (a.T >= 2) {
      // ---- sweep t = 0: beta_0 = 0, x_i = [u < 1/2] (state-independent; R3, R5) ----
      t0 = 1;
      if constexpr (PK) {
        // Every decision of sweep 0 is state-independent, so the new state x' is known at once
        // and phi' = phi - sum over flipped items j of delta_j Q_j: the Q rows are summed into
        // packed registers (exact integer sums in any order; every partial sum is phi of the state
        // with the flips added so far, so it stays within the proven |phi| bound and no 16-bit
        // half carries).
        uint32_t xn = 0;                                  // bit b = x'_{32b + lane}
        for (int g = 0; g < NG; ++g) {
          const uint4 uw = philox_group_lazy_ks(a.ks, g, lane, 0, k, ws->srho);
          cnt_add(ws, kCntPhilox, 32);
#pragma unroll
          for (int bb = 0; bb < 4; ++bb) {
            const int b = 4 * g + bb;
            if (b < NB) {
              const bool valid = lane < N - 32 * b;
              if (valid && (sel4(uw, bb) >> 31) == 0u) xn |= 1u << b;   // u < 1/2  <=>  w < 2^31
              cnt_add(ws, kCntUnif, __popc(__ballot_sync(kFull, valid)));
            }
          }
        }
        const uint32_t dx = xn ^ xm;                      // flipped blocks of this lane
        constexpr int PW = (NPL + 1) / 2;                 // packed phi words holding items
        uint32_t acc[PW];
#pragma unroll
        for (int p = 0; p < PW; ++p) acc[p] = phw[32 * p];
        for (int b = 0; b < NPL; ++b) {
          uint32_t fb = __ballot_sync(kFull, ((dx >> b) & 1u) && 32 * b + lane < n);
          const uint32_t up = __ballot_sync(kFull, (xn >> b) & 1u);
          while (fb) {
            const int L = __ffs(fb) - 1;
            fb &= fb - 1u;
            const uint32_t *row = sQl + (32 * b + L) * (QW * 32);
            const uint32_t rowa = sQa + (uint32_t)((32 * b + L) * (QW * 128));
            if ((up >> L) & 1u) {                         // 0 -> 1: phi -= Q_j
#pragma unroll
              for (int w = 0; w < QW; ++w) {
                const uint32_t word = qword(row, rowa, w);
#pragma unroll
                for (int h = 0; h < 2; ++h)
                  if (2 * w + h < PW) acc[2 * w + h] = acc[2 * w + h] - __byte_perm(word, 0u, h ? 0x4342u : 0x4140u) + 0x00800080u;
              }
            } else {                                      // 1 -> 0: phi += Q_j
#pragma unroll
              for (int w = 0; w < QW; ++w) {
                const uint32_t word = qword(row, rowa, w);
#pragma unroll
                for (int h = 0; h < 2; ++h)
                  if (2 * w + h < PW) acc[2 * w + h] = acc[2 * w + h] + __byte_perm(word, 0u, h ? 0x4342u : 0x4140u) - 0x00800080u;
              }
            }
          }
        }
#pragma unroll
        for (int p = 0; p < PW; ++p) phw[32 * p] = acc[p];
        int load = 0;                                     // sum_i A_ext,i x'_i (exact)
#pragma unroll
        for (int m = 0; m < NBP; ++m) {
          if ((dx >> m) & 1u) asg[32 * m] = -asg[32 * m];
          if ((xn >> m) & 1u) load += (int)sAl[32 * m];
          nflip += __popc(__ballot_sync(kFull, (dx >> m) & 1u));
        }
        load = __reduce_add_sync(kFull, load);
        xm = xn;
        if (has_con) r2 = (float)(2 * ((long long)load - Hp->b0));
      } else {
        for (int g = 0; g < NG; ++g) {
          const uint4 uw = philox_group(ws->key, g, lane, 0, k, ws->srho);
          cnt_add(ws, kCntPhilox, 32);
#pragma unroll
          for (int bb = 0; bb < 4; ++bb) {
            const int b = 4 * g + bb;
            if (b < NB) {
              const bool valid = lane < N - 32 * b;
              const int xb = (xm >> b) & 1u;
              const int nx = (sel4(uw, bb) >> 31) == 0u;   // u < 1/2  <=>  w < 2^31
              uint32_t fm = __ballot_sync(kFull, valid && nx != xb);
              cnt_add(ws, kCntUnif, __popc(__ballot_sync(kFull, valid)));
              const float A = sAl[32 * b];
              while (fm) {
                const int L = __ffs(fm) - 1;
                fm &= fm - 1u;
                apply_flip(b, L, __shfl_sync(kFull, A, L), __shfl_sync(kFull, nx, L) ? 1.0f : -1.0f);
              }
            }
          }
        }
      }
    }
    const bool freeze_exit = !(a.flags & SAIM_FLAG_NO_FREEZE_EXIT);
    const bool hot_loop = a.T >= 2 && !(a.flags & SAIM_FLAG_QKP_NO_HOT_LOOP);
    qmask = 0u;                                         // new Lambda_k: every group is scanned again
    dense = 0u;
    for (int t = t0; t < a.T; ++t) {
#ifdef SAIM_PROF
      const long long prof_c0 = clock64();
      const uint32_t prof_f0 = nflip;
#endif
      // ---- Hot-block loop ----
      // Every block but one (b) is certified quiet: those keep their spins whatever happens in b
      // as long as nothing flips.  While b's own decisions flip nothing, its fields stay constant
      // and a whole sweep is just b's 32 decisions: run such sweeps back to back here.  The sweep
      // in which b would flip a spin (or turns quiet) is left to the general path below, which
      // re-derives the same decisions from the same state and uniforms.  Sweeps are evaluated
      // 32 / pw at a time (pw = width of b's unsaturated lanes), one lane per (spin, sweep).
      if (hot_loop && qmask != allb && !((allb & ~qmask) & ((allb & ~qmask) - 1u))) {
        const int b = __ffs(allb & ~qmask) - 1;
        const int bb = b & 3, gq = b >> 2;
        const float A = sAl[32 * b];
        bool xb = (xm >> b) & 1u;
        float sg = xb ? -1.0f : 1.0f;
        const float phib = PK ? phi_pk(b) : -sg * phs[32 * b];   // phi: constant (items do not flip here)
        float v = fmaf(A, sg, r2);
        const bool mine = lane < N - 32 * b;
        const float k1s = ws->k1s, k2s = ws->k2s, k3s = ws->k3s;
        // The fields are constant here, so z = t z1 and S = t S1 with z1, S1 per unit t: 5
        // roundings of S at most (3 of the fp32 constants and z1, one of t z1), inside the 2^-20 S
        // bound the decisions below use.
        const float Ak2 = A * k2s, Ak3 = A * k3s;
        float z1 = fmaf(k1s, phib, -fmaf(Ak2, v, Ak3));
        float S1 = fmaf(k1s, fabsf(phib), fmaf(fabsf(Ak2), fabsf(v), fabsf(Ak3)));
        float tf = (float)t;                                // exact (t < 2^24)
        // the current window: sweeps [wb, wb + pS), lane j holding spin lane sp = plo + j % pw at
        // sweep wb + sj (sj = j / pw), its Philox word w and logit l
        int wb = -1, plo = 0, pw = 32, sj = 0, sp = 0, pS = 0;
        uint32_t grp = kFull, w = 0;
        float l = 0.0f;
        for (; t < a.T;) {
          // One step covers sweeps [t, t + pS): on sweep t the saturated lanes of b are certified
          // for every later sweep too (constant fields, |z| = t |z1| grows with t); the pw lanes
          // [plo, plo + pw) that are not saturated at t are evaluated for pS = 32 / pw sweeps at
          // once, lane j taking spin lane sp = plo + j % pw at sweep t + j / pw with its own
          // Philox word.  All sweeps before the first one with a flip are complete (nothing
          // changed); that sweep is finished here if its only flip is an in-window slack flip,
          // else left to the general path.
          const float z = tf * z1, S = tf * S1;
          const bool sat = fabsf(z) * kZScale - S > kSatThr20;
          const uint32_t need = __ballot_sync(kFull, mine && !sat);
          if (!need) break;                               // b quiet: general path
          const uint32_t fs = __ballot_sync(kFull, mine && sat && (z > 0.0f) != xb);   // saturated flips at t
          // A new window unless the current one still covers sweep t and every unsaturated lane
          // (after an in-place slack flip the later sweeps' words stay valid: uniforms depend on
          // (spin, sweep) only)
          if (wb < 0 || t - wb >= pS || (need & ~(grp << plo))) {
            plo = __ffs(need) - 1;
            pw = 32 - __clz(need) - plo;
            const uint32_t dm = kDivMagic[pw];
            sj = (int)(((uint32_t)lane * dm) >> 16);      // lane / pw
            sp = plo + lane - sj * pw;
            pS = min((int)((32u * dm) >> 16), a.T - t);
            grp = (pw == 32) ? kFull : ((1u << pw) - 1u);
            wb = t;
            // R2 counter of (spin 32 b + sp, sweep t + sj); key schedule from the parameter bank
            w = sel4(philox4x32_10_ks(make_uint4(32u * (uint32_t)gq + (uint32_t)sp, (uint32_t)(t + sj), (uint32_t)k,
                                                 ws->srho), a.ks), bb);
            l = logit_f32(w);
            nphil += 32u;
          }
          const int c0 = t - wb;                          // first sweep of the window still open
          const bool valid = sj >= c0 && sj < pS;
          const float z1j = __shfl_sync(kFull, z1, sp), S1j = __shfl_sync(kFull, S1, sp);
          const int xbj = __shfl_sync(kFull, (int)xb, sp);
          const float tfj = (float)(wb + sj);             // exact
          const float zj = tfj * z1j, Sj = tfj * S1j;
          const bool satj = fabsf(zj) * kZScale - Sj > kSatThr20;
          const float d = zj - l;
          int nxj = satj ? (zj > 0.0f) : (d > 0.0f);
          const bool band = valid && !satj &&
                            !(fabsf(d) > (Sj * (1.0f / kZScale) + kLogitAbs + kLogitRel * fabsf(l)) * 1.0001f);
          if (__any_sync(kFull, band)) {                  // rare: fp64 re-evaluation
            const float phj = __shfl_sync(kFull, phib, sp), vj = __shfl_sync(kFull, v, sp);
            const float Aj = __shfl_sync(kFull, A, sp);
            if (band) {
              const int rs = decide_fp64<RP>(phj, vj, Aj, wb + sj, Hp, ws, w);
              nxj = rs & 1;
              atomicAdd(&ws->cnt[kCntFp64], 1u);
              if (rs & 2) atomicAdd(&ws->cnt[kCntUncert], 1u);
            }
          }
          const uint32_t fmj = __ballot_sync(kFull, valid && nxj != xbj);
          const uint32_t ndj = __ballot_sync(kFull, valid && !satj);
          // cf = first window sweep (>= c0) with a flip, q = first one in which every lane of b is
          // saturated (pS if none): sweeps [wb + c0, wb + min(cf, q)) are complete
          const int cf = fs ? c0 : (fmj ? __shfl_sync(kFull, sj, __ffs(fmj) - 1) : pS);
          const uint32_t qv = __ballot_sync(kFull, valid && sp == plo && ((ndj >> ((sj * pw) & 31)) & grp) == 0u);
          const int q = qv ? __shfl_sync(kFull, sj, __ffs(qv) - 1) : pS;
          const int c = min(cf, q);
          const int cw = c * pw;
          nunif += __popc(cw >= 32 ? ndj : (ndj & ((1u << cw) - 1u)));   // (bits below c0 pw are 0)
          t = wb + c;
          tf = (float)t;
          if (c == pS) { wb = -1; continue; }             // window done
          if (q == c) break;                              // b quiet at t: the general path certifies it
          // Sweep t has a flip; the first one in spin order is lane L.  (cw < 32 here.)
          const uint32_t F = (((fmj >> cw) & grp) << plo) | fs;
          const int L = __ffs(F) - 1;
          const float dl = __shfl_sync(kFull, (int)xb, L) ? -1.0f : 1.0f;
          const float r2n = fmaf(dl + dl, __shfl_sync(kFull, A, L), r2);
          if (32 * b + L < n || fabsf(r2n - r2c) > a.rtol2) break;
          // A single slack flip inside the certificates' window: the later lanes of b are
          // re-evaluated on the new r with the same uniforms (held by lanes cw + lane - plo)
          const float v2 = fmaf(A, sg, r2n);
          const float z2 = tf * fmaf(k1s, phib, -fmaf(Ak2, v2, Ak3));
          const float S2 = tf * fmaf(k1s, fabsf(phib), fmaf(fabsf(Ak2), fabsf(v2), fabsf(Ak3)));
          const bool mine2 = mine && lane > L;
          const bool sat2 = fabsf(z2) * kZScale - S2 > kSatThr20;
          int nx2 = z2 > 0.0f;
          const uint32_t need2 = __ballot_sync(kFull, mine2 && !sat2);
          if (need2 & ~(grp << plo)) break;               // (words not at hand: general path)
          const int src = (cw + lane - plo) & 31;
          const float l2 = __shfl_sync(kFull, l, src);
          bool band2 = false;
          if (mine2 && !sat2) {
            const float d2 = z2 - l2;
            nx2 = d2 > 0.0f;
            band2 = !(fabsf(d2) > (S2 * (1.0f / kZScale) + kLogitAbs + kLogitRel * fabsf(l2)) * 1.0001f);
          }
          if (__any_sync(kFull, band2)) {
            const uint32_t w2 = __shfl_sync(kFull, w, src);
            if (band2) {
              const int rs = decide_fp64<RP>(phib, v2, A, t, Hp, ws, w2);
              nx2 = rs & 1;
              atomicAdd(&ws->cnt[kCntFp64], 1u);
              if (rs & 2) atomicAdd(&ws->cnt[kCntUncert], 1u);
            }
          }
          if (__ballot_sync(kFull, mine2 && nx2 != (int)xb)) break;
          r2 = r2n;                                       // apply the slack flip: r += delta A_L
          if (lane == L) {
            xm ^= (1u << b);
            if constexpr (!PK) phs[32 * b] = -phs[32 * b];
            asg[32 * b] = -asg[32 * b];
            xb = !xb;
            sg = -sg;
          }
          v = fmaf(A, sg, r2);
          z1 = fmaf(k1s, phib, -fmaf(Ak2, v, Ak3));
          S1 = fmaf(k1s, fabsf(phib), fmaf(fabsf(Ak2), fabsf(v), fabsf(Ak3)));
          ++nflip;
          nunif += __popc((((ndj >> cw) & grp) << plo) | need2);
          ++t;
          tf += 1.0f;
        }
        if (t >= a.T) break;
      }
      const float tf = (a.T >= 2) ? (float)t : 1.0f;     // exact
      bool active = false;                            // any non-quiet lane in this sweep?
      // fp32 sweep constants (two roundings each; the bounds below keep a >= 3x margin)
      const float K1 = tf * ws->k1s, K2 = tf * ws->k2s, K3 = tf * ws->k3s;
      // Scan threshold: quiet <=> (2x-1) z_f32 > kSatThr + t*(e0s + e1s*A), where the second term
      // bounds |z_f32 - z| for every reachable state (phi_bound, v_bound; 4x margin over 3*2^-24).
      const float B0 = fmaf(tf, ws->e0s, kSatThr), B1 = tf * ws->e1s;
      int g = 0;                                          // current 128-spin group (4 blocks)

      // Exact sequential processing of block b (bb = b % 4) from the current state: rounds of
      // evaluate -> ballot first flipper -> flip, until every lane of the block is decided.
      // Returns bit 0: a spin of the block flipped; bit 1: some lane was not saturated.
      auto process_block = [&](int b, int bb) -> int {
        const int hi = N - 32 * b;                        // lanes < hi hold a spin
        const float A = sAl[32 * b];
        const bool xb = (xm >> b) & 1u;
        const float AK2 = A * K2, AK3 = A * K3;
        const float sg = xb ? -1.0f : 1.0f;              // 1 - 2x_i
        bool flipped = false;
        // logit of this lane's uniform, once per visit (99.8% of visits need some lane's at config 2)
        const uint32_t w = ws->uw[bb][lane];
        const float l = logit_f32(w);
        const float el = kLogitAbs + kLogitRel * fabsf(l);
        uint32_t drew = 0;                                // lanes that needed their uniform in this visit
        int lo = 0;                                       // lanes in [lo, hi) are still pending
        for (;;) {
          const float phib = PK ? phi_pk(b) : -sg * phs[32 * b];   // phi_i
          const float v = fmaf(A, sg, r2);                // 2 r0 + A
          const float z = fmaf(K1, phib, -fmaf(AK2, v, AK3));            // beta_t F_i (fp32)
          const float S = fmaf(K1, fabsf(phib), fmaf(fabsf(AK2), fabsf(v), fabsf(AK3)));
          const bool mine = lane >= lo && lane < hi;
          const bool sat = fabsf(z) * kZScale - S > kSatThr20;
          int nx = z > 0.0f;
          if constexpr (NPL <= 4) {
            // small instances (<= 128 items, configs 0-1): branch-free decision, only the rare
            // fp64 re-evaluation behind a vote (measured 1.7-4% faster there; at NPL = 10 the
            // branchy form below is 1% faster)
            const bool ns = mine && !sat;
            drew |= __ballot_sync(kFull, ns);
            const float d = z - l;
            if (ns) nx = d > 0.0f;
            const bool band = ns && !(fabsf(d) > (S * (1.0f / kZScale) + el) * 1.0001f);
            if (__any_sync(kFull, band)) {
              if (band) {
                const int rs = decide_fp64<RP>(phib, v, A, a.T >= 2 ? t : 1, Hp, ws, w);
                nx = rs & 1;
                atomicAdd(&ws->cnt[kCntFp64], 1u);
                if (rs & 2) atomicAdd(&ws->cnt[kCntUncert], 1u);
              }
            }
          } else {
            const uint32_t need = __ballot_sync(kFull, mine && !sat);
            if (need) {
              drew |= need;
              if (mine && !sat) {
                const float d = z - l;
                if (fabsf(d) > (S * (1.0f / kZScale) + el) * 1.0001f) {
                  nx = d > 0.0f;
                } else {
                  const int rs = decide_fp64<RP>(phib, v, A, a.T >= 2 ? t : 1, Hp, ws, w);
                  nx = rs & 1;
                  atomicAdd(&ws->cnt[kCntFp64], 1u);
                  if (rs & 2) atomicAdd(&ws->cnt[kCntUncert], 1u);
                }
              }
            }
          }
          const uint32_t fm = __ballot_sync(kFull, mine && nx != (int)xb);
          if (!fm) break;
          const int L = __ffs(fm) - 1;
          apply_flip(b, L, __shfl_sync(kFull, A, L), __shfl_sync(kFull, nx, L) ? 1.0f : -1.0f);
          flipped = true;
          lo = L + 1;
          if (lo >= hi) break;
        }
        nunif += __popc(drew);
        return (flipped ? 1 : 0) | (drew ? 2 : 0);
      };

      // Speculative scan of one block on the current state: bit bb of nq is set if this lane's
      // spin is not certified quiet (saturated towards its current value).  With zz = (2x-1) z:
      //   zz = K1 (2x-1)phi - (2x-1)A (K2 v + K3),  v = 2r - (2x-1)A  = 2 r0 + A,
      //   quiet <=> zz > B0 + B1 |A|;  NaN padding (spins >= N) compares false -> quiet.
      auto scan_one = [&](uint32_t &nq, int b, int bb) {
        const float as = asg[32 * b];
        // (2x-1) phi: PK flips phi's sign bit with that of (2x-1) A (signed zero when A = 0)
        const float ph = PK ? __uint_as_float(__float_as_uint(phi_pk(b)) ^ (__float_as_uint(as) & 0x80000000u))
                            : phs[32 * b];
        const float v = r2 - as;
        const float tq = fmaf(K2, v, K3);
        const float zz = fmaf(K1, ph, -(as * tq));
        if (zz <= fmaf(B1, fabsf(as), B0)) nq |= 1u << bb;
      };
      // Process the non-quiet blocks of group g in order (exactly); after a flip the later
      // blocks' speculation is stale, so they are rescanned.
      // Dense groups (DESIGN.md 6.1 "Dense groups", dg): while every block of group g is
      // non-quiet (early in an anneal), its blocks are processed in order with no rescan after a
      // flip -- process_block alone decides every spin exactly; the first block found entirely
      // saturated with no flip sends the group back to scanning.
      auto handle_group = [&](uint32_t m, bool dg) {
        active = true;
        for (;;) {
          int bstart = 4;
          while (m) {
            const int bb = __ffs(m) - 1;
            m &= m - 1u;
            const int st = process_block(4 * g + bb, bb);
            if (dg) {
              if (!st) dense &= ~(1u << g);
            } else if (st & 1) {
              bstart = bb + 1;
              break;
            }
          }
          if (bstart >= 4) return;
          uint32_t nq = 0;
#pragma unroll
          for (int bb = 0; bb < 4; ++bb)
            if (bb >= bstart && 4 * g + bb < NB) scan_one(nq, 4 * g + bb, bb);
          m = __reduce_or_sync(kFull, nq);
          if (!m) return;
        }
      };

      // Quiet carry-over: a block whose every spin was certified
      // saturated towards its value stays so while no spin flips -- the fields are unchanged and
      // beta_t only grows, so (2x-1) z only moves away from the threshold.  Only the blocks not
      // so certified are scanned (4 per group in one pass); a flip voids every certificate, so
      // all later blocks follow.
      uint32_t todo = allb & ~qmask;
      while (todo) {
        g = (__ffs(todo) - 1) >> 2;
        const uint32_t gb = (todo >> (4 * g)) & 15u;        // blocks of group g to scan
        todo &= ~(15u << (4 * g));
        const bool dg = (dense >> g) & 1u;
        uint32_t m = gb;
        if (!dg) {
          uint32_t nq = 0;
#pragma unroll
          for (int bb = 0; bb < 4; ++bb)
            if ((gb >> bb) & 1u) scan_one(nq, 4 * g + bb, bb);
          m = __reduce_or_sync(kFull, nq);
          if (gb & ~m) certify((gb & ~m) << (4 * g));      // scanned and quiet: certified
          if (m == gb && gb == ((allb >> (4 * g)) & 15u)) dense |= 1u << g;   // no quiet block: dense
        }
        if (m) {
          // the group's uniform words, drawn once per visit of a group with a non-quiet block
          const uint4 u4 = philox_group_lazy_ks(a.ks, g, lane, t, k, ws->srho);
          ws->uw[0][lane] = u4.x; ws->uw[1][lane] = u4.y; ws->uw[2][lane] = u4.z; ws->uw[3][lane] = u4.w;
          __syncwarp();
          nphil += 32u;
          const uint32_t nf0 = nflip;
          handle_group(m, dg);
          if (nflip != nf0) {
            // item flips voided the certificates; slack flips only moved r -- the certificates
            // hold while 2r stays within the tolerance (checked before a certified block is skipped)
            if (fabsf(r2 - r2c) > a.rtol2) qmask = 0u;
            todo = allb & ~qmask & ~((16u << (4 * g)) - 1u);
          }
        }
      }
      // Frozen anneal: a sweep in which every spin was certified
      // saturated towards its current value changed nothing; fields stay constant and beta only
      // grows, so every later sweep of this anneal is certified the same way -- x_k is final.
#ifdef SAIM_PROF
      if (lane == 0) {
        const int pb = min(15, (int)(16LL * t / a.T));
        ws->prof[pb] += (uint32_t)(clock64() - prof_c0);
        ws->prof[16 + pb] += 1u;
        ws->prof[32 + pb] += nflip - prof_f0;
      }
#endif
      if (!active && freeze_exit && a.T >= 2) {
        cnt_add(ws, kCntSweeps, (uint32_t)(a.T - 1 - t));   // sweeps certified unchanged, not evaluated
        break;
      }
    }
    // ---- readout of x_k (Algorithm 1 "store feasible") ----
    int fpart = 0, load = 0;
#pragma unroll
    for (int m = 0; m < NPL; ++m) {
      if (((xm >> m) & 1u) && 32 * m + lane < n) {
        fpart += sC[32 * m + lane] - (int)(PK ? phi_pk(m) : phs[32 * m]);   // x_i (c_i - phi_i); phs = phi when x_i = 1
        load += (int)sAl[32 * m];
      }
    }
    const long long f = warp_sum_i64((long long)fpart) / 2;  // f = 1/2 sum_i x_i (c_i - phi_i)
    load = __reduce_add_sync(kFull, load);
    const bool feas = !has_con || (long long)load <= Hp->b0;
    uint32_t myword = 0;
    for (int b = 0; b < NB; ++b) {
      const uint32_t wb = __ballot_sync(kFull, (xm >> b) & 1u);
      if (lane == b) myword = wb;
    }
    const long long rl = (long long)(0.5f * r2);
    const long long Lam = ws->Lam;
    const size_t row = ((size_t)s * a.R + ridx) * a.K + k;
    if (lane == 0) {
      if (a.out.tr_f) a.out.tr_f[row] = f;
      if (a.out.tr_feas) a.out.tr_feas[row] = (uint8_t)feas;
      if (has_con && a.out.tr_r) a.out.tr_r[row] = rl;
      if (has_con && a.out.tr_lam) a.out.tr_lam[row] = Lam;
    }
    if (a.out.tr_x && lane < a.WN) a.out.tr_x[row * a.WN + lane] = myword;
    if (feas) {
      const bool better = f < ws->best_f;
      if (better) {
        const int rem = n - 32 * lane;
        ws->best_word[lane] = rem >= 32 ? myword : (rem > 0 ? (myword & ((1u << rem) - 1u)) : 0u);
      }
      __syncwarp();
      if (lane == 0) {
        ws->nfeas += 1;
        if (better) { ws->best_f = f; ws->best_k = k; }
      }
    }
    __syncwarp();
    if (lane == 0) {                                  // lambda_{k+1} = lambda_k + eta g(x_k)  (R10)
      const double Lnew = (double)(Lam + rl);
      ws->Lam = Lam + rl;
      ws->k3s = (float)(ws->bstep * (Hp->c_l * Lnew));
      ws->e1s = (float)(ws->bstep * ((Hp->c_p * Hp->v_bound + Hp->c_l * fabs(Lnew)) * 0x1p-20 +
                                     1.001 * Hp->c_p * (double)a.rtol2));
    }
    __syncwarp();
  }

  // ---- outputs ----
  const size_t ri = (size_t)s * a.R + ridx;
  const int rho = a.rep0 + ridx;
  // main kernel: a decision the fp64 level could not certify flags the replica for the exact
  // replay, which then supplies its outputs, its instance-best candidate and its counters
  // (SAIM_FLAG_TEST_REPLAY: every replica that reached the fp64 level at all)
  const bool defer = !RP && (ws->cnt[kCntUncert] != 0 || (ws->force_dd && ws->cnt[kCntFp64] != 0));
  if (lane == 0) {
    a.out.best_f[ri] = ws->best_f;
    a.out.best_k[ri] = ws->best_k;
    a.out.n_feasible[ri] = ws->nfeas;
    if (defer) {
      a.replay[replay_slot(threadIdx.x >> 5)] = 1;
      if (a.out.counters) atomicAdd(reinterpret_cast<unsigned long long *>(a.out.counters) + SAIM_CNT_REPLAYED, 1ull);
    }
    if (!defer && ws->best_k >= 0 && a.out.inst_best)
      atomicMin(reinterpret_cast<long long *>(a.out.inst_best) + s, (ws->best_f << 20) | (long long)rho);
    if (has_con && a.out.final_lam) a.out.final_lam[ri] = ws->Lam;
    if (a.out.rep_flips) a.out.rep_flips[ri] = nflip;
  }
  if (lane < a.Wn) a.out.best_x[ri * a.Wn + lane] = ws->best_word[lane];
  if (a.out.final_x) {
    uint32_t myword = 0;
    for (int b = 0; b < NB; ++b) {
      const uint32_t wb = __ballot_sync(kFull, (xm >> b) & 1u);
      if (lane == b) myword = wb;
    }
    if (lane < a.WN) a.out.final_x[ri * a.WN + lane] = myword;
  }
#ifdef SAIM_PROF
  if (lane == 0)
    for (int i = 0; i < 48; ++i) atomicAdd(&saim_prof[i], (unsigned long long)ws->prof[i]);
#endif
  if (lane == 0 && a.out.counters && !defer) {
    unsigned long long *c = reinterpret_cast<unsigned long long *>(a.out.counters);
    atomicAdd(c + SAIM_CNT_DECISIONS, (unsigned long long)a.K * a.T * N);
    atomicAdd(c + SAIM_CNT_FLIPS, (unsigned long long)nflip);
    atomicAdd(c + SAIM_CNT_UNIFORMS, (unsigned long long)ws->cnt[kCntUnif] + nunif);
    atomicAdd(c + SAIM_CNT_FP64, (unsigned long long)ws->cnt[kCntFp64]);
    atomicAdd(c + SAIM_CNT_UNCERTIFIED, (unsigned long long)ws->cnt[kCntUncert]);
    atomicAdd(c + SAIM_CNT_FEASIBLE, (unsigned long long)ws->nfeas);
    atomicAdd(c + SAIM_CNT_PHILOX, (unsigned long long)ws->cnt[kCntPhilox] + nphil);
    atomicAdd(c + SAIM_CNT_SWEEPS, (unsigned long long)a.K * a.T - ws->cnt[kCntSweeps]);
  }
}

}  // namespace saim
