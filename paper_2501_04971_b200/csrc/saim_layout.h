// saim_layout.h -- device data layout of a compiled SAIM problem (host <-> kernel contract).
//
// HBM holds, per instance s, one contiguous 16-byte aligned "blob" that the kernel's prologue
// stages into shared memory with a single TMA bulk copy (cp.async.bulk):
//
//   QKP kernel (M <= 1, quadratic objective):
//     [A_ext]                float[NBP*32]: item weights, then slack weights 1,2,..,2^(q-1), then
//                            NaN (no spin).
//     [c]                    int32[NPL*32]: objective linear term per item, 0 beyond n.
//     [Q rows, lane-major]   n rows x QW words x 32 lanes x 4 B.  Word w of lane l in row j packs
//                            the entries Q[j][32*(E*w+e) + l] (e = 0..E-1, E = 4/qbytes) as
//                            unsigned (Q + 2^(8*qbytes-1)); entries of non-existent items are the
//                            code of 0.  A flip of item j streams one row: lane l reads QW words.
//     (A_ext and c first: their sizes depend only on the kernel's (NPL, QB) instantiation, so all
//     three arrays sit at compile-time offsets from one base.)
//   MKP kernels (linear objective, 2 <= M <= 32): see MkpLayout below -- fp32 item columns
//     (exact integers), per-item constants, c, b, the slack bit count of each row and the O(3n)
//     band of adjacent column products.  Slack spins have no stored column: slack bit q of row
//     m has the single weight 2^q in row m, derived from qrow in the kernel.
//
// All integer state of the hot path stays exactly representable: the host proves the bounds of
// DESIGN.md Appendix B before accepting a problem (SAIM_ERANGE otherwise).
#pragma once
#include <cstdint>

#include "../../include/saim.h"

namespace saim {

// Per-instance compiled scalars (array in HBM, read once per warp).
struct InstHdr {
  int32_t N;        // spins incl. slack
  int32_t n_slack;  // sum_k q_k
  int64_t b0;       // capacity of row 0 (QKP kernel)
  double c_o;       // 1 / s_o            (objective scale)
  double c_p;       // P / s_c^2          (Eq. 3 penalty, normalised)
  double c_l;       // eta / s_c^2        (Eq. 5 with lambda = eta/s_c * Lambda, R10)
  int64_t s_o, s_c;
  int32_t slack_off;  // MKP: offset of this instance's slack table (entries), unused by QKP
  int32_t pad;
  double phi_bound;   // max_i |c_i| + sum_j |Q_ij|  >= |phi_i| for every state (host-proven)
  double v_bound;     // 2 max|r| + max A_ext      >= |2 r0 + A_i| for every state
  double r_bound;     // max|r_k| over every state and row (host-proven)
  double P, eta, beta_max;  // the run constants exactly as given (double-double slow path, R18)
  const double *logit_tab;  // logit((2m+1) 2^-24) for m < 2^23 (fp64 slow path; one table per device)
};

inline __host__ __device__ uint32_t align16u(uint32_t v) { return (v + 15u) & ~15u; }

// MKP blob (per instance), MM = padded constraint count (4, 8, 16 or 32):
//   acol   float [n][MM]   item columns A[.][i], zero-padded rows m >= M
//   iconst float4[n]       (c_o*phi_i = -c_o c_i, c_p a_i with a_i = sum_m A_mi^2, |A_i|_1, E0_i)
//   cint   int32 [n]       c_i (exact objective for the readout)
//   brow   int64 [MM]      b_m
//   qrow   int32 [MM]      slack bit count q_m (0 for padded rows)
//   band   float [3][n+1]  G_d[i] = A_{.i} . A_{.i-d}, d = 1..3 (0 where i < d): the O(3n) band of
//                          nearby item-column products used by the lookahead / outcome trees --
//                          not the dense A^T A
struct MkpLayout {
  uint32_t acol, iconst, cint, brow, qrow, band, bytes;
};
inline __host__ __device__ MkpLayout mkp_layout(int n, int MM) {
  MkpLayout L;
  uint32_t o = 0;
  L.acol = o;   o += align16u((uint32_t)(n + 1) * MM * 4u);     // + one zero column (lookahead past n-1)
  L.iconst = o; o += (uint32_t)n * 16u;
  L.cint = o;   o += align16u((uint32_t)n * 4u);
  L.brow = o;   o += (uint32_t)MM * 8u;
  L.qrow = o;   o += align16u((uint32_t)MM * 4u);
  L.band = o;   o += 3u * align16u((uint32_t)(n + 1) * 4u);
  L.bytes = o;
  return L;
}
inline __host__ __device__ uint32_t mkp_band_stride(int n) { return align16u((uint32_t)(n + 1) * 4u) / 4u; }
// Per-warp MKP shared memory (lockstep kernel): x bits [WN][32 lanes], logits of the current
// 128-spin group [128][32] floats, Lambda [MM][32] int64.
// With producer warps (prod = 1): two logit buffers [2][128][32] (groups alternate by parity) and
// the consumer/producer mbarriers full[2], empty[2] after Lambda.  Last: r [MM][32] and c_l Lambda
// [MM][32] floats, the per-lane copies the row-interleaved slack phase indexes by row.
inline __host__ __device__ uint32_t mkp_warp_bytes(int WN, int MM, int prod = 0) {
  return align16u((uint32_t)WN * 128u) + (prod ? 2u : 1u) * 128u * 128u + (uint32_t)MM * 256u + (prod ? 32u : 0u) +
         2u * (uint32_t)MM * 128u;
}
// Per-warp shared memory of the row-split kernel with S lanes per replica (G = 32/S replicas):
// x bits [WN][G] words, logits of the current 128-spin group [128][G] floats, Lambda of each
// lane's MM/S rows [MM/S][32 lanes] int64.
inline __host__ __device__ uint32_t mkps_warp_bytes(int WN, int S, int MM) {
  const uint32_t G = 32u / (uint32_t)S;
  return align16u((uint32_t)WN * G * 4u) + 128u * G * 4u + (uint32_t)(MM / S) * 256u;
}
// Per-warp shared memory of the outcome-tree kernel with L lanes per replica (G = 32/L replica
// groups): x bits [WN][G] words, logits of the current 128-spin group [128][G] floats, Lambda
// [MM][G] int64.
inline __host__ __device__ uint32_t mkpt_warp_bytes(int WN, int L, int MM) {
  const uint32_t G = 32u / (uint32_t)L;
  return align16u((uint32_t)WN * G * 4u) + 128u * G * 4u + (uint32_t)MM * G * 8u;
}

// Speculative sub-warp MKP kernel (saim_mkp_spec.cuh, G lanes per chain): after the blob, the spin
// table of all NS = 32 WN spins, one row of MM + 4 floats per spin (column A_{.i}, then c_p a_i,
// -c_o c_i, |A_i|_1, E0_i); then per chain: x words [WN], Lambda [MM] int64, and one float4 per spin
// (T_i = -c_o c_i - A_i . c_l Lambda and the error slope of this iteration; logit and logit
// tolerance of the chain's current sweep).
inline __host__ __device__ uint32_t mkpx_table_bytes(int WN, int MM) {
  return (uint32_t)WN * 32u * ((uint32_t)MM * 4u + 16u);
}
inline __host__ __device__ uint32_t mkpx_chain_bytes(int WN, int MM) {
  return align16u((uint32_t)WN * 4u) + (uint32_t)MM * 8u + (uint32_t)WN * 32u * 16u;
}
inline __host__ __device__ uint32_t mkpx_warp_bytes(int WN, int G, int MM) {
  return (32u / (uint32_t)G) * mkpx_chain_bytes(WN, MM);
}

struct RunArgs {
  const unsigned char *blob;  // [n_inst][blob_bytes]
  const InstHdr *hdr;         // [n_inst]
  uint32_t blob_bytes;        // per instance, multiple of 16
  uint32_t a_off, c_off, x_off;  // byte offsets inside the blob (Q at 0 for QKP)
  int32_t n, M;               // items, constraints
  int32_t Wn, WN;             // ceil(n/32), ceil(N_max/32)
  int32_t R, rep0, K, T;
  int32_t flags;              // saim_params.flags
  uint64_t seed;
  uint32_t ks[20];            // Philox key schedule of seed (saim_dev.cuh philox4x32_10_ks)
  double beta_max;
  int32_t mkp_prod;           // MKP lockstep: 1 = producer warps draw the logits
  float rtol2;                // QKP: 2D, a quiet certificate holds while |2r - 2r_cert| <= 2D
  uint8_t *replay;            // [n_inst][grid.x][32] warp slots flagged for the exact replay (zeroed per run)
  saim_outputs out;           // device pointers
};

}  // namespace saim
