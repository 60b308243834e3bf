// saim_layout.h -- device data layout of a compiled SAIM problem (host <-> kernel contract).
//
// HBM holds, per instance s, one contiguous 16-byte aligned "blob" that the kernel's prologue
// stages into shared memory with a single TMA bulk copy (cp.async.bulk):
//
//   QKP kernel (M <= 1, quadratic objective):
//     [Q rows, lane-major]   n rows x QW words x 32 lanes x 4 B.  Word w of lane l in row j packs
//                            the entries Q[j][32*(E*w+e) + l] (e = 0..E-1, E = 4/qbytes) as
//                            unsigned (Q + 2^(8*qbytes-1)); entries of non-existent items are the
//                            code of 0.  A flip of item j streams one row: lane l reads QW words.
//     [A_ext]                float[NB*32]: item weights, then slack weights 1,2,..,2^(q-1), then 0.
//     [c]                    int32[NPL*32]: objective linear term per item, 0 beyond n.
//   MKP kernel (linear objective, M <= 32):
//     [Acol]                 int16 x M x n_pad (item columns A[.][i]), stored [i][M] so one spin's
//                            column is contiguous.
//     [c]                    int32[n_pad]
//     [slack]                per slack spin: (row, shift)
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
};

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
  double beta_max;
  saim_outputs out;           // device pointers
};

}  // namespace saim
