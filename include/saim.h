/*
 * saim.h -- C ABI of libsaim, the B200 (sm_100a) hot path of the Self-Adaptive Ising Machine
 * (SAIM, arXiv 2501.04971).  Citations: PAPER.md = /root/reference/PAPER.md line numbers,
 * DESIGN.md readings R1..R25 (the paper-gap ledger).
 *
 * What one saim_run computes, per instance s and replica rho (independent chains, R22):
 *   Algorithm 1: Lambda_0 = 0; for k = 0..K-1:
 *     x_k  <- T sweeps of sequential p-bit Gibbs updates (Eq. 9-10) of
 *             L_k(x) = f(x)/s_o + P*||r/s_c||^2 + (eta/s_c^2) Lambda_k . r     (Eq. 3 + Eq. 5)
 *             with r = A_ext x - b (slack bits appended), s_o, s_c the
 *             normalisation scales, beta_t = beta_max*t/(T-1) (R3), spins in
 *             ascending order (R4), state carried across anneals (R5), last sample read (R6);
 *     store x_k if A x_items <= b (R12), keep the smallest f (first k on ties, R13);
 *     Lambda_{k+1} = Lambda_k + r(x_k)    (<=> lambda_{k+1} = lambda_k + eta*g(x_k), PAPER.md:114;
 *                                          lambda_k = (eta/s_c) Lambda_k exactly, R10)
 *   Every decision x_i <- [u < sigma(beta_t F_i)] is the EXACT real predicate (R1, R18) with u the
 *   Philox4x32-10 uniform keyed on (seed, s, rho, k, t, i) (R2); the kernel certifies each
 *   decision (fp32 fast path with a rigorous error bound, fp64 second level, double-double third
 *   level on the exact integers) and counts any decision not certified even in double-double
 *   (SAIM_CNT_UNCERTIFIED; its band is ~2^-80 wide, so the count is 0 in practice).
 *
 * Conventions: all functions return 0 (SAIM_OK) or a negative SAIM_E* code; saim_last_error()
 * returns a thread-local message for the last failure.  No function aborts the process.
 */
#ifndef SAIM_H_
#define SAIM_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SAIM_OK 0
#define SAIM_EINVAL (-1)      /* malformed shapes/values (asymmetric Q, nonzero diagonal, A<0, b<1, NaN, ...) */
#define SAIM_ERANGE (-2)      /* integer state would leave the exactly-representable range (DESIGN.md App. B) */
#define SAIM_ESMEM (-3)       /* instance does not fit shared-memory residency on sm_100a */
#define SAIM_ECUDA (-4)       /* CUDA runtime error (incl. an earlier asynchronous kernel fault) */
#define SAIM_EUNSUPPORTED (-5)/* problem class without a kernel (quadratic objective with M > 1) */
#define SAIM_ENOMEM (-6)

/* Counters (uint64[SAIM_NUM_COUNTERS]) accumulated by saim_run over all replicas. */
#define SAIM_CNT_DECISIONS 0     /* attempted p-bit updates = n_inst*R*K*T*N */
#define SAIM_CNT_FLIPS 1         /* decisions that changed x_i (identical to the oracle's count) */
#define SAIM_CNT_SWEEPS 2        /* sweeps actually evaluated (the rest were certified frozen, see flags) */
#define SAIM_CNT_UNIFORMS 3      /* decisions the kernel could not settle without u (not certified saturated) */
#define SAIM_CNT_FP64 4          /* decisions re-evaluated on the fp64 slow path */
#define SAIM_CNT_UNCERTIFIED 5   /* decisions not certified even in double-double (expected 0) */
#define SAIM_CNT_FEASIBLE 6      /* feasible samples x_k */
#define SAIM_CNT_PHILOX 7        /* Philox4x32-10 evaluations (per lane) */
#define SAIM_CNT_REPLAYED 8      /* QKP: replicas re-run by the exact replay (a decision its fp64 level
                                  * could not certify; DESIGN.md 6.1 "Exact replay"); their counts
                                  * above are those of the replay */
#define SAIM_NUM_COUNTERS 9

/* Problem batch: n_inst instances sharing (n_items, n_cons).  HOST pointers; copied by
 * saim_create (the caller may free them on return).  Row-major, instance-major. */
typedef struct {
  int32_t n_inst;          /* >= 1, < 4096 (RNG counter field, R2) */
  int32_t n_items;         /* n >= 1 */
  int32_t n_cons;          /* M >= 0 */
  const int32_t *Q;        /* [n_inst][n][n] symmetric, zero diagonal; NULL => linear objective (MKP) */
  const int32_t *c;        /* [n_inst][n]      f(x) = 1/2 x^T Q x + c^T x (minimised; QKP: Q=-W, c=-h) */
  const int32_t *A;        /* [n_inst][M][n]   constraint weights, >= 0 */
  const int64_t *b;        /* [n_inst][M]      capacities, >= 1 (A x_items <= b) */
} saim_problem;

typedef struct {
  const double *P;         /* [n_inst] penalty P >= 0 of Eq. 3 (PAPER.md:102 P = alpha d N; chosen by the caller;
                            * P = 0 drops the quadratic penalty, leaving the Lagrange term alone).
                            * Finite; SAIM_EINVAL otherwise */
  double eta;              /* Lagrange step eta >= 0 (Algorithm 1); eta = 0 is the penalty-method baseline */
  double beta_max;         /* final inverse temperature of the linear ramp, > 0 */
  int32_t device;          /* CUDA device ordinal */
  int32_t flags;           /* SAIM_FLAG_* */
} saim_params;

/* saim_params.flags.  By default an anneal stops evaluating sweeps once a whole sweep was
 * certified frozen (every spin saturated towards its current value): the fields are then
 * constant and beta_t only grows, so all later sweeps of that anneal provably change nothing
 * (DESIGN.md "Exact early exit").  Results are bit-identical either way. */
#define SAIM_FLAG_NO_FREEZE_EXIT 1
/* Kernel selection for linear objectives with M >= 2 constraints (MKP).  Default: the
 * speculative sub-warp kernel with G = 8 lanes per replica for M <= 8 (SAIM_FLAG_MKP_SPEC8 below;
 * the outcome tree with L = 2 if it does not fit shared memory), the lane-per-replica lockstep
 * kernel for M > 8 (the faster one on B200 for each).  These flags force the lockstep kernel,
 * the outcome tree with a given L, or the row-split kernel (each replica's constraint rows over
 * 2 lanes; honoured for M > 8 only).  At most one kernel-selection flag may be set.  All give
 * identical results. */
#define SAIM_FLAG_MKP_LOCKSTEP 2
#define SAIM_FLAG_MKP_L2 4
#define SAIM_FLAG_MKP_L4 8
#define SAIM_FLAG_MKP_SPLIT2 16
/* QKP kernel: disable the hot-block loop (sweeps in which a single uncertified block flips nothing
 * run back to back without the general block machinery).  Results are identical either way. */
#define SAIM_FLAG_QKP_NO_HOT_LOOP 32
/* MKP lockstep kernel: no producer warps (each consumer warp draws its own logits).  Identical
 * results either way. */
#define SAIM_FLAG_MKP_NO_PRODUCER 64
/* Test hook for the certification chain: every decision that reaches the fp64 level is treated as
 * uncertified there, so it is re-decided at the double-double level (MKP: at once; QKP: by the
 * exact replay of the whole replica).  Results are identical either way; only slower. */
#define SAIM_FLAG_TEST_REPLAY 128
/* MKP, M <= 8: the speculative sub-warp kernel with G = 2, 4, 8, 16 or 32 lanes per replica (the
 * lanes hold the replica's next G spins that are not final; the first flipping lane of a round is
 * applied and the later lanes are re-evaluated: DESIGN.md 6.5).  Kernel-selection flags (at most
 * one of these and the four above).  SAIM_ESMEM if M > 8 or the tables do not fit.  Identical
 * results. */
#define SAIM_FLAG_MKP_SPEC2 1024
#define SAIM_FLAG_MKP_SPEC4 256
#define SAIM_FLAG_MKP_SPEC8 512
#define SAIM_FLAG_MKP_SPEC16 2048
#define SAIM_FLAG_MKP_SPEC32 4096

/* Outputs of saim_run: CALLER-OWNED DEVICE pointers (e.g. torch CUDA tensors), written
 * asynchronously on the run's stream.  R = replicas per instance, Wn = ceil(n/32),
 * WN = ceil(N_max/32) (saim_info.words_full).  Optional pointers may be NULL. */
typedef struct {
  int64_t *best_f;         /* [n_inst][R]  smallest feasible f, INT64_MAX if none */
  uint32_t *best_x;        /* [n_inst][R][Wn] item bits of that sample (bit i%32 of word i/32) */
  int32_t *best_k;         /* [n_inst][R]  iteration of the best sample, -1 if none */
  int32_t *n_feasible;     /* [n_inst][R]  feasible samples among the K */
  int64_t *inst_best;      /* [n_inst]     min over replicas, packed (f << 20) | rho; INT64_MAX if none */
  uint64_t *counters;      /* [SAIM_NUM_COUNTERS] (zeroed by saim_run) */
  /* optional trace (trace rows), each [n_inst][R][K]... */
  int64_t *tr_f;           /* [n_inst][R][K]      f(x_k) */
  uint8_t *tr_feas;        /* [n_inst][R][K]      feasibility flag */
  int64_t *tr_r;           /* [n_inst][R][K][M]   r(x_k) = A_ext x_k - b */
  int64_t *tr_lam;         /* [n_inst][R][K][M]   Lambda_k (lambda_k = eta/s_c * Lambda_k) */
  uint32_t *tr_x;          /* [n_inst][R][K][WN]  full sample x_k incl. slack bits */
  uint32_t *final_x;       /* [n_inst][R][WN]     state after the last sweep */
  int64_t *final_lam;      /* [n_inst][R][M]      Lambda_K */
  uint32_t *rep_flips;     /* [n_inst][R]         spin flips of each replica's chain over the whole run
                            * (incl. the beta = 0 sweeps): a fingerprint of the full trajectory, not
                            * only of the K readouts (the oracle counts the same) */
} saim_outputs;

typedef struct {
  int32_t n_inst, n_items, n_cons;
  int32_t n_spins_max;     /* max over instances of N = n + sum_k q_k */
  int32_t words_items;     /* Wn = ceil(n/32) */
  int32_t words_full;      /* WN = ceil(N_max/32) */
  int32_t kernel;          /* 1 = QKP warp-per-replica kernel (M <= 1), 2 = MKP kernels (lanes_per_replica: 1 lockstep,
                            * 2/4 outcome tree or row split, 2..32 speculative sub-warp) */
  int32_t smem_bytes;      /* dynamic shared memory per CTA */
  int32_t q_bytes;         /* bytes per stored Q entry (1 or 2), 0 if no Q */
  int32_t lanes_per_replica;
  int32_t phi_packed;      /* QKP: 1 if phi is held as biased int16 pairs (int8 Q and |phi| <= 32767
                            * in every state, host-proven), 0 = fp32 phi */
} saim_info;

typedef struct saim_ctx saim_ctx;

/* Validate and compile a problem batch (slack extension PAPER.md:162, scales PAPER.md:170,
 * integer-range proofs, device layout) and upload it to `par->device`.  Synchronous.
 * On success *out owns all device memory.  Errors: SAIM_EINVAL, SAIM_ERANGE, SAIM_ESMEM,
 * SAIM_EUNSUPPORTED, SAIM_ECUDA, SAIM_ENOMEM. */
int saim_create(const saim_problem *prob, const saim_params *par, saim_ctx **out);

/* Run R replicas per instance of K Lagrange iterations of T sweeps, with uniforms keyed on
 * `seed` and GLOBAL replica indices rep0 .. rep0+R-1 (so replica ranges may be split across
 * calls or GPUs with bit-identical results).  Asynchronous on `cuda_stream` (a cudaStream_t,
 * e.g. torch.cuda.current_stream().cuda_stream; NULL = legacy default stream).  Launch and
 * argument errors return synchronously; kernel faults surface at the next stream sync or call
 * (SAIM_ECUDA).  Requires 1 <= R, rep0 + R <= 2^20, K >= 1, T >= 1, K * max|r| < 2^62 (int64
 * Lambda) and K * max|r| * max A_ext * M < 2^62 (int64 kappa on the slow path); SAIM_ERANGE
 * otherwise. */
int saim_run(saim_ctx *ctx, uint64_t seed, int32_t rep0, int32_t R, int32_t K, int32_t T,
             void *cuda_stream, const saim_outputs *out);

/* Fill *out with the compiled shape; per-instance values via saim_get_instance. */
int saim_get_info(const saim_ctx *ctx, saim_info *out);

/* Per-instance compiled scalars: N (spins), s_o, s_c, and the slack bit count of each row
 * (q[] of length n_cons, may be NULL). */
int saim_get_instance(const saim_ctx *ctx, int32_t inst, int32_t *N, int64_t *s_o, int64_t *s_c, int32_t *q);

/* Free all device memory of ctx; NULL-safe. */
void saim_destroy(saim_ctx *ctx);

/* Self-tests of device primitives (synchronous; device `device`):
 *  which = 0: device Philox4x32-10 on n (ctr[4], key[2]) inputs; in_u32 = host uint32[n][6],
 *             out_u32 = host uint32[n][4].
 *  which = 1: exhaustive sweep of the fp32 logit used by the fast path over all 2^23 uniforms
 *             (R18); out_f64[0] = max |logit_f32(u) - logit(u)| / (2^-17 + 2^-19 |logit(u)|)
 *             (must be < 1 for the certification bound to hold), out_f64[1] = max abs error.
 *  which = 2: the double-double decision level (R18) on n records; in_u32 points to n
 *             80-byte records {int64 phi, pi, kappa, s_o, s_c; double P, eta, beta_max; int32 tn,
 *             td; uint32 w; int32 pad} (beta_t = beta_max tn/td, u from the Philox word w as in R2);
 *             out_u32[i] = x | (uncertified << 1) for record i.
 *  which = 3: the fp64 slow path's logit table (one per device, built by saim_create): for n Philox
 *             words in_u32, out_f64[2i] = the table entry the slow path reads, out_f64[2i+1] =
 *             ln(u) - ln(1 - u) computed directly on the device (must be identical). */
int saim_selftest(int which, int device, int n, const uint32_t *in_u32, uint32_t *out_u32, double *out_f64);

/* Thread-local message of the last failing call ("" if none). */
const char *saim_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* SAIM_H_ */
