/*
 * oracle/saim_oracle.c -- plain, slow, obviously-correct CPU SAIM (arXiv 2501.04971).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg may load, call or execute anything under oracle/.  It shares no code,
 * header, table or constant generator with paper_2501_04971_b200/ (the product path).
 *
 * What it computes (citations are /root/reference/PAPER.md line numbers, equations by label):
 *   - Problem (Eq. 2 "primal_problem"): min f(x) s.t. g(x) = 0, x in {0,1}^N,
 *     with f(x) = 1/2 x^T Q x + c^T x (QKP Eq. 12; MKP Eq. 14).
 *   - Slack bits: each inequality row k gets q_k = floor(log2(b_k)+1) binary slack
 *     variables with weights 1, 2, ..., 2^(q_k-1); g_k(x) = sum_j A_ext[k][j] x_j - b_k (equality form).
 *   - Normalisation: f is divided by s_o = max(|Q|,|c|), A and b by
 *     s_c = max(|A|,|b|) (scalar over the whole arrays, reading R9).
 *   - Lagrange function (Eq. 3 "penalty_energy" + Eq. 5 "Lagrange_energy"):
 *        L(x) = f(x)/s_o + P * sum_k (r_k/s_c)^2 + sum_k lambda_k r_k/s_c,  r = A_ext x - b.
 *   - Algorithm 1: lambda_0 = 0; for k = 1..K: minimise L_k with the p-bit IM,
 *     store feasible samples, lambda_{k+1} = lambda_k + eta * g(x_k) (g normalised: r/s_c).
 *     Because lambda_0 = 0 and g = r/s_c, lambda_k = (eta/s_c) * Lambda_k exactly, with the
 *     integer Lambda_k = sum_{k'<k} r(x_k') (reading R10).
 *   - p-bit IM (Eq. 9 "Ii_eq", Eq. 10 "mi_eq"): sequential Gibbs
 *     updates in ascending spin order, linear beta_t = beta_max * t/(T-1), read the last sample.
 *     In binary form (R1): x_i <- [u < sigma(beta * F_i)] with
 *        F_i = -(L(x with x_i=1) - L(x with x_i=0)) = phi_i/s_o - (P/s_c^2) pi_i - (eta/s_c^2) kappa_i
 *        phi_i = -(c_i + sum_j Q_ij x_j)        (items; 0 for slack bits)
 *        pi_i  = sum_k ((r0_k + A_ki)^2 - r0_k^2),  r0 = r - A_{.i} x_i
 *        kappa_i = sum_k Lambda_k A_ki
 *     u = (2*floor(w/2^9)+1) * 2^-24, w a Philox4x32-10 word keyed on (seed, inst, replica, k, t, i)
 *     (R2).  This equals Eq. 10 with rand(-1,1) = 1 - 2u.
 *   - Decisions are the EXACT real predicate u < sigma(z) (R18): evaluated in fp64 with a
 *     rigorous error bound, re-evaluated in __float128 when within the bound.  Ties are impossible.
 *   - Readout per k: feasible <=> A x_items <= b; f(x) = 1/2 x^T Q x + c^T x;
 *     best = first k with the smallest f among feasible samples (R13).
 *
 * Two field modes: FROM_DEFINITION recomputes phi, r, pi, kappa from x at every decision;
 * INCREMENTAL keeps phi and r up to date on flips (same integers, so identical decisions).
 *
 * Build: gcc -O2 -std=gnu11 -fPIC -shared -ffp-contract=off -pthread saim_oracle.c -lquadmath -lm
 */
#include <math.h>
#include <pthread.h>
#include <quadmath.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define ORC_FROM_DEFINITION 0
#define ORC_INCREMENTAL 1

typedef struct {
  int32_t n, M;            /* items, constraints */
  const int32_t *Q;        /* [n][n] row-major, symmetric, zero diagonal; NULL: no quadratic term */
  const int32_t *c;        /* [n] */
  const int32_t *A;        /* [M][n], entries >= 0 */
  const int64_t *b;        /* [M], >= 1 */
  double P, eta, beta_max; /* penalty, Lagrange step, final inverse temperature */
  int32_t inst;            /* instance index s (enters the RNG counter) */
} orc_problem;

typedef struct {
  uint64_t seed;
  int32_t rep0, nrep;      /* global replica indices rep0 .. rep0+nrep-1 */
  int32_t K, T;            /* Lagrange iterations, sweeps per anneal */
  int32_t field_mode;      /* ORC_FROM_DEFINITION | ORC_INCREMENTAL */
  int32_t nthreads;        /* worker threads (>=1) */
  const uint8_t *x_init;   /* [nrep][N] initial state, or NULL for all zeros */
} orc_run_args;

typedef struct {
  int64_t *best_f;         /* [nrep]; INT64_MAX when no feasible sample */
  uint32_t *best_x;        /* [nrep][ceil(n/32)] item bits of the best sample */
  int32_t *best_k;         /* [nrep]; -1 when none */
  int32_t *n_feasible;     /* [nrep] */
  int64_t *tr_f;           /* optional [nrep][K]: f(x_k) */
  uint8_t *tr_feas;        /* optional [nrep][K] */
  int64_t *tr_r;           /* optional [nrep][K][M]: r(x_k) = A_ext x_k - b */
  int64_t *tr_lam;         /* optional [nrep][K][M]: Lambda_k used during anneal k */
  uint32_t *tr_x;          /* optional [nrep][K][ceil(N/32)]: x_k incl. slack bits */
  uint32_t *final_x;       /* optional [nrep][ceil(N/32)] */
  int64_t *final_lam;      /* optional [nrep][M]: Lambda_K */
  uint64_t counters[8];    /* see ORC_CNT_* */
} orc_out;

enum { ORC_CNT_DECISIONS = 0, ORC_CNT_UNSATURATED = 1, ORC_CNT_FLIPS = 2, ORC_CNT_NEAR_TIES = 3,
       ORC_CNT_QUAD = 4, ORC_CNT_FEASIBLE = 5 };

/* ------------------------------------------------------------------------------------------ */
/* Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11), written from the published definition.    */
static void philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
  uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
  uint32_t k0 = key_in[0], k1 = key_in[1];
  for (int round = 0; round < 10; ++round) {
    if (round > 0) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
    uint64_t p0 = (uint64_t)0xD2511F53u * c0;
    uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

void orc_philox(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) { philox4x32_10(ctr, key, out); }

/* The uniform of decision (seed, s, rho, k, t, i) (R2):
 *   key = (lo32 seed, hi32 seed); ctr = (32*floor(i/128) + i%32, t, k, (s<<20)|rho);
 *   w = word floor(i/32) % 4;  u = (2*floor(w/2^9) + 1) * 2^-24  (odd numerator, never 1/2). */
double orc_uniform(uint64_t seed, int32_t s, int32_t rho, int32_t k, int32_t t, int32_t i) {
  uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  uint32_t ctr[4] = {(uint32_t)(32 * (i / 128) + (i % 32)), (uint32_t)t, (uint32_t)k,
                     ((uint32_t)s << 20) | (uint32_t)rho};
  uint32_t w[4];
  philox4x32_10(ctr, key, w);
  uint32_t word = w[(i / 32) % 4];
  return (double)(2u * (word >> 9) + 1u) * 0x1p-24;
}

/* ------------------------------------------------------------------------------------------ */
/* Compiled problem: slack extension and scales.                 */
typedef struct {
  const orc_problem *p;
  int n, M, N;
  int64_t *Aext;           /* [M][N] */
  int64_t s_o, s_c;
} compiled;

static int bit_length(int64_t v) { int q = 0; while (v > 0) { ++q; v >>= 1; } return q; }

static int compile_problem(const orc_problem *p, compiled *cp) {
  memset(cp, 0, sizeof(*cp));
  cp->p = p; cp->n = p->n; cp->M = p->M;
  int N = p->n;
  for (int k = 0; k < p->M; ++k) {
    if (p->b[k] < 1) return -1;
    N += bit_length(p->b[k]);                     /* q_k = floor(log2 b_k) + 1 */
  }
  cp->N = N;
  cp->Aext = (int64_t *)calloc((size_t)p->M * N, sizeof(int64_t));
  int col = p->n;
  for (int k = 0; k < p->M; ++k) {
    for (int j = 0; j < p->n; ++j) cp->Aext[(size_t)k * N + j] = p->A[(size_t)k * p->n + j];
    int q = bit_length(p->b[k]);
    for (int bit = 0; bit < q; ++bit) cp->Aext[(size_t)k * N + col++] = (int64_t)1 << bit;  /* 1,2,..,2^(q-1) */
  }
  int64_t so = 0, sc = 0;
  for (int i = 0; i < p->n; ++i) {
    if (llabs(p->c[i]) > so) so = llabs(p->c[i]);
    if (p->Q) for (int j = 0; j < p->n; ++j) if (llabs(p->Q[(size_t)i * p->n + j]) > so) so = llabs(p->Q[(size_t)i * p->n + j]);
  }
  for (int k = 0; k < p->M; ++k) {
    if (p->b[k] > sc) sc = p->b[k];
    for (int j = 0; j < p->n; ++j) if (p->A[(size_t)k * p->n + j] > sc) sc = p->A[(size_t)k * p->n + j];
  }
  if (so == 0) so = 1;                            /* all-zero objective: any positive scale */
  if (sc == 0) sc = 1;                            /* unconstrained (M = 0): g is empty */
  cp->s_o = so; cp->s_c = sc;
  return 0;
}

int orc_num_spins(const orc_problem *p) {
  int N = p->n;
  for (int k = 0; k < p->M; ++k) N += bit_length(p->b[k]);
  return N;
}

int orc_scales(const orc_problem *p, int64_t out[2]) {
  compiled cp;
  if (compile_problem(p, &cp)) return -1;
  out[0] = cp.s_o; out[1] = cp.s_c;
  free(cp.Aext);
  return 0;
}

/* ------------------------------------------------------------------------------------------ */
/* Field components from the definition (used by FROM_DEFINITION mode and exported for tests). */
static int64_t phi_def(const compiled *cp, const uint8_t *x, int i) {
  const orc_problem *p = cp->p;
  if (i >= cp->n) return 0;                        /* slack bits carry no objective */
  int64_t s = p->c[i];
  if (p->Q) for (int j = 0; j < cp->n; ++j) s += (int64_t)p->Q[(size_t)i * cp->n + j] * x[j];
  return -s;
}

static void residual_def(const compiled *cp, const uint8_t *x, int64_t *r) {
  for (int k = 0; k < cp->M; ++k) {
    int64_t s = -cp->p->b[k];
    for (int j = 0; j < cp->N; ++j) s += cp->Aext[(size_t)k * cp->N + j] * x[j];
    r[k] = s;
  }
}

/* pi_i = sum_k ((r0_k + A_ki)^2 - r0_k^2), kappa_i = sum_k Lambda_k A_ki (Eq. 3 and Eq. 5 differences). */
static void pen_lag(const compiled *cp, const int64_t *r, const int64_t *Lam, const uint8_t *x, int i,
                    __int128 *pi, __int128 *kappa) {
  __int128 ps = 0, ks = 0;
  for (int k = 0; k < cp->M; ++k) {
    __int128 a = cp->Aext[(size_t)k * cp->N + i];
    __int128 r0 = (__int128)r[k] - a * x[i];
    ps += (r0 + a) * (r0 + a) - r0 * r0;
    ks += (__int128)Lam[k] * a;
  }
  *pi = ps; *kappa = ks;
}

/* ------------------------------------------------------------------------------------------ */
/* Certified decision x_i <- [u < sigma(beta_t F_i)]  (Eq. 10 in binary form, R1, R18). */
typedef struct { uint64_t dec, unsat, flips, near, quad; } cnts;

static const double LN_2P24_M1 = 16.635532333438687;   /* ln(2^24 - 1): |z| above => saturated */

static int decide(const compiled *cp, double u, int t, int T, int64_t phi, __int128 pi, __int128 kappa,
                  cnts *cn) {
  const orc_problem *p = cp->p;
  cn->dec++;
  if (T >= 2 && t == 0) {                          /* beta_0 = 0: sigma(0) = 1/2 exactly */
    cn->unsat++;
    if (fabs(u - 0.5) < 0x1p-20) cn->near++;
    return u < 0.5;
  }
  double beta = (T >= 2) ? p->beta_max * (double)t / (double)(T - 1) : p->beta_max;
  double so = (double)cp->s_o, sc = (double)cp->s_c;
  double t1 = (double)phi / so;
  double t2 = (p->P / (sc * sc)) * (double)pi;
  double t3 = (p->eta / (sc * sc)) * (double)kappa;
  double F = t1 - t2 - t3;
  double z = beta * F;
  double sig = 1.0 / (1.0 + exp(-z));
  double S = beta * (fabs(t1) + fabs(t2) + fabs(t3));
  double bound = (S + 4.0) * 0x1p-48;              /* >> the few-ulp fp64 error of z and sigma */
  if (fabs(z) <= LN_2P24_M1) cn->unsat++;
  if (fabs(u - sig) < 0x1p-20) cn->near++;
  if (fabs(u - sig) > bound) return u < sig;
  /* Re-evaluate in binary128 from the exact inputs. */
  cn->quad++;
  __float128 bq = (T >= 2) ? (__float128)p->beta_max * (__float128)t / (__float128)(T - 1)
                           : (__float128)p->beta_max;
  __float128 soq = (__float128)cp->s_o, scq = (__float128)cp->s_c;
  __float128 q1 = (__float128)phi / soq;
  __float128 q2 = ((__float128)p->P / (scq * scq)) * (__float128)pi;
  __float128 q3 = ((__float128)p->eta / (scq * scq)) * (__float128)kappa;
  __float128 zq = bq * (q1 - q2 - q3);
  __float128 sq = 1.0Q / (1.0Q + expq(-zq));
  __float128 Sq = bq * (fabsq(q1) + fabsq(q2) + fabsq(q3));
  __float128 bnd = (Sq + 4.0Q) * 0x1p-100Q;
  __float128 uq = (__float128)u;
  if (fabsq(uq - sq) > bnd) return uq < sq;
  fprintf(stderr, "saim_oracle: undecidable near-tie (u=%.17g); aborting\n", u);
  abort();
}

/* Exported for tests: the decision for given exact components (counts discarded). */
int orc_decide(const orc_problem *p, double u, int t, int T, int64_t phi, int64_t pi, int64_t kappa) {
  compiled cp;
  if (compile_problem(p, &cp)) return -1;
  cnts cn = {0};
  int d = decide(&cp, u, t, T, phi, pi, kappa, &cn);
  free(cp.Aext);
  return d;
}

/* Exported for tests: field components of spin i at state x (length N) and Lambda (length M),
 * from the definition.  out_int = {phi, pi, kappa}; returns F in fp64 via *F. */
int orc_field(const orc_problem *p, const uint8_t *x, const int64_t *Lam, int i, int64_t out_int[3], double *F) {
  compiled cp;
  if (compile_problem(p, &cp)) return -1;
  int64_t *r = (int64_t *)calloc(cp.M ? cp.M : 1, sizeof(int64_t));
  residual_def(&cp, x, r);
  __int128 pi, kappa;
  int64_t phi = phi_def(&cp, x, i);
  pen_lag(&cp, r, Lam, x, i, &pi, &kappa);
  out_int[0] = phi; out_int[1] = (int64_t)pi; out_int[2] = (int64_t)kappa;
  double sc = (double)cp.s_c;
  *F = (double)phi / (double)cp.s_o - (p->P / (sc * sc)) * (double)pi - (p->eta / (sc * sc)) * (double)kappa;
  free(r); free(cp.Aext);
  return 0;
}

/* f(x) = 1/2 x^T Q x + c^T x over the items (Eq. 12/14), exact integer. */
static int64_t objective(const compiled *cp, const uint8_t *x) {
  const orc_problem *p = cp->p;
  int64_t f = 0;
  for (int i = 0; i < cp->n; ++i) {
    if (!x[i]) continue;
    f += p->c[i];
    if (p->Q) for (int j = i + 1; j < cp->n; ++j) if (x[j]) f += p->Q[(size_t)i * cp->n + j];
  }
  return f;
}

/* Feasibility on the items against the original inequality (R12). */
static int feasible(const compiled *cp, const uint8_t *x) {
  for (int k = 0; k < cp->M; ++k) {
    int64_t s = 0;
    for (int j = 0; j < cp->n; ++j) s += (int64_t)cp->p->A[(size_t)k * cp->n + j] * x[j];
    if (s > cp->p->b[k]) return 0;
  }
  return 1;
}

/* Exported for tests: f(x), feasibility and r(x) of a full state x (length N). */
int orc_readout(const orc_problem *p, const uint8_t *x, int64_t *f, int32_t *feas, int64_t *r) {
  compiled cp;
  if (compile_problem(p, &cp)) return -1;
  *f = objective(&cp, x);
  *feas = feasible(&cp, x);
  residual_def(&cp, x, r);
  free(cp.Aext);
  return 0;
}

/* ------------------------------------------------------------------------------------------ */
/* One replica: Algorithm 1 around the annealed p-bit sampler. */
typedef struct {
  const compiled *cp;
  const orc_run_args *a;
  orc_out *o;
  int next;               /* shared work counter */
  pthread_mutex_t mu;
  cnts total;
  uint64_t n_feas_total;
} job;

static void run_replica(const compiled *cp, const orc_run_args *a, orc_out *o, int ridx, cnts *cn,
                        uint64_t *nfeas_total) {
  const orc_problem *p = cp->p;
  const int n = cp->n, M = cp->M, N = cp->N, K = a->K, T = a->T;
  const int rho = a->rep0 + ridx;
  const int Wn = (n + 31) / 32, WN = (N + 31) / 32;
  uint8_t *x = (uint8_t *)calloc(N, 1);
  int64_t *phi = (int64_t *)calloc(N, sizeof(int64_t));
  int64_t *r = (int64_t *)calloc(M ? M : 1, sizeof(int64_t));
  int64_t *Lam = (int64_t *)calloc(M ? M : 1, sizeof(int64_t));   /* Lambda_0 = 0  (lambda_0 = 0) */
  if (a->x_init) memcpy(x, a->x_init + (size_t)ridx * N, N);
  for (int i = 0; i < N; ++i) phi[i] = phi_def(cp, x, i);
  residual_def(cp, x, r);

  int64_t best_f = INT64_MAX; int best_k = -1; int nfeas = 0;
  uint8_t *best_x = (uint8_t *)calloc(n ? n : 1, 1);

  for (int k = 0; k < K; ++k) {
    /* --- minimise L_k with the p-bit IM: T sweeps, linear beta ramp, last sample --- */
    for (int t = 0; t < T; ++t) {
      for (int i = 0; i < N; ++i) {
        int64_t ph;
        __int128 pi, kap;
        if (a->field_mode == ORC_FROM_DEFINITION) {
          ph = phi_def(cp, x, i);
          residual_def(cp, x, r);
        } else {
          ph = phi[i];
        }
        pen_lag(cp, r, Lam, x, i, &pi, &kap);
        double u = orc_uniform(a->seed, p->inst, rho, k, t, i);
        int xn = decide(cp, u, t, T, ph, pi, kap, cn);
        if (xn != x[i]) {
          int delta = xn - x[i];
          x[i] = (uint8_t)xn;
          cn->flips++;
          if (a->field_mode == ORC_INCREMENTAL) {
            if (i < n && p->Q) for (int j = 0; j < n; ++j) phi[j] -= (int64_t)delta * p->Q[(size_t)j * n + i];
            for (int m = 0; m < M; ++m) r[m] += (int64_t)delta * cp->Aext[(size_t)m * N + i];
          }
        }
      }
    }
    if (a->field_mode == ORC_FROM_DEFINITION) residual_def(cp, x, r);
    /* --- store feasible x_k --- */
    int feas = feasible(cp, x);
    int64_t f = objective(cp, x);
    if (feas) {
      nfeas++;
      if (f < best_f) { best_f = f; best_k = k; memcpy(best_x, x, n); }
    }
    if (o->tr_f) o->tr_f[(size_t)ridx * K + k] = f;
    if (o->tr_feas) o->tr_feas[(size_t)ridx * K + k] = (uint8_t)feas;
    for (int m = 0; m < M; ++m) {
      if (o->tr_r) o->tr_r[((size_t)ridx * K + k) * M + m] = r[m];
      if (o->tr_lam) o->tr_lam[((size_t)ridx * K + k) * M + m] = Lam[m];
    }
    if (o->tr_x) {
      uint32_t *w = o->tr_x + ((size_t)ridx * K + k) * WN;
      memset(w, 0, sizeof(uint32_t) * WN);
      for (int i = 0; i < N; ++i) if (x[i]) w[i / 32] |= 1u << (i % 32);
    }
    /* --- update lambda_{k+1} = lambda_k + eta g(x_k)  <=>  Lambda += r (R10) --- */
    for (int m = 0; m < M; ++m) Lam[m] += r[m];
  }
  o->best_f[ridx] = best_f;
  o->best_k[ridx] = best_k;
  o->n_feasible[ridx] = nfeas;
  uint32_t *bw = o->best_x + (size_t)ridx * Wn;
  memset(bw, 0, sizeof(uint32_t) * Wn);
  if (best_k >= 0) for (int i = 0; i < n; ++i) if (best_x[i]) bw[i / 32] |= 1u << (i % 32);
  if (o->final_x) {
    uint32_t *w = o->final_x + (size_t)ridx * WN;
    memset(w, 0, sizeof(uint32_t) * WN);
    for (int i = 0; i < N; ++i) if (x[i]) w[i / 32] |= 1u << (i % 32);
  }
  if (o->final_lam) for (int m = 0; m < M; ++m) o->final_lam[(size_t)ridx * M + m] = Lam[m];
  *nfeas_total += (uint64_t)nfeas;
  free(x); free(phi); free(r); free(Lam); free(best_x);
}

static void *worker(void *arg) {
  job *jb = (job *)arg;
  cnts local = {0};
  uint64_t nf = 0;
  for (;;) {
    pthread_mutex_lock(&jb->mu);
    int ridx = jb->next++;
    pthread_mutex_unlock(&jb->mu);
    if (ridx >= jb->a->nrep) break;
    run_replica(jb->cp, jb->a, jb->o, ridx, &local, &nf);
  }
  pthread_mutex_lock(&jb->mu);
  jb->total.dec += local.dec; jb->total.unsat += local.unsat; jb->total.flips += local.flips;
  jb->total.near += local.near; jb->total.quad += local.quad; jb->n_feas_total += nf;
  pthread_mutex_unlock(&jb->mu);
  return NULL;
}

/* Run replicas rep0..rep0+nrep-1 of one instance.  Returns 0, or -1 on invalid input. */
int orc_run(const orc_problem *p, const orc_run_args *a, orc_out *o) {
  if (p->n < 1 || p->M < 0 || a->nrep < 0 || a->K < 0 || a->T < 1) return -1;
  if (a->rep0 < 0 || a->rep0 + a->nrep > (1 << 20) || p->inst < 0 || p->inst >= (1 << 12)) return -1;
  compiled cp;
  if (compile_problem(p, &cp)) return -1;
  job jb;
  memset(&jb, 0, sizeof(jb));
  jb.cp = &cp; jb.a = a; jb.o = o;
  pthread_mutex_init(&jb.mu, NULL);
  int nt = a->nthreads < 1 ? 1 : a->nthreads;
  if (nt > a->nrep) nt = a->nrep > 0 ? a->nrep : 1;
  pthread_t *th = (pthread_t *)calloc(nt, sizeof(pthread_t));
  for (int w = 0; w < nt; ++w) pthread_create(&th[w], NULL, worker, &jb);
  for (int w = 0; w < nt; ++w) pthread_join(th[w], NULL);
  free(th);
  pthread_mutex_destroy(&jb.mu);
  memset(o->counters, 0, sizeof(o->counters));
  o->counters[ORC_CNT_DECISIONS] = jb.total.dec;
  o->counters[ORC_CNT_UNSATURATED] = jb.total.unsat;
  o->counters[ORC_CNT_FLIPS] = jb.total.flips;
  o->counters[ORC_CNT_NEAR_TIES] = jb.total.near;
  o->counters[ORC_CNT_QUAD] = jb.total.quad;
  o->counters[ORC_CNT_FEASIBLE] = jb.n_feas_total;
  free(cp.Aext);
  return 0;
}
