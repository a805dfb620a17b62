/*
 * fmo.h -- CPU ORACLE for the fast MaxEnt sampler (arXiv 2509.13230).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load this library.  The product path
 * (paper_2509_13230_b200/) never includes, links or calls anything in oracle/.
 * It shares no code, header, table or constant generator with the CUDA path.
 *
 * Citations: P:Ln = /root/reference/PAPER.md line n (section / equation / Alg. 1).
 * The contract (readings of the paper where it is silent or ambiguous) is
 * DESIGN.md section 3; every reading used here is named there.
 *
 * All floating point is IEEE binary64, one operation at a time in the written
 * order (compiled with -ffp-contract=off); transcendental functions are libm's
 * log() and log1p().
 */
#ifndef FMO_H
#define FMO_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { FMO_UBCM = 0, FMO_ECM = 1 };
enum { FMO_UNDIRECTED = 0, FMO_BIPARTITE = 1, FMO_DIRECTED = 2 };
enum { FMO_OK = 0, FMO_ERR_INVALID = -1, FMO_ERR_NOMEM = -2, FMO_ERR_STATE = -5 };
enum { FMO_FLAG_WEIGHT_SATURATED = 1u };

typedef struct fmo_plan fmo_plan;
typedef struct fmo_result fmo_result;

/* Philox4x32-10 (Salmon et al., SC'11), the RNG of contract reading R1. */
void fmo_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
/* u01(k) = (k + 0.5) * 2^-32, reading R2. */
double fmo_u01(uint32_t k);
/* floor(-log(u01(k)) / h) as int64, or -1 when the quotient is >= 2^62 or not finite (skip law). */
int64_t fmo_skip(uint32_t k, double h);

/* a1-a4: validate, key, sort, suffix max, plan; undirected. */
int fmo_plan_create(int model, int64_t n, const double *x, const double *y, int64_t seg_target,
                    fmo_plan **out);
/* bipartite (+ set rows x1,y1 against - set candidates x2,y2) and directed (out-fitness x1,y1,
 * in-fitness x2,y2, n1 == n2, no self loops) plans; kind FMO_UNDIRECTED ignores set 2 */
int fmo_plan_create2(int model, int kind, int64_t n1, const double *x1, const double *y1, int64_t n2,
                     const double *x2, const double *y2, int64_t seg_target, fmo_plan **out);
void fmo_plan_free(fmo_plan *p);
int64_t fmo_plan_nc(const fmo_plan *p);
void fmo_plan_export_cand(const fmo_plan *p, int32_t *cperm, double *ckappa, double *cy, double *cly,
                          int32_t *excl);
int64_t fmo_plan_n(const fmo_plan *p);
int64_t fmo_plan_nseg(const fmo_plan *p);
int fmo_plan_F(const fmo_plan *p);
/* copies of the plan arrays; any pointer may be NULL */
void fmo_plan_export(const fmo_plan *p, int32_t *perm, double *kappa_s, double *y_s, double *ymax,
                     uint64_t *P, int32_t *seg_u, int32_t *seg_a, int32_t *seg_b, int32_t *seg_sigma,
                     double *seg_h0, double *seg_x0, double *seg_d0, double *seg_omT, double *seg_iomT,
                     double *ly_s);

/* a5-a6: sample.  rows == NULL -> every row; otherwise only the listed sorted-rank rows
 * (ascending, for spot checks at full size).  Edges of each sample are in canonical order
 * (row u, segment sigma, draw order); orientation (min id, max id). */
int fmo_sample(const fmo_plan *p, uint64_t seed, int64_t first_sample, int64_t n_samples,
               const int32_t *rows, int64_t n_rows, int nthreads, fmo_result **out);
/* with options: FMO_SAMPLE_BETA_REFRESH (ECM: per-candidate beta_min refresh, DESIGN R17) */
enum { FMO_SAMPLE_BETA_REFRESH = 1u };
int fmo_sample_ex(const fmo_plan *p, uint64_t seed, int64_t first_sample, int64_t n_samples,
                  const int32_t *rows, int64_t n_rows, int nthreads, uint32_t flags, fmo_result **out);

/* Level-1 oracle: the plain definition, O(N^2) independent Bernoulli trials per pair with
 * an unrelated RNG (xoshiro256**), weights by sequential Bernoulli trials (Eq. 3-5). */
int fmo_bruteforce(int model, int64_t n, const double *x, const double *y, uint64_t seed,
                   int64_t n_samples, fmo_result **out);
int fmo_bruteforce2(int model, int kind, int64_t n1, const double *x1, const double *y1, int64_t n2,
                    const double *x2, const double *y2, uint64_t seed, int64_t n_samples, fmo_result **out);
void fmo_expected2(int model, int kind, int64_t n1, const double *x1, const double *y1, int64_t n2,
                   const double *x2, const double *y2, double *kout, double *kout_var, double *kin,
                   double *kin_var);

int64_t fmo_result_n_samples(const fmo_result *r);
int64_t fmo_result_n_edges(const fmo_result *r);
void fmo_result_export(const fmo_result *r, int64_t *offsets, int32_t *edges, int32_t *weights,
                       int64_t counters[3], uint32_t *flags);
void fmo_result_free(fmo_result *r);

/* Closed forms: for each listed node i (nodes == NULL -> all), over j != i:
 *   k[i] = sum p_ij, kvar[i] = sum p_ij (1 - p_ij)                          (Eq. 4)
 *   s[i] = sum p_ij/(1-t_ij), svar[i] = sum Var[w_ij]  (ECM only)        (Eq. 3-5)
 * p from the plain definition in fitness form: UBCM X/(1+X), X = x_i x_j;
 * ECM z/(1 - t + z), z = x_i x_j y_i y_j, t = y_i y_j.  s/svar may be NULL for UBCM. */
void fmo_expected(int model, int64_t n, const double *x, const double *y, const int32_t *nodes,
                  int64_t n_nodes, int nthreads, double *k, double *kvar, double *s, double *svar);
/* rich club: e_top[m] = edges among the first m nodes of `order` (rank -> id), m = 0..n;
 * and its expectation / variance under the model (independent pairs) */
void fmo_richclub_count(int64_t n, const int32_t *order, int64_t n_edges, const int32_t *edges, int64_t *e_top);
void fmo_expected_richclub(int model, int64_t n, const double *x, const double *y, const int32_t *order,
                           double *mean, double *var);
/* sum_{i<j} p_ij exactly, O(N^2), threaded */
double fmo_expected_edges(int model, int64_t n, const double *x, const double *y, int nthreads);

#ifdef __cplusplus
}
#endif
#endif
