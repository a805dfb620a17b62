/*
 * fmo.c -- CPU ORACLE for the fast MaxEnt sampler of arXiv 2509.13230
 *          ("Fast unbiased sampling of networks with given expected degrees and strengths").
 *
 * TEST INFRASTRUCTURE ONLY -- see fmo.h.  Plain, slow, obviously-correct C following the
 * paper's algorithm step by step.  No code is shared with the CUDA path.
 *
 * Notation (paper -> here):  alpha_i, beta_i enter only through the fitness
 * variables x_i = exp(-alpha_i), y_i = exp(-beta_i) (BASELINE.json north_star).  In sorted
 * rank space the focal node is i (paper's i), the candidate j (paper's j), the proposal
 * probability q, the true probability p.
 *
 * Build: gcc -O2 -std=c11 -ffp-contract=off -fno-fast-math -fPIC -shared -pthread -lm
 */
#define _GNU_SOURCE
#include "fmo.h"

#include <float.h>
#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

#define FMO_G 16 /* work units: one expected draw = 2^G */

/* ------------------------------------------------------------------------------------------ */
/* Philox4x32-10 (reading R1).  Round function of Salmon, Moraes, Dror, Shaw, "Parallel random  */
/* numbers: as easy as 1, 2, 3" (SC'11): multipliers 0xD2511F53, 0xCD9E8D57, Weyl key bumps    */
/* 0x9E3779B9, 0xBB67AE85, ten rounds.                                                          */
/* ------------------------------------------------------------------------------------------ */
void fmo_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4])
{
    uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
    uint32_t k0 = key[0], k1 = key[1];
    for (int round = 0; round < 10; round++) {
        uint64_t prod0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
        uint64_t prod1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
        uint32_t hi0 = (uint32_t)(prod0 >> 32), lo0 = (uint32_t)prod0;
        uint32_t hi1 = (uint32_t)(prod1 >> 32), lo1 = (uint32_t)prod1;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        uint32_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* Reading R2: a 32-bit word k maps to the open-interval uniform (k + 0.5) * 2^-32 (exact). */
double fmo_u01(uint32_t k) { return ((double)k + 0.5) * 0x1p-32; }

/* Geometric skip (P:L110 caption "q(1-q)^{L-1}", "(1-p)^L p"; reading R4):
 * number of skipped candidates = floor(E / h), E = -log U, h = -log(1 - q). */
int64_t fmo_skip(uint32_t k, double h)
{
    double E = -log(fmo_u01(k));
    double R = E / h;
    if (!(R < 0x1p62)) return -1;
    return (int64_t)floor(R);
}

/* ------------------------------------------------------------------------------------------ */
/* Plan                                                                                         */
/* ------------------------------------------------------------------------------------------ */
struct fmo_plan {
    int model;
    int kind;         /* FMO_UNDIRECTED, FMO_BIPARTITE, FMO_DIRECTED            */
    int64_t n, nc, S; /* n rows (the + set / out-nodes), nc candidates (the - set / in-nodes)   */
    int F;
    /* rows, in rank order of their own sort (P:L133 (i)) */
    int32_t *perm;    /* perm[r] = original id of sorted rank r                          */
    double *kappa_s;  /* sort key in rank order: x (UBCM) or x*y (ECM)                   */
    double *y_s;      /* ECM: y in rank order                                            */
    double *ly_s;     /* ECM: log(y) in rank order (weights, reading R8)                 */
    /* candidates (undirected: the same arrays as the rows) */
    int32_t *cperm;
    double *ckappa, *cy, *cly;
    double *ymax;     /* ECM: ymax[t] = max_{w>=t} cy[w], ymax[nc] = 0 (beta_min, R6)    */
    uint64_t *P;      /* fixed-point prefix of ckappa, nc+1 entries (planner, 3.4)       */
    int32_t *excl;    /* directed: excl[u] = candidate rank of row u's own node (no self loops) */
    int64_t *row_seg; /* first segment of each row, n+1 entries                          */
    int64_t nseg;
    int32_t *seg_u, *seg_a, *seg_b, *seg_sigma;
    double *seg_h0, *seg_x0, *seg_d0, *seg_omT, *seg_iomT;
};

typedef struct {
    double kappa;
    int32_t id;
} key_t_;

/* Sort order of P:L133 step (i) "ascending order of alpha_i" = descending x, and Alg. 1 line 3
 * "increasing alpha_i + beta_i" = descending x*y; ties by ascending id (reading R9).
 * The comparator is a total order, so qsort's result is unique. */
static int cmp_key(const void *pa, const void *pb)
{
    const key_t_ *a = (const key_t_ *)pa, *b = (const key_t_ *)pb;
    if (a->kappa > b->kappa) return -1;
    if (a->kappa < b->kappa) return 1;
    return (a->id < b->id) ? -1 : (a->id > b->id);
}

static int ceil_log2_i64(int64_t n)
{
    int L = 0;
    while (((int64_t)1 << L) < n) L++;
    return L;
}

/* first candidate of row u: undirected j > i, bipartite/directed every - node */
static int64_t row_c0(const fmo_plan *p, int64_t u) { return p->kind == FMO_UNDIRECTED ? u + 1 : 0; }

/* W_u(v): integer estimate (units 2^-G draws) of the draws a row-u chain makes over candidates
 * [c0, v); saturated part counts 1 per candidate, the rest r_u * sum kappa. */
static int64_t plan_W(const fmo_plan *p, int64_t c0, double r, int64_t sat, int64_t v)
{
    int64_t vs = v < sat ? v : sat;
    int64_t A = (vs - c0) * ((int64_t)1 << FMO_G);
    int64_t B = 0;
    if (v > sat) {
        uint64_t D = p->P[v] - p->P[sat];
        B = (int64_t)floor(ldexp(r * (double)D, FMO_G - p->F));
    }
    return A + B;
}

void fmo_plan_free(fmo_plan *p)
{
    if (!p) return;
    if (p->cperm != p->perm) { free(p->cperm); free(p->ckappa); free(p->cy); free(p->cly); }
    free(p->perm); free(p->kappa_s); free(p->y_s); free(p->ly_s); free(p->ymax); free(p->P); free(p->excl);
    free(p->row_seg);
    free(p->seg_u); free(p->seg_a); free(p->seg_b); free(p->seg_sigma);
    free(p->seg_h0); free(p->seg_x0); free(p->seg_d0); free(p->seg_omT); free(p->seg_iomT);
    free(p);
}

/* a1 + a2 for one node set: validate, key, sort; returns the rank-order arrays */
static int sort_set(int model, int64_t n, const double *x, const double *y, int32_t **perm, double **kappa_s,
                    double **y_s, double **ly_s, double *kmax_out)
{
    for (int64_t i = 0; i < n; i++) {
        if (!isfinite(x[i]) || x[i] < 0.0) return FMO_ERR_INVALID;
        if (model == FMO_ECM && (!isfinite(y[i]) || y[i] < 0.0 || y[i] >= 1.0)) return FMO_ERR_INVALID;
    }
    key_t_ *keys = (key_t_ *)malloc(sizeof(key_t_) * (size_t)n);
    if (!keys) return FMO_ERR_NOMEM;
    double kmax = 0.0;
    for (int64_t i = 0; i < n; i++) {
        keys[i].kappa = (model == FMO_UBCM) ? x[i] : x[i] * y[i];
        keys[i].id = (int32_t)i;
        if (keys[i].kappa > kmax) kmax = keys[i].kappa;
    }
    if (!isfinite((kmax * kmax) * (kmax * kmax))) { free(keys); return FMO_ERR_INVALID; } /* R10 products */
    qsort(keys, (size_t)n, sizeof(key_t_), cmp_key);
    *perm = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
    *kappa_s = (double *)malloc(sizeof(double) * (size_t)n);
    if (model == FMO_ECM) {
        *y_s = (double *)malloc(sizeof(double) * (size_t)n);
        *ly_s = (double *)malloc(sizeof(double) * (size_t)n);
    }
    if (!*perm || !*kappa_s || (model == FMO_ECM && (!*y_s || !*ly_s))) { free(keys); return FMO_ERR_NOMEM; }
    for (int64_t r = 0; r < n; r++) { (*perm)[r] = keys[r].id; (*kappa_s)[r] = keys[r].kappa; }
    if (model == FMO_ECM)
        for (int64_t r = 0; r < n; r++) { (*y_s)[r] = y[(*perm)[r]]; (*ly_s)[r] = log((*y_s)[r]); }
    free(keys);
    *kmax_out = kmax;
    return FMO_OK;
}

int fmo_plan_create2(int model, int kind, int64_t n1, const double *x1, const double *y1, int64_t n2,
                     const double *x2, const double *y2, int64_t seg_target, fmo_plan **out)
{
    *out = NULL;
    /* ---- a1: validate ---- */
    if (model != FMO_UBCM && model != FMO_ECM) return FMO_ERR_INVALID;
    if (kind != FMO_UNDIRECTED && kind != FMO_BIPARTITE && kind != FMO_DIRECTED) return FMO_ERR_INVALID;
    if (kind == FMO_UNDIRECTED) { n2 = n1; x2 = x1; y2 = y1; }
    if (kind == FMO_DIRECTED && n1 != n2) return FMO_ERR_INVALID;
    if (n1 < (kind == FMO_UNDIRECTED ? 2 : 1) || n1 > INT32_MAX || !x1) return FMO_ERR_INVALID;
    if (n2 < 1 || n2 > INT32_MAX || !x2) return FMO_ERR_INVALID;
    if (model == FMO_ECM && (!y1 || !y2)) return FMO_ERR_INVALID;
    if (seg_target == 0) seg_target = 256;
    if (seg_target < 8 || seg_target > ((int64_t)1 << 40)) return FMO_ERR_INVALID;

    fmo_plan *p = (fmo_plan *)calloc(1, sizeof(fmo_plan));
    if (!p) return FMO_ERR_NOMEM;
    p->model = model; p->kind = kind; p->n = n1; p->nc = n2; p->S = seg_target;
    const int64_t n = n1, nc = n2;
    /* ---- a2: sort both sets (P:L133 (i); "sorted according to ...") ---- */
    double kmax1 = 0.0, kmax2 = 0.0;
    int rc = sort_set(model, n1, x1, y1, &p->perm, &p->kappa_s, &p->y_s, &p->ly_s, &kmax1);
    if (rc != FMO_OK) { fmo_plan_free(p); return rc; }
    if (kind == FMO_UNDIRECTED) {
        p->cperm = p->perm; p->ckappa = p->kappa_s; p->cy = p->y_s; p->cly = p->ly_s; kmax2 = kmax1;
    } else {
        rc = sort_set(model, n2, x2, y2, &p->cperm, &p->ckappa, &p->cy, &p->cly, &kmax2);
        if (rc != FMO_OK) { fmo_plan_free(p); return rc; }
    }
    /* R10's cross products (X * D with X <= kmax1 * kmax2) stay finite: implied by each set's
     * kmax^4 being finite (checked in sort_set) */
    (void)kmax1; (void)kmax2;
    if (kind == FMO_DIRECTED) { /* the row node's own in-copy is not a candidate */
        int32_t *crank = (int32_t *)malloc(sizeof(int32_t) * (size_t)nc);
        p->excl = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
        if (!crank || !p->excl) { free(crank); fmo_plan_free(p); return FMO_ERR_NOMEM; }
        for (int64_t r = 0; r < nc; r++) crank[p->cperm[r]] = (int32_t)r;
        for (int64_t u = 0; u < n; u++) p->excl[u] = crank[p->perm[u]];
        free(crank);
    }

    /* ---- a3: beta_min via suffix maximum of the candidates' y (R6) ---- */
    if (model == FMO_ECM) {
        p->ymax = (double *)malloc(sizeof(double) * (size_t)(nc + 1));
        if (!p->ymax) goto nomem;
        p->ymax[nc] = 0.0;
        for (int64_t t = nc - 1; t >= 0; t--) p->ymax[t] = fmax(p->cy[t], p->ymax[t + 1]);
    }

    /* ---- a4: planner (not in the paper -- validity from the memoryless skip,
     *      P:L117-124, which lets a row restart with a fresh bound at any candidate) ---- */
    {
        int e = 0;
        if (p->ckappa[0] > 0.0) frexp(p->ckappa[0], &e);
        p->F = 61 - e - ceil_log2_i64(nc);
        p->P = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)(nc + 1));
        p->row_seg = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n + 1));
        if (!p->P || !p->row_seg) goto nomem;
        p->P[0] = 0;
        for (int64_t v = 0; v < nc; v++)
            p->P[v + 1] = p->P[v] + (uint64_t)floor(ldexp(p->ckappa[v], p->F));
    }
    /* pass 1: segment counts per row */
    const int64_t unit = (int64_t)1 << FMO_G;
    int64_t *m = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
    double *rr = (double *)malloc(sizeof(double) * (size_t)n);
    int64_t *sat = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
    int64_t *wtot = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
    if (!m || !rr || !sat || !wtot) { free(m); free(rr); free(sat); free(wtot); goto nomem; }
    int64_t nseg = 0;
    for (int64_t i = 0; i < n; i++) {
        p->row_seg[i] = nseg;
        const int64_t c0 = row_c0(p, i);
        if (c0 >= nc) { m[i] = 0; continue; } /* no candidates (the last undirected row), no draws */
        double r = p->kappa_s[i];
        if (model == FMO_ECM) r = p->kappa_s[i] / (1.0 - p->y_s[i] * p->ymax[c0]);
        int64_t s = c0; /* smallest v in [c0, nc] with v == nc or r*ckappa[v] < 1 (linear scan) */
        while (s < nc && !(r * p->ckappa[s] < 1.0)) s++;
        int64_t Wt = plan_W(p, c0, r, s, nc) + unit;
        int64_t mi = (Wt + seg_target * unit - 1) / (seg_target * unit);
        rr[i] = r; sat[i] = s; wtot[i] = Wt; m[i] = mi;
        nseg += mi;
    }
    p->row_seg[n] = nseg;
    p->nseg = nseg;
    p->seg_u = (int32_t *)malloc(sizeof(int32_t) * (size_t)(nseg + 1));
    p->seg_a = (int32_t *)malloc(sizeof(int32_t) * (size_t)(nseg + 1));
    p->seg_b = (int32_t *)malloc(sizeof(int32_t) * (size_t)(nseg + 1));
    p->seg_sigma = (int32_t *)malloc(sizeof(int32_t) * (size_t)(nseg + 1));
    p->seg_h0 = (double *)malloc(sizeof(double) * (size_t)(nseg + 1));
    p->seg_x0 = (double *)malloc(sizeof(double) * (size_t)(nseg + 1));
    p->seg_d0 = (double *)malloc(sizeof(double) * (size_t)(nseg + 1));
    p->seg_omT = (double *)malloc(sizeof(double) * (size_t)(nseg + 1));
    p->seg_iomT = (double *)malloc(sizeof(double) * (size_t)(nseg + 1));
    if (!p->seg_u || !p->seg_a || !p->seg_b || !p->seg_sigma || !p->seg_h0 || !p->seg_x0 || !p->seg_d0 ||
        !p->seg_omT || !p->seg_iomT) {
        free(m); free(rr); free(sat); free(wtot); goto nomem;
    }
    /* pass 2: cuts and segments */
    int bad = 0;
    for (int64_t i = 0; i < n && !bad; i++) {
        const int64_t g0 = p->row_seg[i], mi = m[i], c0 = row_c0(p, i);
        int64_t prev = c0;
        for (int64_t k = 0; k < mi; k++) {
            int64_t a = prev, b;
            if (k == mi - 1) {
                b = nc;
            } else {
                /* cut k+1: smallest v in [c0+1, nc-1] with W(v) >= floor((k+1) Wtot / m) */
                int64_t theta = (int64_t)(((__int128)(k + 1) * (__int128)wtot[i]) / (__int128)mi);
                int64_t lo = c0 + 1, hi = nc - 1; /* answer in [lo, hi]; hi if none */
                while (lo < hi) {
                    int64_t mid = lo + (hi - lo) / 2;
                    if (plan_W(p, c0, rr[i], sat[i], mid) >= theta) hi = mid; else lo = mid + 1;
                }
                b = lo;
                if (!(b > a) || !(b < nc)) { bad = 1; break; } /* cannot happen for S >= 8 */
            }
            int64_t g = g0 + k;
            p->seg_u[g] = (int32_t)i; p->seg_a[g] = (int32_t)a; p->seg_b[g] = (int32_t)b;
            p->seg_sigma[g] = (int32_t)k;
            prev = b;
        }
    }
    free(m); free(rr); free(sat); free(wtot);
    if (bad) { fmo_plan_free(p); return FMO_ERR_STATE; }
    /* initial bound of every segment at the virtual previous position a-1 (reading R3; the first
     * candidate itself when a = 0 in the bipartite case), kept as numerator x0 and denominator d0
     * of q = x0/d0 (reading R10):
     * UBCM q = X/(1+X), X = kappa_i kappa_{a-1}; -log(1-q) = log1p(X)
     * ECM  q = z/(1-T+z), z = kappa_i kappa_{a-1}, T = y_i ymax[a]; -log(1-q) = log1p(z/(1-T)),
     *      with z/(1-T) evaluated as z * RN(1/(1-T)) */
    for (int64_t g = 0; g < nseg; g++) {
        int64_t i = p->seg_u[g], a = p->seg_a[g];
        int64_t bp = a > 0 ? a - 1 : 0;
        double kq = p->kappa_s[i] * p->ckappa[bp];
        p->seg_x0[g] = kq;
        if (model == FMO_UBCM) {
            p->seg_omT[g] = 1.0;
            p->seg_iomT[g] = 1.0;
            p->seg_d0[g] = 1.0 + kq;
            p->seg_h0[g] = log1p(kq);
        } else {
            double T = p->y_s[i] * p->ymax[a];
            double omT = 1.0 - T;
            double iomT = 1.0 / omT;
            p->seg_omT[g] = omT;
            p->seg_iomT[g] = iomT;
            p->seg_d0[g] = omT + kq;
            p->seg_h0[g] = log1p(kq * iomT);
        }
    }
    *out = p;
    return FMO_OK;
nomem:
    fmo_plan_free(p);
    return FMO_ERR_NOMEM;
}

int fmo_plan_create(int model, int64_t n, const double *x, const double *y, int64_t seg_target,
                    fmo_plan **out)
{
    return fmo_plan_create2(model, FMO_UNDIRECTED, n, x, y, n, x, y, seg_target, out);
}

int64_t fmo_plan_n(const fmo_plan *p) { return p->n; }
int64_t fmo_plan_nc(const fmo_plan *p) { return p->nc; }
int64_t fmo_plan_nseg(const fmo_plan *p) { return p->nseg; }
int fmo_plan_F(const fmo_plan *p) { return p->F; }

void fmo_plan_export(const fmo_plan *p, int32_t *perm, double *kappa_s, double *y_s, double *ymax,
                     uint64_t *P, int32_t *seg_u, int32_t *seg_a, int32_t *seg_b, int32_t *seg_sigma,
                     double *seg_h0, double *seg_x0, double *seg_d0, double *seg_omT, double *seg_iomT,
                     double *ly_s)
{
    size_t n = (size_t)p->n, nc = (size_t)p->nc, s = (size_t)p->nseg;
    if (perm) memcpy(perm, p->perm, n * sizeof(int32_t));
    if (kappa_s) memcpy(kappa_s, p->kappa_s, n * sizeof(double));
    if (y_s && p->y_s) memcpy(y_s, p->y_s, n * sizeof(double));
    if (ymax && p->ymax) memcpy(ymax, p->ymax, (nc + 1) * sizeof(double));
    if (P) memcpy(P, p->P, (nc + 1) * sizeof(uint64_t));
    if (seg_u) memcpy(seg_u, p->seg_u, s * sizeof(int32_t));
    if (seg_a) memcpy(seg_a, p->seg_a, s * sizeof(int32_t));
    if (seg_b) memcpy(seg_b, p->seg_b, s * sizeof(int32_t));
    if (seg_sigma) memcpy(seg_sigma, p->seg_sigma, s * sizeof(int32_t));
    if (seg_h0) memcpy(seg_h0, p->seg_h0, s * sizeof(double));
    if (seg_x0) memcpy(seg_x0, p->seg_x0, s * sizeof(double));
    if (seg_d0) memcpy(seg_d0, p->seg_d0, s * sizeof(double));
    if (seg_omT) memcpy(seg_omT, p->seg_omT, s * sizeof(double));
    if (seg_iomT) memcpy(seg_iomT, p->seg_iomT, s * sizeof(double));
    if (ly_s && p->ly_s) memcpy(ly_s, p->ly_s, n * sizeof(double));
}

void fmo_plan_export_cand(const fmo_plan *p, int32_t *cperm, double *ckappa, double *cy, double *cly,
                          int32_t *excl)
{
    size_t nc = (size_t)p->nc, n = (size_t)p->n;
    if (cperm) memcpy(cperm, p->cperm, nc * sizeof(int32_t));
    if (ckappa) memcpy(ckappa, p->ckappa, nc * sizeof(double));
    if (cy && p->cy) memcpy(cy, p->cy, nc * sizeof(double));
    if (cly && p->cly) memcpy(cly, p->cly, nc * sizeof(double));
    if (excl) {
        if (p->excl) memcpy(excl, p->excl, n * sizeof(int32_t));
        else for (size_t u = 0; u < n; u++) excl[u] = -1;
    }
}

/* ------------------------------------------------------------------------------------------ */
/* Result buffers                                                                               */
/* ------------------------------------------------------------------------------------------ */
struct fmo_result {
    int64_t n_samples, n_edges;
    int64_t *offsets;
    int32_t *edges;
    int32_t *weights;
    int64_t draws, landed, accepted;
    uint32_t flags;
};

typedef struct {
    int32_t *e, *w;
    int64_t n, cap;
    int64_t draws, landed, accepted;
    uint32_t flags;
    int err;
} buf_t;

/* undirected pairs are stored as (min id, max id); bipartite (+ id, - id) and directed (out, in)
 * pairs as they are (ordered != 0) */
static void buf_push(buf_t *b, int32_t s, int32_t d, int32_t w, int ordered)
{
    if (b->err) return;
    if (b->n == b->cap) {
        int64_t nc = b->cap ? 2 * b->cap : 1024;
        int32_t *ne = (int32_t *)realloc(b->e, sizeof(int32_t) * 2 * (size_t)nc);
        if (!ne) { b->err = FMO_ERR_NOMEM; return; }
        b->e = ne;
        int32_t *nw = (int32_t *)realloc(b->w, sizeof(int32_t) * (size_t)nc);
        if (!nw) { b->err = FMO_ERR_NOMEM; return; }
        b->w = nw;
        b->cap = nc;
    }
    b->e[2 * b->n] = (ordered || s < d) ? s : d;
    b->e[2 * b->n + 1] = (ordered || s < d) ? d : s;
    b->w[b->n] = w;
    b->n++;
}

static int result_alloc(fmo_result **out, int64_t n_samples, int64_t n_edges, int weighted)
{
    fmo_result *r = (fmo_result *)calloc(1, sizeof(fmo_result));
    if (!r) return FMO_ERR_NOMEM;
    r->n_samples = n_samples;
    r->n_edges = n_edges;
    r->offsets = (int64_t *)calloc((size_t)n_samples + 1, sizeof(int64_t));
    r->edges = (int32_t *)malloc(sizeof(int32_t) * 2 * (size_t)(n_edges + 1));
    r->weights = weighted ? (int32_t *)malloc(sizeof(int32_t) * (size_t)(n_edges + 1)) : NULL;
    if (!r->offsets || !r->edges || (weighted && !r->weights)) { fmo_result_free(r); return FMO_ERR_NOMEM; }
    *out = r;
    return FMO_OK;
}

int64_t fmo_result_n_samples(const fmo_result *r) { return r->n_samples; }
int64_t fmo_result_n_edges(const fmo_result *r) { return r->n_edges; }
void fmo_result_export(const fmo_result *r, int64_t *offsets, int32_t *edges, int32_t *weights,
                       int64_t counters[3], uint32_t *flags)
{
    if (offsets) memcpy(offsets, r->offsets, sizeof(int64_t) * (size_t)(r->n_samples + 1));
    if (edges) memcpy(edges, r->edges, sizeof(int32_t) * 2 * (size_t)r->n_edges);
    if (weights && r->weights) memcpy(weights, r->weights, sizeof(int32_t) * (size_t)r->n_edges);
    if (counters) { counters[0] = r->draws; counters[1] = r->landed; counters[2] = r->accepted; }
    if (flags) *flags = r->flags;
}
void fmo_result_free(fmo_result *r)
{
    if (!r) return;
    free(r->offsets); free(r->edges); free(r->weights); free(r);
}

/* ------------------------------------------------------------------------------------------ */
/* a5: the chain of one segment (P:L133-136 steps (ii)-(iv); Alg. 1 P:L152-162 as corrected  */
/* by readings R3-R8).  Segment g covers candidates [a, b) of focal row i.                     */
/* ------------------------------------------------------------------------------------------ */
static void chain_ubcm(const fmo_plan *p, const uint32_t key[2], uint32_t s_abs, int64_t g, buf_t *out)
{
    const int64_t i = p->seg_u[g], b = p->seg_b[g];
    const uint32_t sigma = (uint32_t)p->seg_sigma[g];
    const double kappa_i = p->kappa_s[i];
    int64_t j = p->seg_a[g] - 1;  /* last evaluated position (virtual a-1 at the start; -1 at a
                                   * bipartite row start: the bound is then the first candidate) */
    double xq = p->seg_x0[g];     /* proposal q = xq / dq >= p_ij for every remaining j       */
    double dq = p->seg_d0[g];
    double h = p->seg_h0[g];      /* h = -log(1 - q)                                          */
    const int32_t id_i = p->perm[i];
    const int ordered = p->kind != FMO_UNDIRECTED;
    const int64_t excl = p->excl ? p->excl[i] : -1; /* directed: no self loop */
    for (uint32_t d = 0;; d++) {
        uint32_t ctr[4] = {d >> 1, sigma, (uint32_t)i, s_abs}, W[4];
        fmo_philox4x32_10(ctr, key, W);
        uint32_t w_skip = W[2 * (d & 1)], w_acc = W[2 * (d & 1) + 1];
        out->draws++;
        /* skip L ~ Geometric(q): L - 1 = floor(-log U / -log(1-q)) */
        double E = -log(fmo_u01(w_skip));
        double R = E / h;
        if (!(R < (double)(b - 1 - j))) break; /* end of candidate list (R5) */
        j = j + 1 + (int64_t)floor(R);
        out->landed++;
        if (j == excl) continue; /* p = 0: never accepted, q unchanged (still a valid bound) */
        /* p_ij = x_i x_j / (1 + x_i x_j)  (P:L92 with x = e^-alpha), as X / D */
        double X = kappa_i * p->ckappa[j];
        double D = 1.0 + X;
        if (X * dq > xq * D * (1.0 + 0x1p-50)) out->err = FMO_ERR_STATE; /* contract p <= q */
        /* accept with probability p/q: u < (X/D) / (xq/dq), cross-multiplied (R10) */
        if ((fmo_u01(w_acc) * xq) * D < X * dq) {
            out->accepted++;
            buf_push(out, id_i, p->cperm[j], 1, ordered);
        }
        /* q <- p_ij; -log(1 - q) = log1p(X) */
        xq = X;
        dq = D;
        h = log1p(X);
    }
}

/* refresh != 0 (DESIGN R17): after each reached candidate j the bound for the rest
 * of the segment uses beta_min over the candidates still ahead, T' = y_i * ymax[j+1] (Alg. 1 line 5
 * "minimum beta among remaining unprocessed nodes", taken per candidate) */
static void chain_ecm(const fmo_plan *p, const uint32_t key[2], uint32_t s_abs, int64_t g, int refresh,
                      buf_t *out)
{
    const int64_t i = p->seg_u[g], b = p->seg_b[g];
    const uint32_t sigma = (uint32_t)p->seg_sigma[g];
    const double kappa_i = p->kappa_s[i], y_i = p->y_s[i], ly_i = p->ly_s[i];
    const double omT = p->seg_omT[g];   /* 1 - exp(-beta_min) for this segment (R6) */
    const double iomT = p->seg_iomT[g]; /* RN(1 / omT)                                      */
    int64_t j = p->seg_a[g] - 1;
    double zq = p->seg_x0[g];          /* q_hat = zq / dq                                  */
    double dq = p->seg_d0[g];
    double h = p->seg_h0[g];
    const int32_t id_i = p->perm[i];
    const int ordered = p->kind != FMO_UNDIRECTED;
    const int64_t excl = p->excl ? p->excl[i] : -1;
    for (uint32_t d = 0;; d++) {
        uint32_t ctr[4] = {d, sigma, (uint32_t)i, s_abs}, W[4];
        fmo_philox4x32_10(ctr, key, W);
        out->draws++;
        double E = -log(fmo_u01(W[0]));
        double R = E / h;
        if (!(R < (double)(b - 1 - j))) break;
        j = j + 1 + (int64_t)floor(R);
        out->landed++;
        if (j == excl) continue;
        /* Eq. 4 in fitness form: p = z / ((1 - t) + z), z = x_i y_i x_j y_j, t = y_i y_j */
        double z = kappa_i * p->ckappa[j];
        double t = y_i * p->cy[j];
        double Dp = (1.0 - t) + z;
        if (z * dq > zq * Dp * (1.0 + 0x1p-50)) out->err = FMO_ERR_STATE;
        if ((fmo_u01(W[1]) * zq) * Dp < z * dq) { /* Alg. 1 line 10, cross-multiplied (R10) */
            /* Eq. 5: w - 1 ~ Geometric on {0,1,..} with ratio t = y_i y_j; inverse transform
             * with log t = log y_i + log y_j (R8) */
            double G = floor(log(fmo_u01(W[2])) / (ly_i + p->cly[j]));
            int32_t w;
            if (G <= 2147483646.0) {
                w = 1 + (int32_t)G;
            } else {
                w = INT32_MAX;
                out->flags |= FMO_FLAG_WEIGHT_SATURATED;
            }
            out->accepted++;
            buf_push(out, id_i, p->cperm[j], w, ordered);
        }
        /* Alg. 1 line 12: q <- p_hat_ij(beta_min) = z / (1 - T + z) (Eq. 6 as equality, R7) */
        zq = z;
        if (refresh) {
            double omTj = 1.0 - y_i * p->ymax[j + 1]; /* T' = y_i max_{w > j} y_w (R17) */
            dq = omTj + z;
            h = log1p(z * (1.0 / omTj));
        } else {
            dq = omT + z;
            h = log1p(z * iomT);
        }
    }
}

/* ------------------------------------------------------------------------------------------ */
/* Threaded driver: jobs = (sample, block of segments), results concatenated in job order.     */
/* ------------------------------------------------------------------------------------------ */
typedef struct {
    int64_t sample;  /* index within the call */
    int64_t g0, g1;  /* segment range */
} job_t;

typedef struct {
    const fmo_plan *p;
    uint32_t key[2];
    int64_t first_sample;
    job_t *jobs;
    buf_t *bufs;
    int64_t n_jobs;
    int64_t next;
    int refresh;
    pthread_mutex_t mu;
} pool_t;

static void *worker(void *arg)
{
    pool_t *P = (pool_t *)arg;
    for (;;) {
        pthread_mutex_lock(&P->mu);
        int64_t k = P->next++;
        pthread_mutex_unlock(&P->mu);
        if (k >= P->n_jobs) break;
        job_t J = P->jobs[k];
        uint32_t s_abs = (uint32_t)(P->first_sample + J.sample);
        for (int64_t g = J.g0; g < J.g1; g++) {
            if (P->p->model == FMO_UBCM) chain_ubcm(P->p, P->key, s_abs, g, &P->bufs[k]);
            else chain_ecm(P->p, P->key, s_abs, g, P->refresh, &P->bufs[k]);
        }
    }
    return NULL;
}

int fmo_sample(const fmo_plan *p, uint64_t seed, int64_t first_sample, int64_t n_samples,
               const int32_t *rows, int64_t n_rows, int nthreads, fmo_result **out)
{
    return fmo_sample_ex(p, seed, first_sample, n_samples, rows, n_rows, nthreads, 0u, out);
}

int fmo_sample_ex(const fmo_plan *p, uint64_t seed, int64_t first_sample, int64_t n_samples,
                  const int32_t *rows, int64_t n_rows, int nthreads, uint32_t flags, fmo_result **out)
{
    *out = NULL;
    if (!p || n_samples < 0 || first_sample < 0 || first_sample + n_samples > ((int64_t)1 << 32))
        return FMO_ERR_INVALID;
    if (nthreads < 1) nthreads = 1;
    /* job list */
    int64_t per_sample = 0;
    const int64_t BLK = 2048;
    if (rows) {
        for (int64_t r = 0; r < n_rows; r++) {
            if (rows[r] < 0 || rows[r] >= p->n || (r > 0 && rows[r] <= rows[r - 1])) return FMO_ERR_INVALID;
        }
        per_sample = n_rows;
    } else {
        per_sample = (p->nseg + BLK - 1) / BLK;
    }
    int64_t n_jobs = per_sample * n_samples;
    pool_t P;
    memset(&P, 0, sizeof(P));
    P.p = p;
    P.key[0] = (uint32_t)(seed & 0xffffffffu);
    P.key[1] = (uint32_t)(seed >> 32);
    P.first_sample = first_sample;
    P.n_jobs = n_jobs;
    P.refresh = (flags & FMO_SAMPLE_BETA_REFRESH) && p->model == FMO_ECM;
    P.jobs = (job_t *)malloc(sizeof(job_t) * (size_t)(n_jobs + 1));
    P.bufs = (buf_t *)calloc((size_t)n_jobs + 1, sizeof(buf_t));
    if (!P.jobs || !P.bufs) { free(P.jobs); free(P.bufs); return FMO_ERR_NOMEM; }
    for (int64_t s = 0; s < n_samples; s++) {
        for (int64_t k = 0; k < per_sample; k++) {
            job_t *J = &P.jobs[s * per_sample + k];
            J->sample = s;
            if (rows) {
                J->g0 = p->row_seg[rows[k]];
                J->g1 = p->row_seg[rows[k] + 1];
            } else {
                J->g0 = k * BLK;
                J->g1 = (k + 1) * BLK < p->nseg ? (k + 1) * BLK : p->nseg;
            }
        }
    }
    pthread_mutex_init(&P.mu, NULL);
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)nthreads);
    int started = 0;
    for (int t = 1; t < nthreads && th; t++)
        if (pthread_create(&th[t], NULL, worker, &P) == 0) started = t; else break;
    worker(&P);
    for (int t = 1; t <= started; t++) pthread_join(th[t], NULL);
    free(th);
    pthread_mutex_destroy(&P.mu);

    int rc = FMO_OK;
    int64_t total = 0;
    for (int64_t k = 0; k < n_jobs; k++) {
        if (P.bufs[k].err) rc = P.bufs[k].err;
        total += P.bufs[k].n;
    }
    fmo_result *R = NULL;
    if (rc == FMO_OK) rc = result_alloc(&R, n_samples, total, p->model == FMO_ECM);
    if (rc == FMO_OK) {
        int64_t pos = 0;
        for (int64_t k = 0; k < n_jobs; k++) {
            buf_t *B = &P.bufs[k];
            if (B->n) {
                memcpy(R->edges + 2 * pos, B->e, sizeof(int32_t) * 2 * (size_t)B->n);
                if (R->weights) memcpy(R->weights + pos, B->w, sizeof(int32_t) * (size_t)B->n);
            }
            pos += B->n;
            R->draws += B->draws; R->landed += B->landed; R->accepted += B->accepted;
            R->flags |= B->flags;
            R->offsets[P.jobs[k].sample + 1] = pos;
        }
        for (int64_t s = 1; s <= n_samples; s++)
            if (R->offsets[s] < R->offsets[s - 1]) R->offsets[s] = R->offsets[s - 1];
    }
    for (int64_t k = 0; k < n_jobs; k++) { free(P.bufs[k].e); free(P.bufs[k].w); }
    free(P.bufs); free(P.jobs);
    *out = R;
    return rc;
}

/* ------------------------------------------------------------------------------------------ */
/* Level 1: brute force ("evaluates edge probability for every pair of nodes").          */
/* Own RNG: xoshiro256** seeded by splitmix64 -- unrelated to Philox.                          */
/* ------------------------------------------------------------------------------------------ */
typedef struct { uint64_t s[4]; } xo_t;
static uint64_t splitmix64(uint64_t *x)
{
    uint64_t z = (*x += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
static uint64_t xo_next(xo_t *r)
{
    uint64_t *s = r->s;
    uint64_t res = rotl(s[1] * 5, 7) * 9, t = s[1] << 17;
    s[2] ^= s[0]; s[3] ^= s[1]; s[1] ^= s[2]; s[0] ^= s[3]; s[2] ^= t; s[3] = rotl(s[3], 45);
    return res;
}
static double xo_unif(xo_t *r) { return (double)(xo_next(r) >> 11) * 0x1p-53; } /* [0,1) */

static double pair_p(int model, double xi, double xj, double yi, double yj, double *t_out)
{
    if (model == FMO_UBCM) {
        double X = xi * xj;
        *t_out = 0.0;
        return X / (1.0 + X);
    }
    double t = yi * yj;
    double z = (xi * xj) * t;
    *t_out = t;
    return z / (1.0 - t + z);
}

int fmo_bruteforce2(int model, int kind, int64_t n1, const double *x1, const double *y1, int64_t n2,
                    const double *x2, const double *y2, uint64_t seed, int64_t n_samples, fmo_result **out)
{
    *out = NULL;
    if (kind == FMO_UNDIRECTED) { n2 = n1; x2 = x1; y2 = y1; }
    if (n1 < 1 || n2 < 1 || !x1 || !x2 || (model == FMO_ECM && (!y1 || !y2)) || n_samples < 0) return FMO_ERR_INVALID;
    if (kind == FMO_DIRECTED && n1 != n2) return FMO_ERR_INVALID;
    xo_t rng;
    uint64_t sm = seed;
    for (int k = 0; k < 4; k++) rng.s[k] = splitmix64(&sm);
    buf_t B;
    memset(&B, 0, sizeof(B));
    int64_t *off = (int64_t *)calloc((size_t)n_samples + 1, sizeof(int64_t));
    if (!off) return FMO_ERR_NOMEM;
    for (int64_t s = 0; s < n_samples; s++) {
        for (int64_t i = 0; i < n1; i++) {
            for (int64_t j = (kind == FMO_UNDIRECTED ? i + 1 : 0); j < n2; j++) {
                if (kind == FMO_DIRECTED && j == i) continue; /* no self loops */
                double t;
                double pij = pair_p(model, x1[i], x2[j], model == FMO_ECM ? y1[i] : 0.0,
                                    model == FMO_ECM ? y2[j] : 0.0, &t);
                B.draws++;
                if (xo_unif(&rng) < pij) {
                    int32_t w = 1;
                    if (model == FMO_ECM)
                        while (xo_unif(&rng) < t && w < INT32_MAX) w++; /* P(w) = t^{w-1}(1-t) */
                    B.accepted++;
                    buf_push(&B, (int32_t)i, (int32_t)j, w, kind != FMO_UNDIRECTED);
                }
            }
        }
        off[s + 1] = B.n;
    }
    if (B.err) { free(off); free(B.e); free(B.w); return B.err; }
    fmo_result *R = NULL;
    int rc = result_alloc(&R, n_samples, B.n, model == FMO_ECM);
    if (rc == FMO_OK) {
        memcpy(R->offsets, off, sizeof(int64_t) * (size_t)(n_samples + 1));
        if (B.n) {
            memcpy(R->edges, B.e, sizeof(int32_t) * 2 * (size_t)B.n);
            if (R->weights) memcpy(R->weights, B.w, sizeof(int32_t) * (size_t)B.n);
        }
        R->draws = B.draws; R->landed = B.draws; R->accepted = B.accepted;
    }
    free(off); free(B.e); free(B.w);
    *out = R;
    return rc;
}

int fmo_bruteforce(int model, int64_t n, const double *x, const double *y, uint64_t seed,
                   int64_t n_samples, fmo_result **out)
{
    return fmo_bruteforce2(model, FMO_UNDIRECTED, n, x, y, n, x, y, seed, n_samples, out);
}

/* Closed forms for bipartite / directed ensembles (plain O(N1 N2) sums): for + node i
 * kout[i] = sum_j p_ij, kout_var[i] = sum_j p_ij (1 - p_ij); for - node j kin[j], kin_var[j]
 * (directed: j != i).  ECM: p from Eq. 4 with the cross-set fitness. */
void fmo_expected2(int model, int kind, int64_t n1, const double *x1, const double *y1, int64_t n2,
                   const double *x2, const double *y2, double *kout, double *kout_var, double *kin,
                   double *kin_var)
{
    for (int64_t i = 0; i < n1; i++) { kout[i] = 0.0; kout_var[i] = 0.0; }
    for (int64_t j = 0; j < n2; j++) { kin[j] = 0.0; kin_var[j] = 0.0; }
    for (int64_t i = 0; i < n1; i++) {
        for (int64_t j = 0; j < n2; j++) {
            if (kind == FMO_DIRECTED && i == j) continue;
            double t;
            double pij = pair_p(model, x1[i], x2[j], model == FMO_ECM ? y1[i] : 0.0, model == FMO_ECM ? y2[j] : 0.0, &t);
            kout[i] += pij; kout_var[i] += pij * (1.0 - pij);
            kin[j] += pij; kin_var[j] += pij * (1.0 - pij);
        }
    }
}

/* ------------------------------------------------------------------------------------------ */
/* Closed forms (threaded O(N * n_nodes)).                                                     */
/* ------------------------------------------------------------------------------------------ */
typedef struct {
    int model;
    int64_t n;
    const double *x, *y;
    const int32_t *nodes;
    int64_t n_nodes;
    double *k, *kvar, *s, *svar;
    double *rowsum; /* for expected_edges: sum_{j>i} p_ij per i */
    int64_t next;
    pthread_mutex_t mu;
} exp_t;

static void *exp_worker(void *arg)
{
    exp_t *E = (exp_t *)arg;
    for (;;) {
        pthread_mutex_lock(&E->mu);
        int64_t c = E->next++;
        pthread_mutex_unlock(&E->mu);
        if (c >= E->n_nodes) break;
        int64_t i = E->nodes ? E->nodes[c] : c;
        double yi = E->model == FMO_ECM ? E->y[i] : 0.0;
        if (E->rowsum) {
            double acc = 0.0;
            for (int64_t j = i + 1; j < E->n; j++) {
                double t;
                acc += pair_p(E->model, E->x[i], E->x[j], yi, E->model == FMO_ECM ? E->y[j] : 0.0, &t);
            }
            E->rowsum[c] = acc;
            continue;
        }
        double k = 0, kv = 0, s = 0, sv = 0;
        for (int64_t j = 0; j < E->n; j++) {
            if (j == i) continue;
            double t;
            double pij = pair_p(E->model, E->x[i], E->x[j], yi, E->model == FMO_ECM ? E->y[j] : 0.0, &t);
            k += pij;
            kv += pij * (1.0 - pij);
            if (E->model == FMO_ECM) {
                /* w = 0 w.p. 1-p; else Geometric on {1,2,..} with ratio t:
                 * E[w] = p/(1-t), E[w^2] = p(1+t)/(1-t)^2 */
                double omt = 1.0 - t;
                double ew = pij / omt;
                double ew2 = pij * (1.0 + t) / (omt * omt);
                s += ew;
                sv += ew2 - ew * ew;
            }
        }
        if (E->k) E->k[c] = k;
        if (E->kvar) E->kvar[c] = kv;
        if (E->s) E->s[c] = s;
        if (E->svar) E->svar[c] = sv;
    }
    return NULL;
}

static void exp_run(exp_t *E, int nthreads)
{
    pthread_mutex_init(&E->mu, NULL);
    if (nthreads < 1) nthreads = 1;
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)nthreads);
    int started = 0;
    for (int t = 1; t < nthreads && th; t++)
        if (pthread_create(&th[t], NULL, exp_worker, E) == 0) started = t; else break;
    exp_worker(E);
    for (int t = 1; t <= started; t++) pthread_join(th[t], NULL);
    free(th);
    pthread_mutex_destroy(&E->mu);
}

void fmo_expected(int model, int64_t n, const double *x, const double *y, const int32_t *nodes,
                  int64_t n_nodes, int nthreads, double *k, double *kvar, double *s, double *svar)
{
    exp_t E;
    memset(&E, 0, sizeof(E));
    E.model = model; E.n = n; E.x = x; E.y = y; E.nodes = nodes;
    E.n_nodes = nodes ? n_nodes : n;
    E.k = k; E.kvar = kvar; E.s = s; E.svar = svar;
    exp_run(&E, nthreads);
}

double fmo_expected_edges(int model, int64_t n, const double *x, const double *y, int nthreads)
{
    exp_t E;
    memset(&E, 0, sizeof(E));
    E.model = model; E.n = n; E.x = x; E.y = y; E.n_nodes = n;
    E.rowsum = (double *)calloc((size_t)n + 1, sizeof(double));
    if (!E.rowsum) return NAN;
    exp_run(&E, nthreads);
    double tot = 0.0;
    for (int64_t i = 0; i < n; i++) tot += E.rowsum[i];
    free(E.rowsum);
    return tot;
}

/* ---- rich club: density of edges among the top-m nodes, P:L58-60, P:L233 ----
 * The top m nodes are the first m of a given order (rank -> node id `order`).
 * fmo_richclub_count: e_top[m] = #{edges (i,j) of the list : rank(i) < m and rank(j) < m}, m = 0..n,
 *   straight from the definition: an edge is inside the top m iff its larger endpoint rank is < m.
 * fmo_expected_richclub: E[e_top[m]] = sum over pairs of top-m nodes of p_ij, and the variance
 *   sum p_ij (1 - p_ij) (independent edges), m = 0..n, adding one node at a time. */
void fmo_richclub_count(int64_t n, const int32_t *order, int64_t n_edges, const int32_t *edges, int64_t *e_top)
{
    int64_t *rank = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
    int64_t *hist = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t));
    for (int64_t r = 0; r < n; r++) rank[order[r]] = r;
    for (int64_t e = 0; e < n_edges; e++) {
        int64_t a = rank[edges[2 * e]], b = rank[edges[2 * e + 1]];
        hist[a > b ? a : b]++;
    }
    e_top[0] = 0;
    for (int64_t m = 0; m < n; m++) e_top[m + 1] = e_top[m] + hist[m];
    free(rank);
    free(hist);
}

void fmo_expected_richclub(int model, int64_t n, const double *x, const double *y, const int32_t *order,
                           double *mean, double *var)
{
    mean[0] = 0.0;
    var[0] = 0.0;
    for (int64_t m = 0; m < n; m++) {
        int64_t j = order[m];
        double add = 0.0, addv = 0.0;
        for (int64_t r = 0; r < m; r++) {
            int64_t i = order[r];
            double t;
            double pij = pair_p(model, x[i], x[j], model == FMO_ECM ? y[i] : 0.0, model == FMO_ECM ? y[j] : 0.0, &t);
            add += pij;
            addv += pij * (1.0 - pij);
        }
        mean[m + 1] = mean[m] + add;
        var[m + 1] = var[m] + addv;
    }
}
