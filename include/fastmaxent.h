/*
 * fastmaxent.h -- C-ABI of the B200 (sm_100a) sampler for the MaxEnt configuration models of
 * arXiv 2509.13230, "Fast unbiased sampling of networks with given expected degrees and
 * strengths" (PAPER.md, cited P:L<n>).
 *
 * The library samples simple undirected graphs in which every unordered pair {i, j} is an
 * edge independently with probability
 *     UBCM  p_ij = x_i x_j / (1 + x_i x_j)                       (x = e^-alpha)
 *     ECM   p_ij = z / (1 - t + z),  z = x_i y_i x_j y_j, t = y_i y_j   (Eq. 4, y = e^-beta)
 * with ECM edge weights w >= 1, P(w) = t^{w-1} (1 - t)            (Eq. 5),
 * by the Miller-Hagberg-style sorted geometric-skip rejection sampler of P:L127-136 (UBCM)
 * and Algorithm 1, P:L144-166 (ECM), with the readings listed in DESIGN.md section 3.
 *
 * Conventions for every entry point:
 *  - Returns an fm_status; never aborts.  On error nothing is allocated, *out is zeroed, and
 *    fm_last_error() returns a thread-local message.
 *  - Device temporaries come from the device's default stream-ordered memory pool, whose release
 *    threshold the library bounds at the first call on a device (FM_POOL_RELEASE_BYTES, default
 *    3/4 of the device memory): freed memory above it is returned to the device; fm_pool_trim()
 *    returns the cached memory on demand.
 *  - All work is ordered on the caller's CUDA stream `cuda_stream` (cudaStream_t; NULL = the
 *    legacy default stream) on the current device.
 *  - Input pointers may be HOST or DEVICE memory (detected with cudaPointerGetAttributes); they
 *    are borrowed for the duration of the call only.
 *  - Objects returned through *out are library-owned; release them with fm_free().
 *  - Results are pure functions of (x, y, seg_target, seed, sample index): sample k is
 *    bit-identical whether produced alone or inside a batch (R1).
 */
#ifndef FASTMAXENT_H
#define FASTMAXENT_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FM_ABI_VERSION 1

typedef enum {
    FM_OK = 0,
    FM_ERR_INVALID = -1, /* bad argument: N < 2 or > 2^31-1, NULL pointer, x not finite or < 0,
                            y not in [0,1), kappa_max^4 overflow, seg_target out of range,
                            sample range beyond 2^32 */
    FM_ERR_NOMEM = -2,   /* device or host allocation failed */
    FM_ERR_CUDA = -3,    /* CUDA runtime error (no device, launch failure, ...) */
    FM_ERR_BOUND = -4,   /* contract violation p > q (1 + 2^-50) at a landed candidate ("abort,
                            never clamp"; R13).  Checked only when the environment has
                            FM_DEBUG_CHECKS=1 at call time; the call then releases everything and
                            fills nothing.  (FM_DEBUG_BAD_BOUND=1 at fm_sort_plan time is a test
                            hook that builds a plan with too-small initial bounds.) */
    FM_ERR_STATE = -5    /* wrong object / model mismatch / internal invariant violated */
} fm_status;

typedef enum { FM_UBCM = 0, FM_ECM = 1 } fm_model;

/* Graph kind (R16).  Undirected: pairs {i, j} of one node set.  Bipartite:
 * pairs (+i, -j) of two node sets.  Directed: ordered pairs (i, j), i != j, with out-fitness and
 * in-fitness (the bipartite graph of out- and in-copies without the diagonal). */
typedef enum { FM_UNDIRECTED = 0, FM_BIPARTITE = 1, FM_DIRECTED = 2 } fm_graph;

enum {
    FM_FLAG_WEIGHT_SATURATED = 1u, /* an ECM weight exceeded INT32_MAX and was clamped (R8) */
    FM_FLAG_SCRATCH_RERUN = 2u,    /* some chunks overflowed their scratch and were re-run (same result) */
    FM_FLAG_HOST_TRUNCATED = 4u    /* fm_sample_to_host: the host buffers were too small, nothing valid in them */
};

/* Opaque, immutable sampling plan: the sorted order (P:L133 step (i); Alg. 1 line 3), the
 * beta_min suffix maximum, and the segment table of the planner.
 * Device-resident; safe to use concurrently from several streams once created. */
typedef struct fm_plan fm_plan;

/* Sampled edge lists: n_samples graphs, concatenated. */
typedef struct {
    int64_t n_samples;
    int64_t n_edges;   /* total over all samples */
    int64_t *offsets;  /* HOST int64[n_samples + 1]: sample s = edges[offsets[s] .. offsets[s+1]) */
    int32_t *edges;    /* DEVICE int32[2 * n_edges]: pairs in original ids ("Edge list E"; no
                          duplicates): undirected (src, dst) with src < dst, no self loops;
                          bipartite (+ id, - id); directed (source, target), no self loops      */
    int32_t *weights;  /* DEVICE int32[n_edges] (ECM, w >= 1), NULL for UBCM                         */
    int64_t draws;     /* counters summed over samples: geometric draws incl. terminal ones     */
    int64_t landed;    /* proposals (candidates reached, p/q tests)                              */
    int64_t accepted;  /* == n_edges                                                             */
    int64_t segments;  /* plan segments x n_samples                                             */
    int64_t chunks;    /* warp chunks x n_samples                                               */
    uint32_t flags;    /* FM_FLAG_*                                                              */
    void *_owner;      /* internal                                                               */
} fm_edges;

typedef struct {
    int32_t model;
    int32_t kind;         /* fm_graph */
    int64_t n_minus;      /* candidates: the - set (bipartite), in-copies (directed), == n undirected */
    int64_t n;
    int64_t seg_target;
    int32_t F;            /* fixed-point exponent of the planner (DESIGN.md 3.4 step 1) */
    int64_t n_segments;
    int64_t n_chunks;
    int64_t est_draws;    /* planner estimate of draws per sample (sum of segment work) */
} fm_plan_info;

/* a1-a4.  Validate the fitness vectors, sort the nodes by descending kappa (x for UBCM,
 * x*y for ECM; ties by ascending id), build the beta_min suffix maximum (ECM) and the segment
 * plan.  x: float64[n] (x_i = e^{-alpha_i} >= 0), y: float64[n] (ECM: y_i = e^{-beta_i} in
 * [0,1); must be NULL for UBCM).  seg_target S: expected draws per hub-row segment, 0 = 256,
 * otherwise 8 <= S <= 2^40 (S changes results; R15).  Synchronises the stream once. */
fm_status fm_sort_plan(fm_model model, int64_t n, const double *x, const double *y,
                       int64_t seg_target, void *cuda_stream, fm_plan **plan_out);

/* As fm_sort_plan for bipartite (kind FM_BIPARTITE: rows = the + set (x_plus, y_plus), candidates
 * = the - set (x_minus, y_minus), each sorted by its own key) and directed graphs
 * (FM_DIRECTED: x_plus/y_plus = out-fitness, x_minus/y_minus = in-fitness, n_plus == n_minus,
 * self loops excluded).  n_plus, n_minus >= 1.  Sampled with fm_sample_ubcm/ecm. */
fm_status fm_sort_plan_bipartite(fm_model model, fm_graph kind, int64_t n_plus, const double *x_plus,
                                 const double *y_plus, int64_t n_minus, const double *x_minus,
                                 const double *y_minus, int64_t seg_target, void *cuda_stream,
                                 fm_plan **plan_out);

/* a5-a6.  Draw n_samples graphs (sample indices first_sample .. first_sample+n_samples-1,
 * first_sample + n_samples <= 2^32) from the UBCM with Philox key `seed`.
 * Fills *out (device edges, host offsets).  Synchronises the stream once (to size the output).
 * FM_ERR_STATE if the plan is an ECM plan.  n_samples == 0 returns an empty result. */
fm_status fm_sample_ubcm(const fm_plan *plan, uint64_t seed, int64_t first_sample, int64_t n_samples,
                         void *cuda_stream, fm_edges *out);

/* As fm_sample_ubcm for the weighted ECM (Algorithm 1; Eq. 3-6): also fills
 * out->weights.  FM_ERR_STATE if the plan is a UBCM plan. */
fm_status fm_sample_ecm(const fm_plan *plan, uint64_t seed, int64_t first_sample, int64_t n_samples,
                        void *cuda_stream, fm_edges *out);

/* Sampling options (fm_sample_ecm_ex). */
enum { FM_SAMPLE_BETA_REFRESH = 1u };
/* As fm_sample_ecm with options.  FM_SAMPLE_BETA_REFRESH (R17): after each
 * reached candidate cur the bound for the candidates still ahead uses beta_min over them,
 * T' = y_u * max_{w > cur} y_w (Alg. 1 line 5 "minimum beta among remaining unprocessed nodes",
 * P:L153, taken per candidate) instead of the segment-start value: fewer proposals per edge
 * (about 7 % on config 3), the same law, different random streams' use, so a different (equally
 * valid) sample than without the flag.  Unknown flags: FM_ERR_INVALID. */
fm_status fm_sample_ecm_ex(const fm_plan *plan, uint64_t seed, int64_t first_sample, int64_t n_samples,
                           uint32_t flags, void *cuda_stream, fm_edges *out);

/* Counters of a statistics-mode call (sums over its samples). */
typedef struct {
    int64_t draws, landed, accepted;
    uint32_t flags;
} fm_counters;

/* Ensemble statistics without edge lists (the consumer of the samples, P:L232-233,
 * P:L253): draws samples first_sample .. first_sample+n_samples-1 exactly as fm_sample_ubcm/ecm
 * (same plan, seed and streams, so the same graphs) and ADDS, over those samples, each node's
 * degree and (ECM) strength into caller-owned DEVICE arrays (uint64, zero them first to start):
 * undirected: deg_plus[n] (deg_minus/str_minus NULL); bipartite/directed: deg_plus[n] for the
 * + (out) set and deg_minus[n_minus] for the - (in) set; str_* likewise for the ECM (NULL for
 * UBCM).  Integer atomics: the sums are deterministic.  Synchronises the stream once. */
fm_status fm_sample_degrees(const fm_plan *plan, uint64_t seed, int64_t first_sample, int64_t n_samples,
                            void *cuda_stream, uint64_t *deg_plus, uint64_t *deg_minus, uint64_t *str_plus,
                            uint64_t *str_minus, fm_counters *out);

/* Rich-club profile of the ensemble (the top-alpha density of P:L58-60):
 * draws the same samples as fm_sample_ubcm/ecm (undirected plans only, else FM_ERR_STATE) and
 * ADDS to the caller-owned DEVICE array e_top[n+1] (uint64; zero it first to start), for every
 * m = 0..n, the number of sampled edges joining two of the m top-ranked nodes, summed over the
 * samples.  Ranks are the plan's sort order (kappa descending, ties by id; fm_plan_export's perm):
 * for the UBCM the order of expected degree.  Density of the top m: e_top[m] / (R m(m-1)/2).
 * Integer atomics: deterministic.  Synchronises the stream once. */
fm_status fm_sample_richclub(const fm_plan *plan, uint64_t seed, int64_t first_sample, int64_t n_samples,
                             void *cuda_stream, uint64_t *e_top, fm_counters *out);

/* Closed-form expectations under the model (the targets of the statistical gates):
 * for each listed node i (nodes: int32[n_nodes] node ids, HOST or DEVICE; NULL = all n nodes, in
 * order), over every j != i,
 *     k[c] = sum_j p_ij,  kvar[c] = sum_j p_ij (1 - p_ij)             (Eq. 4)
 *     s[c] = sum_j p_ij / (1 - t_ij),  svar[c] = sum_j Var[w_ij]      (ECM only; Eq. 3-5)
 * i.e. the expected degree / strength of node i and their variances (independent pairs, P:L90-93;
 * E[w_ij] = p/(1-t), E[w_ij^2] = p(1+t)/(1-t)^2).  p in fitness form as for the sampler (x, y as in
 * fm_sort_plan, HOST or DEVICE float64[n]).  O(n * n_nodes) fp64 pair evaluations with compensated
 * summation.  Outputs: caller-owned DEVICE float64[n_nodes]; any may be NULL (s/svar must be NULL
 * for the UBCM).  Synchronises the stream. */
fm_status fm_expected_degrees(fm_model model, int64_t n, const double *x, const double *y, const int32_t *nodes,
                              int64_t n_nodes, double *k, double *kvar, double *s, double *svar,
                              void *cuda_stream);

/* fm_sample_ubcm / fm_sample_ecm(_ex) with the result ALSO delivered to caller-owned HOST buffers
 * (the model is the plan's; flags as fm_sample_ecm_ex; Algorithm 1's edge list E):
 * edges_host int32[2*host_cap], weights_host int32[host_cap] (ECM; may be NULL).  The call runs as
 * groups of samples and copies each group's part of the list to the host while the next groups are
 * still being sampled, so the device -> host transfer (the bound of the host path: 8 B per edge over
 * PCIe) starts after the first group instead of after the whole call.  Use page-locked host memory
 * for the copies to be asynchronous (both host copies go in 64 MiB pieces that start at 2 MiB
 * boundaries of the destination: the rate of the transfer depends on that alignment).  `out` is filled as by fm_sample_* (the device list stays
 * valid until fm_free).  If the list holds more than host_cap edges, out->flags has
 * FM_FLAG_HOST_TRUNCATED, the host buffers hold nothing valid, and fm_edges_to_host can be called
 * with larger buffers.  Same results as fm_sample_*; synchronises the stream. */
fm_status fm_sample_to_host(const fm_plan *plan, uint64_t seed, int64_t first_sample, int64_t n_samples, uint32_t flags,
                            void *cuda_stream, int32_t *edges_host, int32_t *weights_host, int64_t host_cap,
                            fm_edges *out);

/* Copy a result to caller-owned HOST buffers: edges_host int32[2*n_edges], weights_host
 * int32[n_edges] (may be NULL).  Stream-ordered; synchronises the stream. */
fm_status fm_edges_to_host(const fm_edges *e, int32_t *edges_host, int32_t *weights_host,
                           void *cuda_stream);

/* Plan metadata (host struct, caller-owned). */
fm_status fm_plan_get_info(const fm_plan *plan, fm_plan_info *info);

/* Inspection: copy plan arrays to caller-owned HOST buffers (any may be NULL):
 * perm int32[n] (rank -> id), kappa_s float64[n], y_s float64[n] (ECM), ymax float64[n+1] (ECM),
 * ly_s float64[n] (ECM, log y_s), seg int32[4*n_segments] as (u, a, b, sigma), and per segment
 * float64[n_segments]: seg_h0 (= -log(1 - q0)), seg_x0 / seg_d0 (q0 = x0 / d0), seg_omT (1 - T),
 * seg_iomT (RN(1/(1 - T))) -- DESIGN.md 3.4 step 6.  Synchronises the current device. */
fm_status fm_plan_export(const fm_plan *plan, int32_t *perm, double *kappa_s, double *y_s, double *ymax, double *ly_s,
                         int32_t *seg, double *seg_h0, double *seg_x0, double *seg_d0, double *seg_omT,
                         double *seg_iomT);

/* Inspection of the candidate set of a bipartite/directed plan (the row arrays when undirected):
 * cperm int32[n_minus], ckappa/cy/cly float64[n_minus], excl int32[n] (directed: candidate rank of
 * each row's own node, else -1).  Any pointer may be NULL.  Synchronises the current device. */
fm_status fm_plan_export_candidates(const fm_plan *plan, int32_t *cperm, double *ckappa, double *cy,
                                    double *cly, int32_t *excl);

/* Device-side phase timing (for benchmarks).  When enabled, CUDA events are recorded on the
 * call's stream around each phase; fm_timing_get synchronises those events and returns the
 * accumulated milliseconds since the last reset.  `launches` counts every kernel the library
 * launched (whether or not timing is enabled). */
typedef struct {
    double plan_ms;     /* fm_sort_plan, all a1-a4 kernels                                  */
    double sample_ms;   /* the sampler kernel(s) k_sample (a5)                              */
    double write_ms;    /* count scan + compaction (a6), incl. overflow re-runs             */
    int64_t sample_launches;
    int64_t launches;
} fm_timing;
fm_status fm_timing_enable(int on);
fm_status fm_timing_get(fm_timing *t, int reset);

/* Diagnostics of the device math (tests only): out[i] = f(in[i]) for i < n on DEVICE buffers,
 * fn 0 = log(x) (x > 0 normal), 1 = log1p(x) (x >= 0), 2 = -log(u01(k)), k = (uint32) in[i]
 * -- the fp64 logarithms the sampler uses in place of libm; fn 3 = in[2i] / in[2i+1]
 * by the sampler's Markstein division (in holds 2n doubles; must equal the IEEE quotient).
 * Stream-ordered. */
fm_status fm_debug_eval(int32_t fn, int64_t n, const double *in_dev, double *out_dev, void *cuda_stream);

/* Release the memory the current device's default pool holds cached beyond keep_bytes (freed
 * temporaries of earlier calls) back to the device.  Synchronises the device. */
fm_status fm_pool_trim(uint64_t keep_bytes);

/* Release an fm_plan* or the buffers of an fm_edges* (the struct itself is caller-owned and
 * is zeroed).  Objects are tagged; NULL is a no-op. */
void fm_free(void *obj);

/* Thread-local message describing the last non-OK status. */
const char *fm_last_error(void);

/* FM_ABI_VERSION of the loaded library. */
int32_t fm_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* FASTMAXENT_H */
