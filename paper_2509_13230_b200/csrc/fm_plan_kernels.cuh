// fm_plan_kernels.cuh -- planner kernels (fm_plan.cu) and sampler kernels (fm_sample.cu),
// declared for the host orchestration in fm_capi.cu.
#pragma once
#include "fm_internal.cuh"
#include "fm_math.cuh"

namespace fm {

struct PlanScalars {
    unsigned long long key_or;
    unsigned long long key_and;
    unsigned int flags;
    int F;
    long long total_work;  // sum over segments of work estimates (units 2^G)
    long long wmax;        // upper bound of any one segment's work (units 2^G)
};

struct RowInfo {
    double r;      // row multiplier r_u
    int64_t sat;   // saturation index sat_u
    int64_t wtot;  // Wtot_u
};

// W_u(v) (DESIGN.md 3.4 step 3): integer estimate of the draws over candidates [c0, v)
__device__ __forceinline__ int64_t plan_W(const uint64_t *P, int F, int64_t c0, double r, int64_t sat, int64_t v)
{
    const int64_t vs = v < sat ? v : sat;
    int64_t W = (vs - c0) * kUnit;
    if (v > sat) {
        const uint64_t D = P[v] - P[sat];
        W += (int64_t)floor(ldexp(__dmul_rn(r, __ull2double_rn(D)), kG - F));
    }
    return W;
}

__global__ void k_validate_key(int model, int64_t n, const double *x, const double *y, uint64_t *keys, int32_t *ids,
                               PlanScalars *sc, unsigned int *hist);
__global__ void k_gather_sorted(int model, int64_t n, const uint64_t *skeys, const double *y, const int32_t *perm,
                                double *kappa_s, double *y_s, double *ly_s);
__global__ void k_set_F(int64_t n, int L, const double *kappa_s, PlanScalars *sc);
__global__ void k_kfx(int64_t n, int L, const double *kappa_s, PlanScalars *sc, uint64_t *kfx);
__global__ void k_rows(int model, int kind, int64_t n, int64_t nc, int64_t S, const double *kappa_s, const double *y_s,
                       const double *ckappa, const double *ymax, const uint64_t *P, PlanScalars *sc, RowInfo *rows,
                       int64_t *row_m);
__global__ void k_emit(int model, int kind, int64_t n, int64_t nc, int64_t n_seg, const double *kappa_s,
                       const double *y_s, const double *ly_s, const int32_t *perm, const int32_t *excl,
                       const double *ckappa, const double *ymax, const uint64_t *P, PlanScalars *sc,
                       const RowInfo *rows, const int64_t *row_seg, const int64_t *seg_row_x, unsigned char *rec,
                       int64_t *seg_work);
__global__ void k_row_starts(int64_t n, const int64_t *row_seg, int64_t *flag);
__global__ void k_rank_of(int64_t nc, const int32_t *cperm, int32_t *crank);
__global__ void k_excl(int64_t n, const int32_t *perm, const int32_t *crank, int32_t *excl);
__global__ void k_chunks(int64_t n_seg, int64_t n_chunks, int64_t target, const int64_t *work_pre, int64_t *chunk_seg,
                         int64_t *chunk_cap);
__global__ void k_fill_caps(int64_t *chunk_cap, int64_t n_chunks, int64_t cap);
// test hook (FM_DEBUG_BAD_BOUND): scale every segment's initial bound numerator x0 by `f` so that
// the first candidates violate p <= q -- exercises the FM_DEBUG_CHECKS path (FM_ERR_BOUND)
__global__ void k_debug_scale_bound(unsigned char *rec, int64_t n_seg, int stride, double f);
__global__ void k_pack_cand(int model, int64_t nc, const double *ckappa, const int32_t *cperm, const double *cy,
                            const double *cly, double2 *cand);

// ------------------------------------------------------------------------------------------
// sampler (fm_sample.cu)
// ------------------------------------------------------------------------------------------
// Task space of one fm_sample_* call (or sample group): three consecutive sample ranges, each with
// its own lane-chunking of the plan -- range 0 the BIG chunks (most samples of a large call: fewer
// task switches), range 1 the coarse ones, range 2 the fine ones (the last samples: the end of the
// persistent queue consists of short tasks, small end-of-launch tail).  Tasks are numbered
// sample-major within each range, hence in canonical output order.  Empty ranges are allowed.
constexpr int kRanges = 3;
struct TaskMap {
    const int64_t *seg[kRanges];  // chunk_seg of the range's chunking, [n_chunks + 1]
    const int64_t *cap[kRanges];  // exclusive prefix of the chunks' scratch slots, [n_chunks + 1]
    int64_t n_chunks[kRanges];
    double inv_chunks[kRanges];   // 1 / n_chunks (quotient estimate, corrected exactly below)
    int64_t s0[kRanges];          // first sample of each range (s0[0] = 0)
    int64_t t0[kRanges];          // first task of each range (t0[0] = 0)
    int64_t cap_per_sample;
};
// (selects, not indexing by a run-time range: a dynamically indexed kernel parameter is copied to
// local memory)
#define FM_TM_SEL(M, field, k) ((k) == 0 ? (M).field[0] : (k) == 1 ? (M).field[1] : (M).field[2])

// t = s n + c, 0 <= c < n, for t < 2^52: the fp64 quotient estimate is off by at most one
__device__ __forceinline__ void divmod_est(int64_t t, int64_t n, double inv, int64_t &q, int64_t &r)
{
    q = (int64_t)__dmul_rz((double)t, inv);
    r = t - q * n;
    if (r < 0) {
        q--;
        r += n;
    } else if (r >= n) {
        q++;
        r -= n;
    }
}

__device__ __forceinline__ int task_range(const TaskMap &M, int64_t t) { return t >= M.t0[2] ? 2 : t >= M.t0[1] ? 1 : 0; }
__device__ __forceinline__ int sample_range(const TaskMap &M, int64_t s) { return s >= M.s0[2] ? 2 : s >= M.s0[1] ? 1 : 0; }
// first task of sample s (s = number of samples: the number of tasks)
__device__ __forceinline__ int64_t sample_first_task(const TaskMap &M, int64_t s)
{
    const int k = sample_range(M, s);
    return FM_TM_SEL(M, t0, k) + (s - FM_TM_SEL(M, s0, k)) * FM_TM_SEL(M, n_chunks, k);
}

__device__ __forceinline__ void task_decode(const TaskMap &M, int64_t t, int64_t &s, int64_t &c, int &k)
{
    k = task_range(M, t);
    int64_t s2;
    divmod_est(t - FM_TM_SEL(M, t0, k), FM_TM_SEL(M, n_chunks, k), FM_TM_SEL(M, inv_chunks, k), s2, c);
    s = FM_TM_SEL(M, s0, k) + s2;
}

// tasks per claim of the sampler's global queue (a warp batch; the fused write's unit)
// 32 = one task per lane and claim, the minimum (a fetch round hands out up to 32 positions and
// opens at most one new batch).  Against 64: config 5 sampler -0.75 %, config 2 -2.9 %, config 4
// -3.3 % (the warps' last claims are smaller: shorter end of the queue); 128: +2.5 ... +44 %.
#ifndef FM_QUEUE_BATCH
#define FM_QUEUE_BATCH 32
#endif
constexpr int kQueueBatch = FM_QUEUE_BATCH;
static_assert(kQueueBatch >= 32, "a fetch round serves up to 32 lanes from at most one new batch");

struct SampleArgs {
    const unsigned char *rec;      // segment records, stride kRecStride(model)
    const double *kappa_s, *y_s, *ly_s;  // CANDIDATE arrays (the - set; the rows themselves if undirected)
    const int32_t *perm;                 // candidate rank -> id
    const double2 *cand;                 // packed gather records (Plan::cand)
    const double *ymax_c;                // ECM beta_min refresh (R17): candidate Ymax [nc+1]; NULL = per segment
    TaskMap tm;                    // task -> (sample, chunking, lane-chunk) and scratch slots
    PhiloxKey key;
    LogConsts lc;                  // log polynomial constants (read as parameter-bank operands)
    uint32_t first_sample;
    int64_t n_tasks;               // tasks in the queue
    const int64_t *task_list;      // NULL: task = queue index; else task_list[queue index]
    int ordered;                   // bipartite / directed: emit (row id, candidate id) as is (R16)
    int rank_out;                  // UBCM: scratch pairs hold (row id, candidate rank), mapped by k_compact
    int64_t il_s[kRanges];         // > 0: queue order chunk-major within each range's samples (il_s[k]
                                   // samples each), so the samples of one lane-chunk run together and
                                   // share its segment records in L2; 0: sample-major (queue = task)
    int buf4;                      // scratch slots 32-byte aligned: edges are written 4 at a time (whole sectors)
    unsigned long long *task_counter;  // global queue head (zeroed before each launch)
    int counters_zeroed;           // the caller cleared task_counter and spill_counter (no memsets at the launch)
    int2 *edges;                   // scratch (normal) or final array (rerun)
    int32_t *weights;              // ECM
    const int64_t *rerun_base;     // rerun mode: per-task output base (final offsets); NULL otherwise
    const unsigned long long *n_tasks_dev;  // rerun mode: number of queued tasks, read on the device
    int64_t out_cap;               // rerun mode: capacity of the final list (writes beyond are dropped)
    int64_t out_base;              // rerun mode: added to rerun_base[t] (the edges of the preceding sample groups)
    int64_t *counts;               // [n_samples * n_chunks] edges produced per task (normal mode)
    int2 *spill_e;                 // spill area for tasks that outgrow their slot (one region of
    int32_t *spill_w;              //   `cap` edges per task, bump-allocated)
    unsigned long long *spill_counter;
    int64_t spill_cap;             // edges in the spill area
    int64_t *spill_off;            // [n_tasks] spill region of each task: -1 none, -2 failed
    unsigned long long *counters;  // draws, landed, accepted
    unsigned int *flags;
    int check;                     // FM_DEBUG_CHECKS: test p <= q (1 + 2^-50) at every landed candidate
    // v3 fused write (fm_sample.cu: copier_loop): a copier warp per block copies the finished queue
    // batches (kQueueBatch canonical tasks) from the scratch slots into the final list
    int fuse;
    int discard;                   // discard.global.L2 of a batch's scratch lines after its copy
    int64_t n_groups;              // queue batches
    unsigned long long *grp_state; // [n_groups] look-back status (flag bits | edge count / prefix)
    int64_t *dest;                 // [n_tasks + 1] final offset of each task (dest[n_tasks] = total)
    int2 *out_e;                   // final list (capacity out_cap)
    int32_t *out_w;
    const int32_t *rank_map;       // UBCM rank-out: candidate rank -> id
    // statistics mode (fm_sample_degrees, NEXT-3): when deg_row != NULL no edge list is written;
    // accepted edges add 1 (and w) to the row node's and the candidate's sums instead
    unsigned long long *deg_row, *deg_col, *str_row, *str_col;
    // rich club (statistics mode, undirected): accepted edges counted by their larger rank
    unsigned long long *rank_hist;
};

cudaError_t launch_sample(int model, const SampleArgs &a, cudaStream_t st);
// tasks whose count exceeds their slot -> overflow list (re-run straight into the final array)
cudaError_t launch_overflow(int64_t n_tasks, const TaskMap &tm, const int64_t *counts, const int64_t *spill_off,
                            unsigned long long *n_overflow, int64_t *overflow_list, cudaStream_t st);
// gather every task's slot (+ spill) into the final contiguous arrays of out_cap elements
cudaError_t launch_compact(int64_t out_cap, int64_t n_tasks, const TaskMap &tm, const int64_t *counts, const int64_t *dest,
                           const int64_t *spill_off, const int2 *scratch_e, const int32_t *scratch_w,
                           const int2 *spill_e, const int32_t *spill_w, int2 *out_e, int32_t *out_w,
                           const int32_t *rank_map, int ordered, int ecm_rec, int small, const int64_t *out_base,
                           cudaStream_t st);
// offsets[s] = *base_in + (first final position of sample s), s <= n_samples; *base_out = the running total
// (base_out_host: optional mapped page-locked host word that receives the running total as well)
cudaError_t launch_offsets(int64_t n_samples, const TaskMap &tm, const int64_t *dest, int64_t *offsets,
                           const int64_t *base_in, int64_t *base_out, int64_t *base_out_host, cudaStream_t st);
// out[i] += in[i], i < n (uint64)
cudaError_t launch_add_u64(const uint64_t *in, uint64_t *out, int64_t n, cudaStream_t st);
cudaError_t launch_debug_eval(int fn, int64_t n, const double *in, double *out, cudaStream_t st);

}  // namespace fm
