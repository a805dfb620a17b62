// fm_capi.cu -- the C-ABI (include/fastmaxent.h): validation, stream-ordered memory, launch
// orchestration of the a1-a6 kernels, status codes.
#include <algorithm>
#include <cmath>
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <set>
#include <string>
#include <type_traits>
#include <vector>

#include <nvtx3/nvToolsExt.h>  // header-only NVTX: host ranges around every entry point (no-ops without a tool)

#include "fm_internal.cuh"
#include "fm_plan_kernels.cuh"

#ifdef FM_TRACE
namespace fm {
void dump_trace();  // fm_sample.cu (timeline instrumentation build)
}
#endif
namespace fm {
void fuse_stats_dump();  // fm_sample.cu (FM_FUSE_STATS instrumentation build; no-op otherwise)
}
namespace fm {
std::atomic<long long> g_launches{0};
void count_launch(int n) { g_launches += n; }
}  // namespace fm

using namespace fm;

namespace {

// ---- optional device-side phase timing (fm_timing_*) ----
enum { kPhasePlan = 0, kPhaseSample = 1, kPhaseWrite = 2 };
struct Pending {
    int phase;
    cudaEvent_t a, b;
};
std::mutex g_tmu;
std::vector<Pending> g_pending;
std::atomic<bool> g_timing{false};
double g_phase_ms[3] = {0, 0, 0};
long long g_sample_launches = 0;
// a sample call's spans: a .. b = first sampler start to last sampler end (the pipelined groups'
// samplers overlap each other and the preceding groups' compactions), b .. c = the exposed rest
struct CallSpan {
    cudaEvent_t a, b, c;
};
std::vector<CallSpan> g_call_spans;

struct PhaseTimer {
    int phase = -1;
    cudaEvent_t a = nullptr, b = nullptr;
    void begin(int ph, cudaStream_t st)
    {
        if (!g_timing.load()) return;
        phase = ph;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a, st);
    }
    void end(cudaStream_t st)
    {
        if (phase < 0) return;
        cudaEventRecord(b, st);
        std::lock_guard<std::mutex> lk(g_tmu);
        g_pending.push_back({phase, a, b});
        phase = -1;
    }
};

// NVTX range of an entry point (or a phase inside it): visible in Nsight Systems / Compute timelines
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

thread_local std::string g_err;
std::mutex g_mu;
std::set<const void *> g_plans;
std::set<const void *> g_owners;

fm_status fail(fm_status s, const char *fmt, ...)
{
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
    return s;
}

fm_status cuda_fail(cudaError_t e, const char *what)
{
    if (e == cudaErrorMemoryAllocation) {
        cudaGetLastError();
        return fail(FM_ERR_NOMEM, "%s: %s", what, cudaGetErrorString(e));
    }
    return fail(FM_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

// cudaMallocAsync from the device's default pool.  The pool keeps freed temporaries cached (release
// threshold: 3/4 of the device memory, configure_pool); a process that makes calls of many different
// sizes can end up with most of the device cached in blocks that fit none of the next requests
// (seen in a 13,000-case fuzz sweep): on an out-of-memory error the stream is synchronised, the
// pool's unused memory is returned to the device and the allocation is tried once more.
cudaError_t malloc_async_retry(void **p, size_t bytes, cudaStream_t st)
{
    cudaError_t e = cudaMallocAsync(p, bytes, st);
    if (e != cudaErrorMemoryAllocation) return e;
    cudaGetLastError();
    int dev = 0;
    cudaMemPool_t pool;
    if (cudaStreamSynchronize(st) != cudaSuccess || cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetDefaultMemPool(&pool, dev) != cudaSuccess || cudaMemPoolTrimTo(pool, 0) != cudaSuccess) {
        cudaGetLastError();
        return cudaErrorMemoryAllocation;
    }
    return cudaMallocAsync(p, bytes, st);
}

// Device allocations of one call; everything not released is freed (stream-ordered) on exit.
struct Allocs {
    cudaStream_t st;
    std::vector<void *> ptrs;
    explicit Allocs(cudaStream_t s) : st(s) {}
    ~Allocs()
    {
        for (void *p : ptrs)
            if (p) cudaFreeAsync(p, st);
    }
    template <typename T>
    cudaError_t get(T **p, size_t count)
    {
        *p = nullptr;
        if (count == 0) count = 1;
        cudaError_t e = malloc_async_retry((void **)p, count * sizeof(T), st);
        if (e == cudaSuccess) ptrs.push_back(*p);
        return e;
    }
    void release(void *p)
    {
        for (auto &q : ptrs)
            if (q == p) q = nullptr;
    }
};

// The stream-ordered temporaries of a call (scratch ~1.3x the edge list) come from the device's
// default pool.  Its release threshold is bounded (FM_POOL_RELEASE_BYTES, default 3/4 of the
// device memory): memory freed by a call stays mapped for the next call up to that size (no
// remapping per call: at 1/4 the 35-50 GB working set of a config-5 call was released and
// re-mapped at every plan's synchronisation, 1-14 ms of jitter), and anything above it is returned
// to the device at the next synchronisation; fm_pool_trim() releases the cached memory on demand.
void configure_pool(int dev)
{
    static std::mutex mu;
    static bool done[kMaxDevices] = {};
    std::lock_guard<std::mutex> lk(mu);
    if (dev < 0 || dev >= kMaxDevices || done[dev]) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        size_t total = 0;
        cudaDeviceProp prop;
        if (cudaGetDeviceProperties(&prop, dev) == cudaSuccess) total = prop.totalGlobalMem;
        const char *v = getenv("FM_POOL_RELEASE_BYTES");
        uint64_t thr = v && *v ? strtoull(v, nullptr, 10) : (uint64_t)(total / 4 * 3);
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    cudaGetLastError();
    done[dev] = true;
}

// one non-blocking side stream per device for the pipelined sample groups (shared by concurrent
// calls: they are ordered by events, sharing only costs overlap)
cudaError_t side_stream(cudaStream_t *out, int which = 0)  // 0: the groups' second stream, 1: D2H copies
{
    static std::mutex mu;
    static cudaStream_t side[kMaxDevices][2] = {};
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 0 || dev >= kMaxDevices) return cudaErrorInvalidDevice;
    std::lock_guard<std::mutex> lk(mu);
    if (!side[dev][which]) {
        e = cudaStreamCreateWithFlags(&side[dev][which], cudaStreamNonBlocking);
        if (e != cudaSuccess) return e;
    }
    *out = side[dev][which];
    return cudaSuccess;
}

bool is_device_ptr(const void *p)
{
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

int ceil_log2(int64_t n)
{
    int L = 0;
    while ((int64_t(1) << L) < n) L++;
    return L;
}

int64_t env_i64(const char *name, int64_t dflt)
{
    const char *v = getenv(name);
    if (!v || !*v) return dflt;
    return strtoll(v, nullptr, 10);
}

// Device -> host copy in pieces of FM_D2H_CHUNK_MB (64) MiB: on the B200 boxes one 12.8 GB
// cudaMemcpyAsync into page-locked memory ran at 51.6 GB/s, the same bytes in 32-256 MiB copies on
// the same stream at 56 GB/s (scripts/d2h_probe.py); 0: one copy (FM_D2H_CHUNK_KB: tests)
cudaError_t copy_to_host_chunked(void *dst, const void *src, size_t bytes, cudaStream_t st)
{
    const int64_t kb = env_i64("FM_D2H_CHUNK_KB", 0);
    const int64_t mb = kb > 0 ? 1 : env_i64("FM_D2H_CHUNK_MB", 64);
    const size_t chunk = kb > 0 ? (size_t)kb << 10 : mb > 0 ? (size_t)mb << 20 : std::max<size_t>(bytes, 1);
    // a short first piece up to the next 2 MiB boundary of the destination: the pieces of a sample
    // group that starts in the middle of the list (fm_sample_to_host) ran at 50 GB/s from an
    // arbitrary byte offset, 56-57 GB/s from an aligned one (FM_PIPE_TRACE timeline of config 5)
    const size_t al = (size_t)env_i64("FM_D2H_ALIGN", 2 << 20);
    size_t o = 0;
    if (mb > 0 && al > 1 && (al & (al - 1)) == 0) {
        const size_t head = std::min(bytes, (al - ((uintptr_t)dst & (al - 1))) & (al - 1));
        if (head > 0) {
            const cudaError_t e = cudaMemcpyAsync(dst, src, head, cudaMemcpyDeviceToHost, st);
            if (e != cudaSuccess) return e;
            o = head;
        }
    }
    for (; o < bytes; o += chunk) {
        const cudaError_t e = cudaMemcpyAsync((char *)dst + o, (const char *)src + o, std::min(chunk, bytes - o),
                                              cudaMemcpyDeviceToHost, st);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

unsigned grid_for(int64_t n, int threads) { return (unsigned)((n + threads - 1) / threads); }

void plan_release(Plan *p)
{
    if (!p) return;
    if (p->cperm && p->cperm != p->perm) {
        cudaFree(p->cperm);
        cudaFree(p->ckappa);
        cudaFree(p->cy);
        cudaFree(p->cly);
    }
    cudaFree(p->excl);
    cudaFree(p->cand);
    cudaFree(p->perm);
    cudaFree(p->kappa_s);
    cudaFree(p->y_s);
    cudaFree(p->ymax);
    cudaFree(p->ly_s);
    cudaFree(p->rec);
    for (int k = 0; k < 3; k++) {
        cudaFree(p->chunk_seg[k]);
        cudaFree(p->chunk_cap[k]);
    }
    cudaFree(p->dev_flags);
    p->magic = 0;
    delete p;
}

bool plan_live(const void *p)
{
    std::lock_guard<std::mutex> lk(g_mu);
    return g_plans.count(p) != 0;
}

}  // namespace

#define CK(expr, what)                                            \
    do {                                                          \
        cudaError_t e_ = (expr);                                  \
        if (e_ != cudaSuccess) return cuda_fail(e_, what);        \
    } while (0)

extern "C" {

const char *fm_last_error(void) { return g_err.c_str(); }
int32_t fm_abi_version(void) { return FM_ABI_VERSION; }

// a1 + a2 for one node set: validate, key (+ digit histograms), radix sort, rank-order arrays.
// Validation failures are OR-ed into sc->flags and read at the planner's one synchronisation.
struct SortedSet {
    int32_t *perm = nullptr;
    double *kappa = nullptr, *y = nullptr, *ly = nullptr;
};

static fm_status sort_node_set(int model, int64_t n, const double *x, const double *y, PlanScalars *sc, Allocs &tmp,
                               cudaStream_t st, SortedSet &out)
{
    const double *xd = x, *yd = y;
    if (!is_device_ptr(x)) {
        double *t;
        CK(tmp.get(&t, n), "alloc x");
        CK(cudaMemcpyAsync(t, x, sizeof(double) * n, cudaMemcpyHostToDevice, st), "copy x");
        xd = t;
    }
    if (model == FM_ECM && !is_device_ptr(y)) {
        double *t;
        CK(tmp.get(&t, n), "alloc y");
        CK(cudaMemcpyAsync(t, y, sizeof(double) * n, cudaMemcpyHostToDevice, st), "copy y");
        yd = t;
    }
    uint64_t *ka, *kb;
    int32_t *ia, *ib;
    unsigned int *hist;
    CK(tmp.get(&hist, 8 * 256), "alloc hist");
    CK(cudaMemsetAsync(hist, 0, sizeof(unsigned int) * 8 * 256, st), "memset hist");
    CK(tmp.get(&ka, n), "alloc keys");
    CK(tmp.get(&kb, n), "alloc keys");
    CK(tmp.get(&ia, n), "alloc ids");
    CK(tmp.get(&ib, n), "alloc ids");
    count_launch();
    k_validate_key<<<(unsigned)std::min<int64_t>(grid_for(n, 256), 148 * 8), 256, 0, st>>>(model, n, xd, yd, ka, ia,
                                                                                             sc, hist);
    CK(cudaGetLastError(), "k_validate_key");
    const size_t tb = radix_tmp_bytes(n);
    char *work;
    CK(tmp.get(&work, tb), "alloc sort tmp");
    uint64_t *skeys;
    int32_t *perm;
    CK(radix_sort_u64_i32(ka, kb, ia, ib, n, ~0ull /* all 8 digit passes are launched; a constant digit's pass degenerates to a copy on the device */, hist,
                          &skeys, &perm, work, tb, st),
       "radix sort");
    tmp.release(perm);
    out.perm = perm;  // adopted by the plan (freed by plan_release)
    CK(malloc_async_retry((void **)&out.kappa, sizeof(double) * n, st), "alloc kappa_s");
    if (model == FM_ECM) {
        CK(malloc_async_retry((void **)&out.y, sizeof(double) * n, st), "alloc y_s");
        CK(malloc_async_retry((void **)&out.ly, sizeof(double) * n, st), "alloc ly_s");
    }
    count_launch();
    k_gather_sorted<<<grid_for(n, 256), 256, 0, st>>>(model, n, skeys, yd, out.perm, out.kappa, out.y, out.ly);
    CK(cudaGetLastError(), "k_gather_sorted");
    return FM_OK;
}

static fm_status sort_plan_impl(fm_model model, fm_graph kind, int64_t n1, const double *x1, const double *y1,
                                int64_t n2, const double *x2, const double *y2, int64_t seg_target,
                                void *cuda_stream, fm_plan **plan_out)
{
    NvtxRange nvtx_("fm_sort_plan (a1-a4)");
    if (!plan_out) return fail(FM_ERR_INVALID, "plan_out is NULL");
    *plan_out = nullptr;
    if (model != FM_UBCM && model != FM_ECM) return fail(FM_ERR_INVALID, "unknown model %d", (int)model);
    if (kind != FM_UNDIRECTED && kind != FM_BIPARTITE && kind != FM_DIRECTED)
        return fail(FM_ERR_INVALID, "unknown graph kind %d", (int)kind);
    if (kind == FM_UNDIRECTED) {
        n2 = n1;
        x2 = x1;
        y2 = y1;
    }
    const int64_t nmin = kind == FM_UNDIRECTED ? 2 : 1;
    if (n1 < nmin || n1 > INT32_MAX) return fail(FM_ERR_INVALID, "n = %lld outside [%lld, 2^31-1]", (long long)n1,
                                                  (long long)nmin);
    if (n2 < 1 || n2 > INT32_MAX) return fail(FM_ERR_INVALID, "n_minus = %lld outside [1, 2^31-1]", (long long)n2);
    if (kind == FM_DIRECTED && n1 != n2) return fail(FM_ERR_INVALID, "directed: out and in sets differ in size");
    if (!x1 || !x2) return fail(FM_ERR_INVALID, "x is NULL");
    if (model == FM_ECM && (!y1 || !y2)) return fail(FM_ERR_INVALID, "ECM needs y");
    if (model == FM_UBCM && (y1 || (kind != FM_UNDIRECTED && y2))) return fail(FM_ERR_INVALID, "UBCM takes no y");
    if (seg_target == 0) seg_target = 256;
    if (seg_target < 8 || seg_target > (int64_t(1) << 40))
        return fail(FM_ERR_INVALID, "seg_target %lld outside [8, 2^40]", (long long)seg_target);

    cudaStream_t st = (cudaStream_t)cuda_stream;
    int dev = 0;
    CK(cudaGetDevice(&dev), "cudaGetDevice");
    configure_pool(dev);
    Allocs tmp(st);
    PhaseTimer timer;
    timer.begin(kPhasePlan, st);

    PlanScalars *sc;
    CK(tmp.get(&sc, 1), "alloc scalars");
    PlanScalars h_sc;
    memset(&h_sc, 0, sizeof(h_sc));
    h_sc.key_and = ~0ull;
    CK(cudaMemcpyAsync(sc, &h_sc, sizeof(h_sc), cudaMemcpyHostToDevice, st), "init scalars");

    Plan *p = new Plan();
    memset(p, 0, sizeof(Plan));
    p->magic = kPlanMagic;
    p->model = (int)model;
    p->kind = (int)kind;
    p->n = n1;
    p->nc = n2;
    p->S = seg_target;
    p->device = dev;
    p->out_ratio = 1.03;
    struct PlanGuard {
        Plan *p;
        ~PlanGuard() { if (p) plan_release(p); }
    } guard{p};

    // ---- a1 + a2: the row set (and the candidate set) ----
    {
        SortedSet r;
        fm_status s = sort_node_set((int)model, n1, x1, y1, sc, tmp, st, r);
        if (s != FM_OK) return s;
        p->perm = r.perm;
        p->kappa_s = r.kappa;
        p->y_s = r.y;
        p->ly_s = r.ly;
    }
    if (kind == FM_UNDIRECTED) {
        p->cperm = p->perm;
        p->ckappa = p->kappa_s;
        p->cy = p->y_s;
        p->cly = p->ly_s;
    } else {
        SortedSet c;
        fm_status s = sort_node_set((int)model, n2, x2, y2, sc, tmp, st, c);
        if (s != FM_OK) return s;
        p->cperm = c.perm;
        p->ckappa = c.kappa;
        p->cy = c.y;
        p->cly = c.ly;
    }
    const int64_t nc = n2;
    const size_t sb = scan_tmp_bytes(std::max(n1, nc) + 1) + 256;
    char *work;
    CK(tmp.get(&work, sb), "alloc scan tmp");
    if (kind == FM_DIRECTED) {
        int32_t *crank;
        CK(tmp.get(&crank, nc), "alloc crank");
        CK(malloc_async_retry((void **)&p->excl, sizeof(int32_t) * n1, st), "alloc excl");
        count_launch();
        k_rank_of<<<grid_for(nc, 256), 256, 0, st>>>(nc, p->cperm, crank);
        count_launch();
        k_excl<<<grid_for(n1, 256), 256, 0, st>>>(n1, p->perm, crank, p->excl);
        CK(cudaGetLastError(), "k_excl");
    }

    // packed gather records: ECM always (32 B); UBCM one 16-byte (kappa, id) record per candidate at
    // every size (config 2 sampler -3 %, config 5 -4 % against two arrays, once the record's dead
    // word no longer stalled the gather; FM_UBCM_CAND_MIN raises the threshold for A/B runs)
    // (not where the sampler takes the rank-out path, N >= FM_UBCM_RANK_OUT_MIN: it gathers kappa
    // alone there; the statistics mode and overflow re-runs then gather from the two arrays --
    // config 4: 160 MB and a 44 us pass less per plan)
    const bool want_cand =
        model == FM_ECM || (n2 >= env_i64("FM_UBCM_CAND_MIN", 0) && n2 < env_i64("FM_UBCM_RANK_OUT_MIN", int64_t(1) << 21));
    if (want_cand)
        CK(malloc_async_retry((void **)&p->cand, sizeof(double2) * kCandWords(model) * std::max<int64_t>(n2, 1), st),
           "alloc cand");
    if (want_cand && n2 > 0) {
        count_launch();
        k_pack_cand<<<grid_for(n2, 256), 256, 0, st>>>((int)model, n2, p->ckappa, p->cperm, p->cy, p->cly, p->cand);
        CK(cudaGetLastError(), "k_pack_cand");
    }

    // ---- a3: suffix max of the candidates' y (beta_min) ----
    if (model == FM_ECM) {
        CK(malloc_async_retry((void **)&p->ymax, sizeof(double) * (nc + 1), st), "alloc ymax");
        CK(suffix_max_f64(p->cy, p->ymax, nc, work, sb, st), "suffix max");
    }

    // ---- a4: planner ----
    uint64_t *P;
    RowInfo *rows;
    int64_t *row_m;
    CK(tmp.get(&P, nc + 1), "alloc P");
    CK(tmp.get(&rows, n1), "alloc rows");
    CK(tmp.get(&row_m, n1 + 1), "alloc row_m");
    count_launch();
    k_kfx<<<grid_for(nc, 256), 256, 0, st>>>(nc, ceil_log2(nc), p->ckappa, sc, P);
    CK(cudaGetLastError(), "k_kfx");
    CK(scan_exclusive_u64(P, P, nc, work, sb, st), "scan P");
    count_launch();
    k_rows<<<grid_for(n1, 256), 256, 0, st>>>((int)model, (int)kind, n1, nc, seg_target, p->kappa_s, p->y_s,
                                              p->ckappa, p->ymax, P, sc, rows, row_m);
    CK(cudaGetLastError(), "k_rows");
    CK(scan_exclusive_i64(row_m, row_m, n1, work, sb, st), "scan rows");
    int64_t n_seg = 0;
    CK(cudaMemcpyAsync(&h_sc, sc, sizeof(h_sc), cudaMemcpyDeviceToHost, st), "read scalars");
    CK(cudaMemcpyAsync(&n_seg, row_m + n1, sizeof(int64_t), cudaMemcpyDeviceToHost, st), "read n_seg");
    CK(cudaStreamSynchronize(st), "sync (rows)");
    if (h_sc.flags & kErrInvalid)
        return fail(FM_ERR_INVALID, "invalid fitness: x must be finite >= 0, y in [0,1), kappa_max^4 finite");
    // the sampler indexes segments with 32-bit integers
    if (n_seg > INT32_MAX)
        return fail(FM_ERR_INVALID, "plan has %lld segments (> 2^31-1): raise seg_target", (long long)n_seg);
    p->F = h_sc.F;
    p->n_seg = n_seg;
    p->wmax = h_sc.wmax;
    p->est_draws = h_sc.total_work >> kG;
    // row_m now holds row_seg (exclusive prefix of the per-row segment counts, n+1 entries)
    int64_t *seg_work;
    CK(tmp.get(&seg_work, n_seg + 1), "alloc seg_work");
    CK(malloc_async_retry((void **)&p->rec, (size_t)kRecStride(model) * std::max<int64_t>(n_seg, 1), st), "alloc rec");
    if (n_seg > 0) {
        // segment -> row map for large plans: exclusive scan of the row-start flags (small plans:
        // a per-block search in k_emit, two launches fewer)
        int64_t *seg_row_x = nullptr;
        if (n_seg >= (int64_t(1) << 20)) {
            CK(tmp.get(&seg_row_x, n_seg + 1), "alloc seg rows");
            CK(cudaMemsetAsync(seg_row_x, 0, sizeof(int64_t) * (n_seg + 1), st), "memset seg rows");
            count_launch();
            k_row_starts<<<grid_for(n1, 256), 256, 0, st>>>(n1, row_m, seg_row_x);
            const size_t rb = scan_tmp_bytes(n_seg + 1);
            char *work_r;
            CK(tmp.get(&work_r, rb), "alloc scan tmp");
            CK(scan_exclusive_i64(seg_row_x, seg_row_x, n_seg, work_r, rb, st), "scan row starts");
        }
        count_launch();
        k_emit<<<grid_for(n_seg, 256), 256, 0, st>>>((int)model, (int)kind, n1, nc, n_seg, p->kappa_s, p->y_s,
                                                     p->ly_s, p->perm, p->excl, p->ckappa, p->ymax, P, sc, rows,
                                                     row_m, seg_row_x, p->rec, seg_work);
        CK(cudaGetLastError(), "k_emit");
        // test hook: a plan whose initial bounds are too small (p > q at the first candidates), for
        // the FM_DEBUG_CHECKS contract check (FM_ERR_BOUND)
        if (env_i64("FM_DEBUG_BAD_BOUND", 0)) {
            count_launch();
            k_debug_scale_bound<<<grid_for(n_seg, 256), 256, 0, st>>>(p->rec, n_seg, kRecStride(model), 1e-3);
            CK(cudaGetLastError(), "k_debug_scale_bound");
        }
    }
    {
        const size_t wb = scan_tmp_bytes(n_seg + 1);
        char *work2;
        CK(tmp.get(&work2, wb), "alloc scan tmp");
        CK(scan_exclusive_i64(seg_work, seg_work, n_seg, work2, wb, st), "scan work");
    }

    // ---- lane-chunking (never changes results): coarse, fine and big (FM_CHUNK_BIG_DRAWS=0: none) ----
    const int64_t total = h_sc.total_work;
    const int64_t lane_draws[3] = {std::max<int64_t>(1, env_i64("FM_CHUNK_LANE_DRAWS", 256)),
                                   std::max<int64_t>(1, env_i64("FM_CHUNK_FINE_DRAWS", 64)),
                                   std::max<int64_t>(0, env_i64("FM_CHUNK_BIG_DRAWS", 512))};
    const int64_t cap_override = env_i64("FM_DEBUG_SCRATCH_CAP", 0);  // test hook: force re-runs
    p->slots_aligned = true;
    p->cap_per_sample = 0;
    for (int k = 0; k < 3; k++) {
        if (lane_draws[k] == 0) {  // (no big chunking)
            p->n_chunks[k] = 0;
            p->chunk_target[k] = 0;
            continue;
        }
        const int64_t target = lane_draws[k] * kUnit;
        p->chunk_target[k] = target;
        const int64_t nch = std::max<int64_t>(1, (total + target - 1) / target);
        p->n_chunks[k] = nch;
        CK(malloc_async_retry((void **)&p->chunk_seg[k], sizeof(int64_t) * (nch + 1), st), "alloc chunks");
        CK(malloc_async_retry((void **)&p->chunk_cap[k], sizeof(int64_t) * (nch + 1), st), "alloc chunk caps");
        count_launch();
        k_chunks<<<grid_for(nch, 256), 256, 0, st>>>(n_seg, nch, target, seg_work, p->chunk_seg[k], p->chunk_cap[k]);
        CK(cudaGetLastError(), "k_chunks");
        const size_t cb = scan_tmp_bytes(nch + 1);
        char *work3;
        CK(tmp.get(&work3, cb), "alloc scan tmp");
        CK(scan_exclusive_i64(p->chunk_cap[k], p->chunk_cap[k], nch, work3, cb, st), "scan chunk caps");
        // sum over chunks of floor(1.25 w_c / 2^G) + 16 <= floor(1.25 total / 2^G) + 16 n_chunks
        // sum over chunks of (floor(1.25 w_c / 2^G) + 16 rounded up to 4) <= floor(1.25 total / 2^G) + 19 n_chunks
        int64_t cps = ((((total + total / 4) >> kG) + 20 * nch + 16) + 3) & ~int64_t(3);
        if (cap_override > 0) {
            count_launch();
            k_fill_caps<<<grid_for(nch + 1, 256), 256, 0, st>>>(p->chunk_cap[k], nch, cap_override);
            CK(cudaGetLastError(), "k_fill_caps");
            cps = cap_override * nch;
            p->slots_aligned = cap_override % 4 == 0;
        }
        p->cap_per_sample = std::max(p->cap_per_sample, cps);
    }

    // the cut invariant (kErrState, impossible for S >= 8) is checked lazily by fm_sample_*: the
    // plan keeps the flag word on the device and returns without a second synchronisation
    CK(malloc_async_retry((void **)&p->dev_flags, sizeof(unsigned int), st), "alloc flags");
    CK(cudaMemcpyAsync(p->dev_flags, &sc->flags, sizeof(unsigned int), cudaMemcpyDeviceToDevice, st), "copy flags");
    timer.end(st);

    guard.p = nullptr;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        g_plans.insert(p);
    }
    *plan_out = (fm_plan *)p;
    return FM_OK;
}

fm_status fm_sort_plan(fm_model model, int64_t n, const double *x, const double *y, int64_t seg_target,
                       void *cuda_stream, fm_plan **plan_out)
{
    return sort_plan_impl(model, FM_UNDIRECTED, n, x, y, n, x, y, seg_target, cuda_stream, plan_out);
}

fm_status fm_sort_plan_bipartite(fm_model model, fm_graph kind, int64_t n_plus, const double *x_plus,
                                 const double *y_plus, int64_t n_minus, const double *x_minus, const double *y_minus,
                                 int64_t seg_target, void *cuda_stream, fm_plan **plan_out)
{
    if (kind == FM_UNDIRECTED) {
        if (plan_out) *plan_out = nullptr;
        return fail(FM_ERR_INVALID, "fm_sort_plan_bipartite needs FM_BIPARTITE or FM_DIRECTED");
    }
    return sort_plan_impl(model, kind, n_plus, x_plus, y_plus, n_minus, x_minus, y_minus, seg_target, cuda_stream,
                          plan_out);
}

// task space of a sample group of n_samples: its last K_fine samples use the fine chunks, the K_mid
// before them the coarse ones, the rest (the bulk of a large call) the big ones.  The call's last
// group: K_fine covers ~FM_TAIL_FACTOR times the work the resident lanes hold in coarse tasks (so
// the end of the queue is short tasks), K_mid likewise for big tasks.
static TaskMap make_task_map(const Plan *p, int64_t n_samples, int64_t K_fine, int64_t K_mid, int64_t *n_tasks)
{
    TaskMap tm;
    const int plan_k[kRanges] = {2, 0, 1};  // range -> the plan's chunking (big, coarse, fine)
    for (int r = 0; r < kRanges; r++) {
        const int k = plan_k[r];
        tm.seg[r] = p->chunk_seg[k];
        tm.cap[r] = p->chunk_cap[k];
        tm.n_chunks[r] = p->n_chunks[k];
        tm.inv_chunks[r] = p->n_chunks[k] > 0 ? 1.0 / (double)p->n_chunks[k] : 0.0;
    }
    tm.cap_per_sample = p->cap_per_sample;
    K_fine = std::max<int64_t>(0, std::min(K_fine, n_samples));
    K_mid = std::max<int64_t>(0, std::min(K_mid, n_samples - K_fine));
    if (p->n_chunks[2] == 0) K_mid = n_samples - K_fine;  // no big chunking
    const int64_t n_big = n_samples - K_fine - K_mid;
    tm.s0[0] = 0;
    tm.s0[1] = n_big;
    tm.s0[2] = n_big + K_mid;
    tm.t0[0] = 0;
    tm.t0[1] = n_big * tm.n_chunks[0];
    tm.t0[2] = tm.t0[1] + K_mid * tm.n_chunks[1];
    *n_tasks = tm.t0[2] + K_fine * tm.n_chunks[2];
    return tm;
}

// samples at the end of a call that do not use the chunking `k` of the plan (0 coarse: they use
// the fine chunks; 2 big: they use the coarse or fine ones): ~FM_TAIL_FACTOR times the work the
// resident lanes hold in tasks of that chunking
static int64_t tail_samples(const Plan *p, int k)
{
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const double lanes = (double)sms * 768.0;
    // (big tasks: a warp claims a queue batch at a time -- 64 entries then: two long tasks per lane --, so the work
    // behind the big range must be larger: with factor 2 configs 3 and 4 lost 5-14 %; 3 against 4:
    // config 5 -0.45 %, config 4 -0.6 %, configs 2 and 3 unchanged)
    const int64_t factor = k == 2 ? env_i64("FM_TAIL_FACTOR_BIG", 3) : env_i64("FM_TAIL_FACTOR", 2);
    const double tail = (double)factor * lanes * (double)(p->chunk_target[k] >> kG);
    const double per = std::max<double>(1.0, (double)p->est_draws);
    return (int64_t)std::ceil(tail / per);
}


// host destination of fm_sample_to_host: the final list is copied to the host group by group while
// the later groups are still being sampled (cap: capacity in edges; w may be NULL)
struct HostDst {
    int32_t *e = nullptr, *w = nullptr;
    int64_t cap = 0;
};

static fm_status sample_impl(int model, const fm_plan *plan_, uint64_t seed, int64_t first_sample, int64_t n_samples,
                             uint32_t flags, void *cuda_stream, fm_edges *out, const HostDst *host = nullptr)
{
    NvtxRange nvtx_(model == FM_UBCM ? "fm_sample_ubcm (a5-a6)" : "fm_sample_ecm (a5-a6)");
    if (!out) return fail(FM_ERR_INVALID, "out is NULL");
    memset(out, 0, sizeof(*out));
    if (!plan_ || !plan_live(plan_)) return fail(FM_ERR_STATE, "not a live fm_plan");
    const Plan *p = (const Plan *)plan_;
    if (p->model != model)
        return fail(FM_ERR_STATE, "plan model %s used with fm_sample_%s", p->model == FM_UBCM ? "UBCM" : "ECM",
                    model == FM_UBCM ? "ubcm" : "ecm");
    if (n_samples < 0 || first_sample < 0 || first_sample + n_samples > (int64_t(1) << 32))
        return fail(FM_ERR_INVALID, "sample range [%lld, +%lld) outside [0, 2^32)", (long long)first_sample,
                    (long long)n_samples);
    cudaStream_t st = (cudaStream_t)cuda_stream;
    Allocs tmp(st);

    int64_t *offsets_h = (int64_t *)calloc((size_t)n_samples + 1, sizeof(int64_t));
    Owner *own = new Owner();
    memset(own, 0, sizeof(Owner));
    own->magic = kOwnerMagic;
    own->offsets_host = offsets_h;
    own->stream = st;
    struct OwnGuard {
        Owner *o;
        ~OwnGuard()
        {
            if (o) {
                free(o->offsets_host);
                if (o->edges) cudaFreeAsync(o->edges, o->stream);
                if (o->weights) cudaFreeAsync(o->weights, o->stream);
                delete o;
            }
        }
    } og{own};
    if (!offsets_h) return fail(FM_ERR_NOMEM, "host offsets");

    // ---- the call = G SAMPLE GROUPS (default G = 1; FM_SAMPLE_GROUPS) ----
    // Group g (consecutive samples) runs sampler -> count scan -> offsets -> overflow list ->
    // compaction on stream g & 1 (the caller's stream and one side stream), so the small-footprint
    // compaction of group g can run next to the persistent sampler of group g + 1 on every SM.
    // Scratch slots are double-buffered over the groups (2/G of the per-call scratch).  The groups'
    // edges are consecutive in the final list: group g's base is the device-side running total
    // gbase[g].  Results do not depend on G.  One host synchronisation at the end of the call.
    // (Measured: the overlap works, but every extra sampler launch pays its own end-of-launch tail
    // and the sampler slows next to the compaction's traffic; one group is the fastest.)
    struct Hdr {
        unsigned long long counters[3];
        unsigned int flags;
        unsigned int pad;
        unsigned long long n_overflow;
        unsigned long long task_counter;
        unsigned long long spill_counter;
    };
    struct Group {
        int64_t s0 = 0, R = 0, n_tasks = 0;
        TaskMap tm;
        int64_t *counts = nullptr, *dest = nullptr, *spill_off = nullptr, *ovl = nullptr;
        SampleArgs a;
    };
    const bool ecm_rec = model == FM_ECM && p->slots_aligned && env_i64("FM_SCRATCH_BUF4", 1) != 0;
    const bool buf4 = p->slots_aligned && env_i64("FM_SCRATCH_BUF4", 1) != 0;
    // v3 fused write (UBCM, opt-in FM_FUSE_WRITE=1): one block per SM whose warp 0
    // copies the block's finished task batches into the final list.  Measured slower than the
    // compaction pass (the copier warp is issue-starved next to 23 sampler warps); one group only.
    const bool rank_out = model == FM_UBCM && p->nc >= env_i64("FM_UBCM_RANK_OUT_MIN", int64_t(1) << 21);
    // (undirected plans only: the fused kernel is instantiated for (min id, max id) pairs; an ordered
    // -- bipartite / directed -- plan with the option set used to skip the compaction and still
    // launch the plain sampler: found by tests/test_gpu_fuzz.py)
    const bool fuse = model == FM_UBCM && p->kind == FM_UNDIRECTED && p->slots_aligned &&
                      env_i64("FM_FUSE_WRITE", 0) != 0 && (!rank_out || env_i64("FM_FUSE_RANKOUT", 0) != 0);
    // the small-footprint compaction needs 32-byte-aligned slots holding pairs (UBCM) or records
    // (ECM) and a warp's 32 tasks spanning < 2^31 output positions (slot <= ~1.25 (chunk + segment))
    const bool small_compact = buf4 && (model == FM_UBCM || ecm_rec) && (p->wmax >> kG) < (int64_t(1) << 22) &&
                               env_i64("FM_COMPACT_SMALL", 1) != 0;
    // group count: FM_SAMPLE_GROUPS (default 1).  Measured on the B200: the
    // co-resident compaction does hide under the next group's sampler, but every extra sampler
    // launch pays its own end-of-launch tail (~0.4 ms on config 5: a block stays resident until its
    // slowest lane ends, so the next group's blocks cannot move in early) and the latency-bound
    // sampler slows by ~1.5 ms per 12.8 GB of compaction traffic next to it, so one group is the
    // fastest on all five configs; the option stays for callers short of memory (scratch is 2/G).
    int64_t G = 1;
    if (n_samples > 1 && small_compact && !fuse) {
        // (a host destination: one group per ~0.8 GB of expected list, 4 to 16 of them from 256 MB --
        // the call is bound by the D2H copies (8 B per edge over PCIe, ~55 GB/s), which hide the
        // groups' tails; with the copies in aligned pieces: config 5 236 -> 233 ms with 16 groups
        // instead of 6 (32: 232), configs 2-4 -2 % with 4 groups instead of 1 (2 groups: +-0))
        int64_t hg = 1;
        if (host && host->e) {
            const double bytes = 8.0 * (double)std::max<int64_t>(1, p->est_draws - p->n_seg) * (double)n_samples;
            const int64_t auto_g = bytes < 256e6 ? 1 : std::min<int64_t>(16, std::max<int64_t>(4, (int64_t)(bytes / 0.8e9)));
            hg = env_i64("FM_HOST_GROUPS", auto_g);
        }
        const int64_t forced = env_i64("FM_SAMPLE_GROUPS", std::max<int64_t>(1, hg));
        if (forced > 0) G = forced;
        G = std::min<int64_t>(G, n_samples);
    }
    // samples of the last K use the fine chunks (short end-of-queue tasks): the call's last group only
    const int64_t K_fine = tail_samples(p, 0), K_big_tail = p->n_chunks[2] > 0 ? tail_samples(p, 2) : 0;
    std::vector<Group> grp((size_t)G);
    int64_t n_tasks = 0, max_R = 0, max_tasks = 0;
    for (int64_t g = 0; g < G; g++) {
        Group &q = grp[(size_t)g];
        q.s0 = n_samples * g / G;
        q.R = n_samples * (g + 1) / G - q.s0;
        // (the call's last group ends with coarse, then fine tasks; the groups before it run into
        // their successors, no tail to shorten)
        const int64_t kf = g == G - 1 ? std::min(K_fine, q.R) : 0;
        const int64_t km = g == G - 1 ? std::max<int64_t>(0, std::min(K_big_tail, q.R) - kf) : 0;
        q.tm = make_task_map(p, q.R, kf, km, &q.n_tasks);
        n_tasks += q.n_tasks;
        max_R = std::max(max_R, q.R);
        max_tasks = std::max(max_tasks, q.n_tasks);
    }
    std::vector<Hdr> h((size_t)G);
    std::vector<int64_t> gbase_h((size_t)G + 1, 0);
    memset(h.data(), 0, sizeof(Hdr) * (size_t)G);
    if (n_tasks > 0) {
        // ---- streams: groups alternate between the caller's stream and the device's side stream ----
        cudaStream_t side = st;
        std::vector<cudaEvent_t> evs;
        struct EvGuard {
            std::vector<cudaEvent_t> &v;
            ~EvGuard()
            {
                for (cudaEvent_t e : v)
                    if (e) cudaEventDestroy(e);
            }
        } evg{evs};
        auto new_event = [&](cudaEvent_t *e, bool timing) -> cudaError_t {
            cudaError_t r = cudaEventCreateWithFlags(e, timing ? cudaEventDefault : cudaEventDisableTiming);
            if (r == cudaSuccess) evs.push_back(*e);
            return r;
        };
        if (G > 1) CK(side_stream(&side), "side stream");
        auto stream_of = [&](int64_t g) { return (g & 1) ? side : st; };
        // host destination (fm_sample_*_host): a copy stream and pinned words for the groups' bases
        const bool to_host = host && host->e;
        cudaStream_t copy_st = st;
        int64_t *pin = nullptr, *pin_dev = nullptr;
        if (to_host) {
            CK(side_stream(&copy_st, 1), "copy stream");
            // (one small mapped allocation per host thread and device, kept: cudaHostAlloc /
            // cudaFreeHost per call cost 15-200 ms next to gigabytes of page-locked user buffers)
            struct PinWords {
                int64_t *p = nullptr;
                size_t n = 0;
                int dev = -1;
            };
            thread_local PinWords pw;
            int dev = 0;
            CK(cudaGetDevice(&dev), "device");
            if (pw.n < (size_t)G + 1 || pw.dev != dev) {
                if (pw.p) cudaFreeHost(pw.p);
                pw.p = nullptr;
                pw.n = 0;
                const size_t want = std::max<size_t>((size_t)G + 1, 64);
                CK(cudaHostAlloc((void **)&pw.p, sizeof(int64_t) * want, cudaHostAllocMapped), "pinned words");
                pw.n = want;
                pw.dev = dev;
            }
            pin = pw.p;
            CK(cudaHostGetDevicePointer((void **)&pin_dev, pin, 0), "mapped words");
        }
        std::vector<char> pin_empty((size_t)G, 0);
        bool host_done = false;  // the list has been copied to the host destination completely

        // ---- device memory (all from the caller's stream, before the fork) ----
        const int64_t slots = max_R * p->cap_per_sample;
        const int64_t spill_cap = slots / 32 + 65536;
        const int64_t slot_words = ecm_rec ? 2 * slots : slots, wslots = ecm_rec ? 0 : slots;
        const int nbuf = G > 1 ? 2 : 1;
        int2 *se[2] = {nullptr, nullptr};
        int32_t *sw[2] = {nullptr, nullptr};
        // (look-back words of every group's count scan: one array, cleared once per pass)
        const size_t stb = (scan_tmp_bytes(max_tasks + 1) + 255) & ~(size_t)255;
        char *scan_tmp;
        CK(tmp.get(&scan_tmp, stb * (size_t)G), "alloc scan tmp");
        for (int b = 0; b < nbuf; b++) {
            CK(tmp.get(&se[b], slot_words + spill_cap), "alloc scratch edges");
            if (model == FM_ECM) CK(tmp.get(&sw[b], wslots + spill_cap), "alloc scratch weights");
        }
        Hdr *hd;
        int64_t *offs_d, *gbase;
        CK(tmp.get(&hd, (size_t)G), "alloc hdr");
        CK(tmp.get(&offs_d, n_samples + 1), "alloc offsets");
        CK(tmp.get(&gbase, (size_t)G + 1), "alloc group bases");
        for (int64_t g = 0; g < G; g++) {
            Group &q = grp[(size_t)g];
            CK(tmp.get(&q.spill_off, q.n_tasks), "alloc spill offsets");
            CK(tmp.get(&q.counts, q.n_tasks + 1), "alloc counts");
            CK(tmp.get(&q.dest, q.n_tasks + 1), "alloc dest");
            CK(tmp.get(&q.ovl, q.n_tasks), "alloc overflow list");
        }
        // fused-write bookkeeping: one look-back status word per queue batch of kQueueBatch tasks
        const int64_t n_batches = (n_tasks + kQueueBatch - 1) / kQueueBatch;
        unsigned long long *grp_state = nullptr;
        if (fuse) CK(tmp.get(&grp_state, n_batches), "alloc batch states");

        // capacity of the final list: the plan's hint (see the end of this block), at most the scratch's
        int64_t out_cap = n_samples * p->cap_per_sample + (n_samples * p->cap_per_sample / 32 + 65536);
        {
            double ratio;
            {
                std::lock_guard<std::mutex> lk(g_mu);
                ratio = p->out_ratio;
            }
            const double per = (double)std::max<int64_t>(1, p->est_draws - p->n_seg);
            const double est = ratio * per * (double)n_samples + 8.0 * std::sqrt(per * (double)n_samples) + 4096.0;
            if (est < (double)out_cap) out_cap = (int64_t)est;
        }
        auto alloc_out = [&](int64_t cap) -> cudaError_t {
            cudaError_t e = malloc_async_retry(&own->edges, sizeof(int2) * std::max<int64_t>(cap, 1), st);
            if (e == cudaSuccess && model == FM_ECM)
                e = malloc_async_retry(&own->weights, sizeof(int32_t) * std::max<int64_t>(cap, 1), st);
            return e;
        };
        auto free_out = [&]() {
            if (own->edges) cudaFreeAsync(own->edges, st);
            if (own->weights) cudaFreeAsync(own->weights, st);
            own->edges = own->weights = nullptr;
        };

        // ---- per-group sampler arguments ----
        for (int64_t g = 0; g < G; g++) {
            Group &q = grp[(size_t)g];
            const int b = nbuf == 2 ? (int)(g & 1) : 0;
            SampleArgs &a = q.a;
            memset(&a, 0, sizeof(a));
            a.rec = p->rec;
            a.kappa_s = p->ckappa;  // candidates (R16): the - set, or the rows themselves
            a.y_s = p->cy;
            a.ly_s = p->cly;
            a.perm = p->cperm;
            a.cand = p->cand;
            a.ymax_c = (model == FM_ECM && (flags & FM_SAMPLE_BETA_REFRESH)) ? p->ymax : nullptr;
            a.ordered = p->kind != FM_UNDIRECTED;
            a.buf4 = buf4;
            // UBCM with a large candidate set (the kappa array no longer L2-resident): the sampler
            // gathers kappa only and the compaction maps candidate ranks to ids (sampler kernel
            // -14 %, compaction +0.55 ms on config 4: a net gain; at N <= 1e6 the compaction's extra
            // gathers cost more than the sampler saves)
            a.rank_out = rank_out;
            // large candidate sets (configs 4, 5): the samples of a lane-chunk run back to back, so its
            // segment records come from DRAM once per launch instead of once per sample (sampler
            // -2.2 % on config 4, -1.9 % on config 5; +1 % (UBCM) / +2.6 % (ECM) at N = 1e5, where
            // the records stay in L2 anyway: off there).  Results do not depend on it.
            // (the fused copy needs batches of consecutive canonical tasks: sample-major queue)
            // chunk-major in the fine range at every N (FM_INTERLEAVE_FINE=0: off), so the last
            // samples' hub-row chunks (sequential chains of up to S draws) start before their light rows
            a.il_s[0] = a.il_s[1] = a.il_s[2] = 0;
            if (!fuse) {
                const bool all = p->nc >= env_i64("FM_INTERLEAVE_MIN", int64_t(1) << 19);
                const bool fine = env_i64("FM_INTERLEAVE_FINE", 1) != 0;
                for (int r = 0; r < kRanges; r++) {
                    if (!all && !(fine && r == 2)) continue;
                    a.il_s[r] = (r + 1 < kRanges ? q.tm.s0[r + 1] : q.R) - q.tm.s0[r];  // (0: empty range, never indexed)
                }
            }
            a.tm = q.tm;
            a.key = philox_key(seed);
            a.lc = log_consts();
            a.first_sample = (uint32_t)(first_sample + q.s0);
            a.n_tasks = q.n_tasks;
            a.task_counter = &hd[g].task_counter;
            a.edges = se[b];
            a.weights = sw[b];
            a.counts = q.counts;
            a.spill_e = se[b] + slot_words;
            a.spill_w = sw[b] ? sw[b] + wslots : nullptr;
            a.spill_counter = &hd[g].spill_counter;
            a.spill_cap = spill_cap;
            a.spill_off = q.spill_off;
            a.counters = hd[g].counters;
            a.flags = &hd[g].flags;
            a.check = env_i64("FM_DEBUG_CHECKS", 0) != 0;
            a.counters_zeroed = 1;  // (hd is cleared at the start of every pass)
            if (fuse) {
                a.fuse = 1;
                a.n_groups = n_batches;
                a.grp_state = grp_state;
                a.dest = q.dest;
                a.discard = env_i64("FM_DISCARD", 1) != 0;
                a.rank_map = a.rank_out ? p->cperm : nullptr;
            }
        }
        // compaction of group g into the list of capacity `cap` (+ the deterministic re-run of its
        // overflowed tasks straight into the list, after the host knows the group bases)
        // the TMA-staged small-footprint kernel is also the faster one alone (config 5: 4.07 vs 4.31 ms,
        // config 2: 0.30 vs 0.34 ms) except with the rank -> id mapping of the rank-out path (its
        // gathers sit in the store loop: config 4 2.5 vs 1.07 ms), where only the groups that run next
        // to a sampler use it; FM_COMPACT_SMALL: 0 never, 2 always
        auto use_small = [&](int64_t g) {
            const int64_t mode = env_i64("FM_COMPACT_SMALL", 1);
            return small_compact && (mode > 1 || g < G - 1 || !rank_out);
        };
        auto compact_group = [&](int64_t g, int64_t cap, cudaStream_t s) -> cudaError_t {
            Group &q = grp[(size_t)g];
            if (q.n_tasks == 0) return cudaSuccess;
            return launch_compact(cap, q.n_tasks, q.tm, q.counts, q.dest, q.spill_off, q.a.edges, q.a.weights, q.a.spill_e,
                                  q.a.spill_w, (int2 *)own->edges, (int32_t *)own->weights,
                                  q.a.rank_out ? p->cperm : nullptr, q.a.ordered, ecm_rec ? 1 : 0,
                                  use_small(g) ? 1 : 0, gbase + g, s);
        };
        auto rerun_group = [&](int64_t g, int64_t cap) -> cudaError_t {
            Group &q = grp[(size_t)g];
            SampleArgs r = q.a;
            r.fuse = 0;
            r.counters_zeroed = 0;
            r.n_tasks_dev = &hd[g].n_overflow;
            r.task_list = q.ovl;
            r.rerun_base = q.dest;
            r.out_base = gbase_h[(size_t)g];
            r.out_cap = cap;
            r.edges = (int2 *)own->edges;
            r.weights = (int32_t *)own->weights;
            return launch_sample(model, r, st);
        };
        unsigned int plan_flags = 0;
        // one pass of the call: every group queued, one synchronisation at the end
        auto run_pass = [&](int64_t cap) -> fm_status {
            CK(alloc_out(cap), "alloc edges");
            CK(cudaMemsetAsync(hd, 0, sizeof(Hdr) * (size_t)G, st), "memset hdr");
            CK(cudaMemsetAsync(gbase, 0, sizeof(int64_t) * ((size_t)G + 1), st), "memset group bases");
            CK(cudaMemsetAsync(scan_tmp, 0, stb * (size_t)G, st), "memset scan words");
            if (fuse) CK(cudaMemsetAsync(grp_state, 0, sizeof(unsigned long long) * n_batches, st), "memset batch states");
            const bool timing = g_timing.load();
            cudaEvent_t t_a = nullptr, t_b = nullptr, t_c = nullptr, ev_prev = nullptr;
            std::vector<cudaEvent_t> ev_off((size_t)G, nullptr), ev_done((size_t)G, nullptr);
            host_done = false;
            if (to_host) pin[0] = 0;
            if (timing) {
                CK(new_event(&t_a, true), "event");
                CK(new_event(&t_b, true), "event");
                CK(new_event(&t_c, true), "event");
                CK(cudaEventRecord(t_a, st), "event record");
            }
            if (G > 1) {  // fork
                cudaEvent_t ev;
                CK(new_event(&ev, false), "event");
                CK(cudaEventRecord(ev, st), "event record");
                CK(cudaStreamWaitEvent(side, ev, 0), "fork");
            }
            // FM_PIPE_TRACE=1: a timeline of the groups' stages (stderr), from events on their streams
            const bool ptrace = env_i64("FM_PIPE_TRACE", 0) != 0;
            struct Mark {
                int64_t g;
                const char *what;
                cudaEvent_t e;
            };
            std::vector<Mark> marks;
            cudaEvent_t t_0 = nullptr;
            auto mark = [&](int64_t g, const char *what, cudaStream_t s) {
                if (!ptrace) return;
                cudaEvent_t e;
                if (new_event(&e, true) != cudaSuccess) return;
                cudaEventRecord(e, s);
                marks.push_back({g, what, e});
            };
            if (ptrace && new_event(&t_0, true) == cudaSuccess) cudaEventRecord(t_0, st);
            for (int64_t g = 0; g < G; g++) {
                Group &q = grp[(size_t)g];
                cudaStream_t s = stream_of(g);
                mark(g, "begin", s);
                if (fuse) {
                    q.a.out_e = (int2 *)own->edges;
                    q.a.out_w = (int32_t *)own->weights;
                    q.a.out_cap = cap;
                }
                if (q.n_tasks > 0) CK(launch_sample(model, q.a, s), "sampler launch");
                mark(g, "sampled", s);
                if (timing && g == G - 1) CK(cudaEventRecord(t_b, s), "event record");
                if (q.n_tasks > 0 && !fuse)
                    CK(scan_exclusive_i64(q.counts, q.dest, q.n_tasks, scan_tmp + stb * (size_t)g, stb, s, g < G - 1, true),
                       "scan counts");
                // the group's base is the running total of the preceding groups (the other stream)
                if (ev_prev) CK(cudaStreamWaitEvent(s, ev_prev, 0), "wait for the preceding group's total");
                // (to_host: the group's end in the list also goes to a mapped page-locked word, for the
                // host's copy of the group's range)
                if (q.n_tasks > 0) {
                    CK(launch_offsets(q.R, q.tm, q.dest, offs_d + q.s0, gbase + g, gbase + g + 1,
                                      to_host ? pin_dev + g + 1 : nullptr, s),
                       "offsets");
                } else {
                    CK(cudaMemcpyAsync(gbase + g + 1, gbase + g, sizeof(int64_t), cudaMemcpyDeviceToDevice, s), "base");
                    if (to_host) pin_empty[(size_t)g] = 1;  // (its end = its start: resolved on the host)
                }
                if (G > 1 || to_host) {
                    CK(new_event(&ev_prev, false), "event");
                    CK(cudaEventRecord(ev_prev, s), "event record");
                    ev_off[(size_t)g] = ev_prev;
                    if (G == 1) ev_prev = nullptr;
                }
                if (q.n_tasks > 0)
                    CK(launch_overflow(q.n_tasks, q.tm, q.counts, q.spill_off, &hd[g].n_overflow, q.ovl, s),
                       "overflow check");
                // the final list was allocated up front (compaction and the re-run of overflowed tasks
                // are queued without a host round trip)
                mark(g, "scanned", s);
                if (!fuse) CK(compact_group(g, cap, s), "compact");
                mark(g, "compacted", s);
                if (to_host) {
                    CK(new_event(&ev_done[(size_t)g], false), "event");
                    CK(cudaEventRecord(ev_done[(size_t)g], s), "event record");
                }
            }
            if (to_host) {
                // every group is queued: copy each group's range of the list to the host as soon as
                // it is compacted, while the later groups are sampled (the host learns the range
                // from the pinned base words; ranges beyond the host capacity are not copied)
                NvtxRange nvtx_c("fm_sample: D2H of finished groups");
                bool all = true;
                for (int64_t g = 0; g < G; g++) {
                    CK(cudaEventSynchronize(ev_off[(size_t)g]), "wait for a group's base");
                    if (pin_empty[(size_t)g]) pin[g + 1] = pin[g];
                    const int64_t lo = pin[g], hi = ((volatile int64_t *)pin)[g + 1];
                    if (hi > cap || hi > host->cap) {  // (list or host buffer too small: handled after the pass)
                        all = false;
                        break;
                    }
                    if (hi == lo) continue;
                    CK(cudaStreamWaitEvent(copy_st, ev_done[(size_t)g], 0), "copy after compaction");
                    CK(copy_to_host_chunked(host->e + 2 * lo, (const int32_t *)own->edges + 2 * lo, sizeof(int32_t) * 2 * (hi - lo),
                                            copy_st),
                       "copy edges to the host");
                    if (host->w && own->weights)
                        CK(copy_to_host_chunked(host->w + lo, (const int32_t *)own->weights + lo, sizeof(int32_t) * (hi - lo), copy_st),
                           "copy weights to the host");
                    mark(g, "on host", copy_st);
                }
                cudaEvent_t ev;
                CK(new_event(&ev, false), "event");
                CK(cudaEventRecord(ev, copy_st), "event record");
                CK(cudaStreamWaitEvent(st, ev, 0), "join copies");
                host_done = all;
            }
            if (G > 1) {  // join
                cudaEvent_t ev;
                CK(new_event(&ev, false), "event");
                CK(cudaEventRecord(ev, side), "event record");
                CK(cudaStreamWaitEvent(st, ev, 0), "join");
            }
            if (timing) {
                CK(cudaEventRecord(t_c, st), "event record");
                // sampler phase = first sampler start .. last sampler end (the groups' samplers
                // overlap each other and the preceding groups' compactions); write phase = the
                // exposed remainder of the call
                std::lock_guard<std::mutex> lk(g_tmu);
                g_call_spans.push_back({t_a, t_b, t_c});  // (destroyed by fm_timing_get)
                g_sample_launches += G;
                for (auto &e : evs)
                    if (e == t_a || e == t_b || e == t_c) e = nullptr;
            }
            CK(cudaMemcpyAsync(offsets_h, offs_d, sizeof(int64_t) * (n_samples + 1), cudaMemcpyDeviceToHost, st),
               "read offsets");
            CK(cudaMemcpyAsync(h.data(), hd, sizeof(Hdr) * (size_t)G, cudaMemcpyDeviceToHost, st), "read hdr");
            CK(cudaMemcpyAsync(gbase_h.data(), gbase, sizeof(int64_t) * ((size_t)G + 1), cudaMemcpyDeviceToHost, st),
               "read group bases");
            // (pageable destinations: these reads are the call's synchronisation; the plan's flag word
            // is read here too, after every launch, not before the sampler)
            CK(cudaMemcpyAsync(&plan_flags, p->dev_flags, sizeof(unsigned int), cudaMemcpyDeviceToHost, st),
               "read plan flags");
            {
                NvtxRange nvtx_w("fm_sample: wait for the device");
                CK(cudaStreamSynchronize(st), "sync (sample)");
            }
            if (ptrace && t_0) {
                if (host)
                    fprintf(stderr, "[pipe] device list %p, host buffer %p\n", (const void *)own->edges, (const void *)host->e);
                for (const Mark &m : marks) {
                    float ms = 0.f;
                    cudaEventElapsedTime(&ms, t_0, m.e);
                    fprintf(stderr, "[pipe] group %lld %-9s %8.3f ms\n", (long long)m.g, m.what, ms);
                }
            }
            return FM_OK;
        };
        {
            fm_status r = run_pass(out_cap);
            if (r != FM_OK) return r;
        }
#ifdef FM_TRACE
        fm::dump_trace();
#endif
        fm::fuse_stats_dump();
        unsigned int hflags = 0;
        unsigned long long n_overflow = 0;
        for (int64_t g = 0; g < G; g++) {
            hflags |= h[(size_t)g].flags;
            n_overflow += h[(size_t)g].n_overflow;
        }
        if (plan_flags & kErrState) return fail(FM_ERR_STATE, "planner invariant violated (cuts)");
        // FM_DEBUG_CHECKS: a p > q contract violation fails the call; nothing stays allocated
        if (hflags & kErrBound) return fail(FM_ERR_BOUND, "p > q (1 + 2^-50) detected at a landed candidate (S:L289)");
        const int64_t total = offsets_h[n_samples];
        {  // capacity hint for the next call on this plan
            const double per = (double)std::max<int64_t>(1, p->est_draws - p->n_seg) * (double)n_samples;
            const double seen = (double)total / per;
            std::lock_guard<std::mutex> lk(g_mu);
            Plan *pm = const_cast<Plan *>(p);
            if (total > out_cap) pm->out_ratio = std::max(pm->out_ratio, seen * 1.02);
            else if (n_samples >= 8) pm->out_ratio = std::max(seen * 1.01, 0.05);
        }
        if (total > out_cap) {
            // the list was too small: the whole call again with an exact-size list (the scratch of
            // the earlier groups is gone: double-buffered, or discarded by the fused copiers); rare:
            // the plan's capacity hint covers every later call
            free_out();
            out_cap = total;
            fm_status r = run_pass(out_cap);
            if (r != FM_OK) return r;
            if (offsets_h[n_samples] != total) return fail(FM_ERR_STATE, "re-run total differs");
        }
        if (n_overflow > 0) {
            for (int64_t g = 0; g < G; g++)
                if (h[(size_t)g].n_overflow > 0) CK(rerun_group(g, out_cap), "rerun");
            CK(cudaStreamSynchronize(st), "sync (sample, rerun)");
        }
        bool host_short = false;
        if (to_host) {
            if (total > host->cap) {
                host_short = true;  // the device list stays valid: fm_edges_to_host with a larger buffer
            } else if ((!host_done || n_overflow > 0) && total > 0) {
                // (the list was redone or tasks were re-run into it after the groups' copies)
                CK(copy_to_host_chunked(host->e, own->edges, sizeof(int32_t) * 2 * total, st),
                   "copy edges to the host");
                if (host->w && own->weights)
                    CK(copy_to_host_chunked(host->w, own->weights, sizeof(int32_t) * total, st),
                       "copy weights to the host");
                CK(cudaStreamSynchronize(st), "sync (copy to the host)");
            }
        }
        out->n_edges = total;
        out->flags = ((hflags & kFlagWeightSat) ? FM_FLAG_WEIGHT_SATURATED : 0u) |
                     (n_overflow ? FM_FLAG_SCRATCH_RERUN : 0u) | (host_short ? FM_FLAG_HOST_TRUNCATED : 0u);
    }
    out->n_samples = n_samples;
    out->offsets = offsets_h;
    out->edges = (int32_t *)own->edges;
    out->weights = (int32_t *)own->weights;
    // every segment ends with exactly one terminal draw; every accepted edge is in the list
    out->draws = 0;
    for (const Hdr &hg : h) out->draws += (int64_t)hg.counters[0];
    out->landed = out->draws - p->n_seg * n_samples;
    out->accepted = out->n_edges;
    out->segments = p->n_seg * n_samples;
    out->chunks = n_tasks;  // tasks of the call (coarse + fine lane-chunks)
    out->_owner = own;
    og.o = nullptr;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        g_owners.insert(own);
    }
    return FM_OK;
}

// statistics-mode sampler launch shared by fm_sample_degrees and fm_sample_richclub
static fm_status stats_impl(const Plan *p, uint64_t seed, int64_t first_sample, int64_t n_samples, cudaStream_t st,
                            uint64_t *deg_plus, uint64_t *deg_minus, uint64_t *str_plus, uint64_t *str_minus,
                            uint64_t *rank_hist, fm_counters *out);

fm_status fm_sample_degrees(const fm_plan *plan_, uint64_t seed, int64_t first_sample, int64_t n_samples,
                            void *cuda_stream, uint64_t *deg_plus, uint64_t *deg_minus, uint64_t *str_plus,
                            uint64_t *str_minus, fm_counters *out)
{
    if (out) memset(out, 0, sizeof(*out));
    if (!plan_ || !plan_live(plan_)) return fail(FM_ERR_STATE, "not a live fm_plan");
    const Plan *p = (const Plan *)plan_;
    if (!deg_plus) return fail(FM_ERR_INVALID, "deg_plus is NULL");
    if (p->kind == FM_UNDIRECTED) {
        if (deg_minus && deg_minus != deg_plus) return fail(FM_ERR_INVALID, "undirected: deg_minus must be NULL");
        deg_minus = deg_plus;
        if (str_minus && str_minus != str_plus) return fail(FM_ERR_INVALID, "undirected: str_minus must be NULL");
        str_minus = str_plus;
    } else if (!deg_minus) {
        return fail(FM_ERR_INVALID, "bipartite/directed: deg_minus is NULL");
    }
    if (p->model == FM_ECM && (!str_plus || !str_minus)) return fail(FM_ERR_INVALID, "ECM: strength arrays needed");
    if (n_samples < 0 || first_sample < 0 || first_sample + n_samples > (int64_t(1) << 32))
        return fail(FM_ERR_INVALID, "sample range outside [0, 2^32)");
    return stats_impl(p, seed, first_sample, n_samples, (cudaStream_t)cuda_stream, deg_plus, deg_minus, str_plus,
                      str_minus, nullptr, out);
}

fm_status fm_sample_richclub(const fm_plan *plan_, uint64_t seed, int64_t first_sample, int64_t n_samples,
                             void *cuda_stream, uint64_t *e_top, fm_counters *out)
{
    if (out) memset(out, 0, sizeof(*out));
    if (!plan_ || !plan_live(plan_)) return fail(FM_ERR_STATE, "not a live fm_plan");
    const Plan *p = (const Plan *)plan_;
    if (p->kind != FM_UNDIRECTED) return fail(FM_ERR_STATE, "rich club: undirected plans only");
    if (!e_top) return fail(FM_ERR_INVALID, "e_top is NULL");
    if (n_samples < 0 || first_sample < 0 || first_sample + n_samples > (int64_t(1) << 32))
        return fail(FM_ERR_INVALID, "sample range outside [0, 2^32)");
    cudaStream_t st = (cudaStream_t)cuda_stream;
    Allocs tmp(st);
    uint64_t *hist, *cum;
    char *work;
    const size_t sb = scan_tmp_bytes(p->n + 1);
    CK(tmp.get(&hist, p->n + 1), "alloc rank histogram");
    CK(tmp.get(&cum, p->n + 1), "alloc rank prefix");
    CK(tmp.get(&work, sb), "alloc scan tmp");
    CK(cudaMemsetAsync(hist, 0, sizeof(uint64_t) * (p->n + 1), st), "memset histogram");
    fm_status r = stats_impl(p, seed, first_sample, n_samples, st, nullptr, nullptr, nullptr, nullptr, hist, out);
    if (r != FM_OK) return r;
    // e_top[m] += sum_{r < m} hist[r]: edges whose larger rank is below m join two top-m nodes
    CK(scan_exclusive_u64(hist, cum, p->n, work, sb, st), "scan histogram");
    CK(launch_add_u64(cum, e_top, p->n + 1, st), "accumulate e_top");
    CK(cudaStreamSynchronize(st), "sync (rich club)");
    return FM_OK;
}

static fm_status stats_impl(const Plan *p, uint64_t seed, int64_t first_sample, int64_t n_samples, cudaStream_t st,
                            uint64_t *deg_plus, uint64_t *deg_minus, uint64_t *str_plus, uint64_t *str_minus,
                            uint64_t *rank_hist, fm_counters *out)
{
    NvtxRange nvtx_("fm_sample statistics mode (NEXT-3)");
    int64_t n_tasks = 0;
    const int64_t kf = std::min(tail_samples(p, 0), n_samples);
    const int64_t km = p->n_chunks[2] > 0 ? std::max<int64_t>(0, std::min(tail_samples(p, 2), n_samples) - kf) : 0;
    const TaskMap tm = make_task_map(p, n_samples, kf, km, &n_tasks);
    if (n_tasks == 0) return FM_OK;
    Allocs tmp(st);
    struct Hdr {
        unsigned long long counters[3];
        unsigned int flags, pad;
        unsigned long long task_counter;
    };
    Hdr *hd;
    CK(tmp.get(&hd, 1), "alloc hdr");
    CK(cudaMemsetAsync(hd, 0, sizeof(Hdr), st), "memset hdr");
    SampleArgs a;
    memset(&a, 0, sizeof(a));
    a.rec = p->rec;
    a.kappa_s = p->ckappa;
    a.y_s = p->cy;
    a.ly_s = p->cly;
    a.perm = p->cperm;
    a.cand = p->cand;
    a.ordered = p->kind != FM_UNDIRECTED;
    a.tm = tm;
    a.key = philox_key(seed);
    a.lc = log_consts();
    a.first_sample = (uint32_t)first_sample;
    a.n_tasks = n_tasks;
    a.task_counter = &hd->task_counter;
    a.counters = hd->counters;
    a.flags = &hd->flags;
    a.deg_row = (unsigned long long *)deg_plus;
    a.deg_col = (unsigned long long *)deg_minus;
    a.str_row = (unsigned long long *)str_plus;
    a.str_col = (unsigned long long *)str_minus;
    a.rank_hist = (unsigned long long *)rank_hist;
    a.check = env_i64("FM_DEBUG_CHECKS", 0) != 0;
    PhaseTimer ts;
    ts.begin(kPhaseSample, st);
    CK(launch_sample(p->model, a, st), "sampler launch (degrees)");
    ts.end(st);
    Hdr h;
    unsigned int plan_flags = 0;
    CK(cudaMemcpyAsync(&h, hd, sizeof(Hdr), cudaMemcpyDeviceToHost, st), "read hdr");
    CK(cudaMemcpyAsync(&plan_flags, p->dev_flags, sizeof(unsigned int), cudaMemcpyDeviceToHost, st), "read flags");
    CK(cudaStreamSynchronize(st), "sync (degrees)");
    if (plan_flags & kErrState) return fail(FM_ERR_STATE, "planner invariant violated (cuts)");
    if (h.flags & kErrBound) return fail(FM_ERR_BOUND, "p > q (1 + 2^-50) detected at a landed candidate (S:L289)");
    if (out) {
        out->draws = (int64_t)h.counters[0];
        out->landed = out->draws - p->n_seg * n_samples;  // one terminal draw per segment
        out->accepted = (int64_t)h.counters[2];
        out->flags = (h.flags & kFlagWeightSat) ? FM_FLAG_WEIGHT_SATURATED : 0u;
    }
    return FM_OK;
}

fm_status fm_sample_ubcm(const fm_plan *plan, uint64_t seed, int64_t first_sample, int64_t n_samples,
                         void *cuda_stream, fm_edges *out)
{
    return sample_impl(FM_UBCM, plan, seed, first_sample, n_samples, 0u, cuda_stream, out);
}

fm_status fm_sample_ecm(const fm_plan *plan, uint64_t seed, int64_t first_sample, int64_t n_samples,
                        void *cuda_stream, fm_edges *out)
{
    return sample_impl(FM_ECM, plan, seed, first_sample, n_samples, 0u, cuda_stream, out);
}

fm_status fm_sample_ecm_ex(const fm_plan *plan, uint64_t seed, int64_t first_sample, int64_t n_samples,
                           uint32_t flags, void *cuda_stream, fm_edges *out)
{
    if (flags & ~(uint32_t)FM_SAMPLE_BETA_REFRESH) {
        if (out) memset(out, 0, sizeof(*out));
        return fail(FM_ERR_INVALID, "unknown fm_sample_ecm_ex flags 0x%x", flags);
    }
    return sample_impl(FM_ECM, plan, seed, first_sample, n_samples, flags, cuda_stream, out);
}

fm_status fm_sample_to_host(const fm_plan *plan, uint64_t seed, int64_t first_sample, int64_t n_samples, uint32_t flags,
                            void *cuda_stream, int32_t *edges_host, int32_t *weights_host, int64_t host_cap,
                            fm_edges *out)
{
    if (out) memset(out, 0, sizeof(*out));
    if (!plan || !plan_live(plan)) return fail(FM_ERR_STATE, "not a live fm_plan");
    const Plan *p = (const Plan *)plan;
    if (flags & ~(uint32_t)FM_SAMPLE_BETA_REFRESH) return fail(FM_ERR_INVALID, "unknown fm_sample_to_host flags 0x%x", flags);
    if (p->model == FM_UBCM && flags) return fail(FM_ERR_INVALID, "FM_SAMPLE_BETA_REFRESH: ECM plans only");
    if (!edges_host || host_cap < 0) return fail(FM_ERR_INVALID, "edges_host is NULL or host_cap < 0");
    HostDst hd;
    hd.e = edges_host;
    hd.w = p->model == FM_ECM ? weights_host : nullptr;
    hd.cap = host_cap;
    return sample_impl(p->model, plan, seed, first_sample, n_samples, flags, cuda_stream, out, &hd);
}

fm_status fm_edges_to_host(const fm_edges *e, int32_t *edges_host, int32_t *weights_host, void *cuda_stream)
{
    NvtxRange nvtx_("fm_edges_to_host");
    if (!e) return fail(FM_ERR_INVALID, "NULL result");
    {
        std::lock_guard<std::mutex> lk(g_mu);
        if (!g_owners.count(e->_owner)) return fail(FM_ERR_STATE, "not a live fm_edges");
    }
    cudaStream_t st = (cudaStream_t)cuda_stream;
    if (e->n_edges > 0) {
        if (!edges_host) return fail(FM_ERR_INVALID, "edges_host is NULL");
        CK(copy_to_host_chunked(edges_host, e->edges, sizeof(int32_t) * 2 * e->n_edges, st),
           "copy edges");
        if (weights_host && e->weights)
            CK(copy_to_host_chunked(weights_host, e->weights, sizeof(int32_t) * e->n_edges, st),
               "copy weights");
    }
    CK(cudaStreamSynchronize(st), "sync (to_host)");
    return FM_OK;
}

fm_status fm_plan_get_info(const fm_plan *plan, fm_plan_info *info)
{
    if (!info) return fail(FM_ERR_INVALID, "info is NULL");
    if (!plan || !plan_live(plan)) return fail(FM_ERR_STATE, "not a live fm_plan");
    const Plan *p = (const Plan *)plan;
    info->model = p->model;
    info->kind = p->kind;
    info->n_minus = p->nc;
    info->n = p->n;
    info->seg_target = p->S;
    info->F = p->F;
    info->n_segments = p->n_seg;
    info->n_chunks = p->n_chunks[0];
    info->est_draws = p->est_draws;
    return FM_OK;
}

fm_status fm_plan_export(const fm_plan *plan, int32_t *perm, double *kappa_s, double *y_s, double *ymax, double *ly_s,
                         int32_t *seg, double *seg_h0, double *seg_x0, double *seg_d0, double *seg_omT,
                         double *seg_iomT)
{
    if (!plan || !plan_live(plan)) return fail(FM_ERR_STATE, "not a live fm_plan");
    const Plan *p = (const Plan *)plan;
    CK(cudaDeviceSynchronize(), "sync");
    const size_t n = (size_t)p->n, s = (size_t)p->n_seg;
    if (perm) CK(cudaMemcpy(perm, p->perm, n * 4, cudaMemcpyDeviceToHost), "perm");
    if (kappa_s) CK(cudaMemcpy(kappa_s, p->kappa_s, n * 8, cudaMemcpyDeviceToHost), "kappa_s");
    if (y_s && p->y_s) CK(cudaMemcpy(y_s, p->y_s, n * 8, cudaMemcpyDeviceToHost), "y_s");
    if (ymax && p->ymax) CK(cudaMemcpy(ymax, p->ymax, ((size_t)p->nc + 1) * 8, cudaMemcpyDeviceToHost), "ymax");
    if (ly_s && p->ly_s) CK(cudaMemcpy(ly_s, p->ly_s, n * 8, cudaMemcpyDeviceToHost), "ly_s");
    if (s && (seg || seg_h0 || seg_x0 || seg_d0 || seg_omT || seg_iomT)) {  // from the packed records
        const size_t stride = (size_t)kRecStride(p->model);
        std::vector<unsigned char> raw(s * stride);
        CK(cudaMemcpy(raw.data(), p->rec, s * stride, cudaMemcpyDeviceToHost), "seg records");
        std::vector<SegRec> r(s);
        for (size_t g = 0; g < s; g++) {
            memset(&r[g], 0, sizeof(SegRec));
            memcpy(&r[g], raw.data() + g * stride, stride);
            if (p->model == FM_UBCM) r[g].omT = r[g].iomT = 1.0;  // (not stored: UBCM's bound has T = 0)
        }
        for (size_t g = 0; g < s; g++) {
            if (seg) {
                seg[4 * g] = r[g].u;
                seg[4 * g + 1] = r[g].a;
                seg[4 * g + 2] = r[g].b;
                seg[4 * g + 3] = r[g].sigma;
            }
            if (seg_h0) seg_h0[g] = r[g].h0;
            if (seg_x0) seg_x0[g] = r[g].x0;
            if (seg_d0) seg_d0[g] = r[g].d0;
            if (seg_omT) seg_omT[g] = r[g].omT;
            if (seg_iomT) seg_iomT[g] = r[g].iomT;
        }
    }
    return FM_OK;
}

fm_status fm_plan_export_candidates(const fm_plan *plan, int32_t *cperm, double *ckappa, double *cy, double *cly,
                                    int32_t *excl)
{
    if (!plan || !plan_live(plan)) return fail(FM_ERR_STATE, "not a live fm_plan");
    const Plan *p = (const Plan *)plan;
    CK(cudaDeviceSynchronize(), "sync");
    const size_t nc = (size_t)p->nc, n = (size_t)p->n;
    if (cperm) CK(cudaMemcpy(cperm, p->cperm, nc * 4, cudaMemcpyDeviceToHost), "cperm");
    if (ckappa) CK(cudaMemcpy(ckappa, p->ckappa, nc * 8, cudaMemcpyDeviceToHost), "ckappa");
    if (cy && p->cy) CK(cudaMemcpy(cy, p->cy, nc * 8, cudaMemcpyDeviceToHost), "cy");
    if (cly && p->cly) CK(cudaMemcpy(cly, p->cly, nc * 8, cudaMemcpyDeviceToHost), "cly");
    if (excl) {
        if (p->excl) CK(cudaMemcpy(excl, p->excl, n * 4, cudaMemcpyDeviceToHost), "excl");
        else for (size_t u = 0; u < n; u++) excl[u] = -1;
    }
    return FM_OK;
}

fm_status fm_expected_degrees(fm_model model, int64_t n, const double *x, const double *y, const int32_t *nodes,
                              int64_t n_nodes, double *k, double *kvar, double *s, double *svar, void *cuda_stream)
{
    if (model != FM_UBCM && model != FM_ECM) return fail(FM_ERR_INVALID, "unknown model %d", (int)model);
    if (n < 1 || n > INT32_MAX) return fail(FM_ERR_INVALID, "n = %lld outside [1, 2^31-1]", (long long)n);
    if (!x || (model == FM_ECM && !y)) return fail(FM_ERR_INVALID, "x (and, for the ECM, y) needed");
    if (model == FM_UBCM && y) return fail(FM_ERR_INVALID, "UBCM takes no y");
    if (!nodes) n_nodes = n;
    if (n_nodes < 0) return fail(FM_ERR_INVALID, "n_nodes < 0");
    if (n_nodes == 0) return FM_OK;
    if (!k && !kvar && !s && !svar) return FM_OK;
    for (const void *o : {(const void *)k, (const void *)kvar, (const void *)s, (const void *)svar})
        if (o && !is_device_ptr(o)) return fail(FM_ERR_INVALID, "outputs must be DEVICE buffers");
    if (model == FM_UBCM && (s || svar)) return fail(FM_ERR_INVALID, "UBCM has no strengths");
    cudaStream_t st = (cudaStream_t)cuda_stream;
    Allocs tmp(st);
    auto dev_copy = [&](const auto *h, int64_t cnt, const auto **d) -> cudaError_t {
        *d = h;
        if (!h || is_device_ptr(h)) return cudaSuccess;
        using T = std::remove_const_t<std::remove_pointer_t<decltype(h)>>;
        T *t;
        cudaError_t e = tmp.get(&t, cnt);
        if (e == cudaSuccess) e = cudaMemcpyAsync(t, h, sizeof(T) * cnt, cudaMemcpyHostToDevice, st);
        *d = t;
        return e;
    };
    const double *xd, *yd;
    const int32_t *nd;
    CK(dev_copy(x, n, &xd), "copy x");
    CK(dev_copy(y, n, &yd), "copy y");
    CK(dev_copy(nodes, n_nodes, &nd), "copy nodes");
    CK(launch_expected((int)model, n, xd, yd, nd, n_nodes, k, kvar, s, svar, st), "expected");
    CK(cudaStreamSynchronize(st), "sync (expected)");
    return FM_OK;
}

fm_status fm_debug_eval(int32_t fn, int64_t n, const double *in_dev, double *out_dev, void *cuda_stream)
{
    if (fn < 0 || fn > 3 || n < 0 || (n > 0 && (!in_dev || !out_dev))) return fail(FM_ERR_INVALID, "bad debug_eval args");
    CK(launch_debug_eval(fn, n, in_dev, out_dev, (cudaStream_t)cuda_stream), "debug eval");
    return FM_OK;
}

fm_status fm_pool_trim(uint64_t keep_bytes)
{
    int dev = 0;
    CK(cudaGetDevice(&dev), "cudaGetDevice");
    cudaMemPool_t pool;
    CK(cudaDeviceGetDefaultMemPool(&pool, dev), "default pool");
    CK(cudaDeviceSynchronize(), "sync");
    CK(cudaMemPoolTrimTo(pool, (size_t)keep_bytes), "trim");
    return FM_OK;
}

fm_status fm_timing_enable(int on)
{
    g_timing.store(on != 0);
    return FM_OK;
}

fm_status fm_timing_get(fm_timing *t, int reset)
{
    if (!t) return fail(FM_ERR_INVALID, "NULL timing");
    std::lock_guard<std::mutex> lk(g_tmu);
    for (auto &pd : g_pending) {
        float ms = 0.f;
        if (cudaEventSynchronize(pd.b) == cudaSuccess && cudaEventElapsedTime(&ms, pd.a, pd.b) == cudaSuccess)
            g_phase_ms[pd.phase] += ms;
        cudaEventDestroy(pd.a);
        cudaEventDestroy(pd.b);
    }
    g_pending.clear();
    for (auto &sp : g_call_spans) {
        float ms = 0.f;
        if (cudaEventSynchronize(sp.c) == cudaSuccess) {
            if (cudaEventElapsedTime(&ms, sp.a, sp.b) == cudaSuccess) g_phase_ms[kPhaseSample] += ms;
            if (cudaEventElapsedTime(&ms, sp.b, sp.c) == cudaSuccess) g_phase_ms[kPhaseWrite] += ms;
        }
        cudaEventDestroy(sp.a);
        cudaEventDestroy(sp.b);
        cudaEventDestroy(sp.c);
    }
    g_call_spans.clear();
    t->plan_ms = g_phase_ms[kPhasePlan];
    t->sample_ms = g_phase_ms[kPhaseSample];
    t->write_ms = g_phase_ms[kPhaseWrite];
    t->sample_launches = g_sample_launches;
    t->launches = g_launches.load();
    if (reset) {
        g_phase_ms[0] = g_phase_ms[1] = g_phase_ms[2] = 0;
        g_sample_launches = 0;
    }
    return FM_OK;
}

void fm_free(void *obj)
{
    if (!obj) return;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        if (g_plans.erase(obj)) {
            cudaDeviceSynchronize();
            plan_release((Plan *)obj);
            return;
        }
    }
    fm_edges *e = (fm_edges *)obj;
    Owner *o = (Owner *)e->_owner;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        if (!o || !g_owners.erase(o)) return;  // not ours: ignore
    }
    if (o->edges) cudaFreeAsync(o->edges, o->stream);
    if (o->weights) cudaFreeAsync(o->weights, o->stream);
    free(o->offsets_host);
    o->magic = 0;
    delete o;
    memset(e, 0, sizeof(*e));
}

}  // extern "C"
