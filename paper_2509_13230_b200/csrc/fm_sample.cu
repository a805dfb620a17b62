// fm_sample.cu -- a5 (the chain) and a6 (count -> scan -> write) on sm_100a.
//
// Work decomposition (v2).  The plan groups consecutive segments (canonical order: row u,
// segment sigma) into LANE-CHUNKS of ~equal estimated work.  A task = (sample s, lane-chunk c).
// The kernel is persistent: every lane runs one task at a time, sequentially over the task's
// segments, and takes the next task from a global queue (one warp-aggregated atomicAdd per
// batch of lanes).  A lane writes its task's edges contiguously, in draw order, into the task's
// scratch slot, so the output of every task -- and after compaction the whole edge list -- is in
// the oracle's canonical order (sample, u, sigma, draw), independent of scheduling.
//
// Per lane-iteration one geometric draw is consumed:
//   3. R = E/h; terminal -> switch to the prefetched next segment; landed -> cur, issue LDG k[cur]
//   4. Philox + -log(u01) for the NEXT draw of every active lane (overlaps the gather latency;
//      convergent for landed and restarted lanes alike)
//   5. landed lanes: p = X/(1+X), accept u01*q < p, q <- p, h <- log1p(X), store the edge
// Decision arithmetic: DESIGN.md 3.5 with RN intrinsics (no contraction); log/log1p are the
// table-driven fm_log/fm_log1p (fm_math.cuh, ~0.5 ulp).
#include <float.h>

#include <cmath>
#include <cstdlib>
#include <mutex>

#include "fm_internal.cuh"
#include "fm_math.cuh"
#include "fm_plan_kernels.cuh"

namespace fm {

__device__ LogTable g_logtab;

namespace {

constexpr int kThreads = 256;
constexpr int kBatch = 64;  // tasks per warp batch

// per-block copy of the log table (file-scope shared: addressed with constant offsets)
__shared__ double2 s_log_ic[kLogTable];
__shared__ double s_log_lo[kLogTable];
struct SmemLogTab {
    __device__ __forceinline__ double2 ic(int i) const { return s_log_ic[i]; }
    __device__ __forceinline__ double lo(int i) const { return s_log_lo[i]; }
    __device__ __forceinline__ LogConsts C() const { return log_consts(); }
};

__device__ __forceinline__ void load_logtab()
{
    for (int j = threadIdx.x; j < kLogTable; j += blockDim.x) {
        s_log_ic[j] = g_logtab.ic[j];
        s_log_lo[j] = g_logtab.logc_lo[j];
    }
    __syncthreads();
}

template <int kModel, int kMinBlocks>
__global__ void __launch_bounds__(kThreads, kMinBlocks) k_sample(const SampleArgs A)
{
    __shared__ SegRec s_next[kThreads];
    load_logtab();
    const SmemLogTab T;
    const int lane = threadIdx.x & 31;
    const uint32_t lt = (1u << lane) - 1u;

    // ---- task (lane-chunk) state ----
    int64_t task = -1, slot = 0, sp = -1;
    // warp batch of task ids [bpos, bend); lane 0 holds the start of the next batch
    unsigned long long next_batch = 0;
    if (lane == 0) next_batch = atomicAdd(A.task_counter, (unsigned long long)kBatch);
    int64_t bpos = 0, bend = 0;
    int32_t g = 0, g_end = 0, cnt = 0, cap = 0;
    uint32_t s_abs = 0;
    bool warp_done = false;
    // ---- current segment ----
    bool act = false;
    int32_t u = 0, b = 0, cur = 0, id_u = 0;
    uint32_t sg = 0, d = 0;
    double xq = 0.0, dq = 1.0, h = 0.0, ku = 0.0, yu = 0.0, lyu = 0.0, omT = 1.0, iomT = 1.0, E = 0.0;
    uint32_t wacc = 0, wwt = 0;
    // ---- counters ----
    uint32_t n_draw = 0, n_land = 0, n_acc = 0;
    bool wsat = false;

    // segment g of the current task becomes current.  The record of segment g+1 is prefetched
    // into this thread's shared-memory slot with cp.async (no registers held), so a restart
    // after a terminal draw reads shared memory instead of waiting on a global load.
    SegRec *my_next = &s_next[threadIdx.x];
    const uint32_t my_next_sa = (uint32_t)__cvta_generic_to_shared(my_next);
    auto start_seg = [&](bool prefetched) {
        const SegRec *r = prefetched ? my_next : A.rec + g;
        if (prefetched) asm volatile("cp.async.wait_all;\n" ::: "memory");
        const int4 p0 = *reinterpret_cast<const int4 *>(r);
        const double2 p1 = *reinterpret_cast<const double2 *>(&r->h0);
        const double2 p2 = *reinterpret_cast<const double2 *>(&r->d0);
        const int4 p3 = *reinterpret_cast<const int4 *>(&r->id_u);
        u = p0.x;
        cur = p0.y - 1;  // virtual previous position a-1 (R3)
        b = p0.z;
        sg = (uint32_t)p0.w;
        h = p1.x;
        xq = p1.y;
        dq = p2.x;
        ku = p2.y;
        id_u = p3.x;
        if (kModel == FM_ECM) {
            const double2 p4 = *reinterpret_cast<const double2 *>(&r->yu);
            const double2 p5 = *reinterpret_cast<const double2 *>(&r->omT);
            yu = p4.x;
            lyu = p4.y;
            omT = p5.x;
            iomT = p5.y;
        }
        d = 0;
        g++;
        act = true;
        if (g < g_end) {
            const char *src = reinterpret_cast<const char *>(A.rec + g);
            constexpr int parts = kModel == FM_ECM ? 6 : 4;
#pragma unroll
            for (int k = 0; k < parts; k++)
                asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(my_next_sa + 16 * k),
                             "l"(src + 16 * k)
                             : "memory");
            asm volatile("cp.async.commit_group;\n" ::: "memory");
        }
    };
    auto draw_words = [&]() {  // E and the accept/weight words of draw d (R1, R2)
        uint32_t ws;
        if (kModel == FM_UBCM) {
            const uint4 W = philox4x32_10(make_uint4(d >> 1, sg, (uint32_t)u, s_abs), A.key);
            ws = (d & 1) ? W.z : W.x;
            wacc = (d & 1) ? W.w : W.y;
        } else {
            const uint4 W = philox4x32_10(make_uint4(d, sg, (uint32_t)u, s_abs), A.key);
            ws = W.x;
            wacc = W.y;
            wwt = W.z;
        }
        E = -fm_log(u01(ws), T);
    };

    for (;;) {
        // ---- 1. task management (lanes whose task has no segment left) ----
        // Tasks come in warp batches of kBatch consecutive ids from the global queue; the next
        // batch is requested (by lane 0) as soon as the current one is opened, so the atomic's
        // latency is never waited for.
        const bool needc = !act;
        if (needc && task >= 0) {
            if (!A.rerun_base) {
                A.counts[task] = cnt;
                A.spill_off[task] = sp;
            }
            task = -1;
        }
        const uint32_t nc = __ballot_sync(0xffffffffu, needc && !warp_done);
        bool fresh = false;
        if (nc) {
            const int k = __popc(nc), rank = __popc(nc & lt);
            const int64_t avail = bend - bpos;
            int64_t my;
            if (k <= avail) {
                my = bpos + rank;
                bpos += k;
            } else {
                const int64_t nb = (int64_t)__shfl_sync(0xffffffffu, next_batch, 0);
                my = rank < avail ? bpos + rank : nb + (rank - avail);
                bpos = nb + (k - avail);
                bend = nb + kBatch;
                if (lane == 0) next_batch = atomicAdd(A.task_counter, (unsigned long long)kBatch);
            }
            if (needc && !warp_done && my < A.n_tasks) {
                const int64_t t = A.task_list ? A.task_list[my] : my;
                const int64_t s = t / A.n_chunks, c = t - s * A.n_chunks;
                task = t;
                g = (int32_t)A.chunk_seg[c];
                g_end = (int32_t)A.chunk_seg[c + 1];
                if (A.rerun_base) {
                    slot = A.rerun_base[t];
                    cap = INT32_MAX;
                } else {
                    slot = s * A.cap_per_sample + A.chunk_cap[c];
                    cap = (int32_t)(A.chunk_cap[c + 1] - A.chunk_cap[c]);
                }
                s_abs = A.first_sample + (uint32_t)s;
                cnt = 0;
                sp = -1;
                if (g < g_end) {
                    start_seg(false);
                    fresh = true;
                }
            }
            if (bpos >= A.n_tasks) warp_done = true;
        }
        if (!__any_sync(0xffffffffu, act)) {
            if (warp_done) break;
            continue;
        }
        // ---- 2. first draw of a freshly fetched task ----
        if (fresh) draw_words();

        // ---- 3. consume one draw ----
        bool landed = false;
        uint32_t w_land = 0, w_wt = 0;
        double kv = 0.0, yv = 0.0, lyv = 0.0;
        int32_t id_v = 0;
        if (act) {
            n_draw++;
            const double R = __ddiv_rn(E, h);
            if (!(R < (double)(b - 1 - cur))) {  // terminal draw (R5)
                if (g < g_end) start_seg(true);
                else act = false;
            } else {
                cur = cur + 1 + (int32_t)R;  // R >= 0: truncation == floor
                kv = A.kappa_s[cur];
                if (kModel == FM_ECM) {
                    yv = A.y_s[cur];
                    lyv = A.ly_s[cur];
                }
                id_v = A.perm[cur];  // issued early; needed only if accepted
                landed = true;
                w_land = wacc;
                w_wt = wwt;
                d++;
                n_land++;
            }
        }
        // ---- 4+5. one straight-line block for every active lane: RNG + E of the next draw
        //      (overlaps the k[cur] gather) interleaved with the p/q test of the landed candidate
        //      (lanes that restarted a segment evaluate a dummy X = 1 and keep their h0, q0) ----
        bool acc = false;
        int32_t w = 1;
        if (act) {
            uint32_t ws;
            if (kModel == FM_UBCM) {
                const uint4 W = philox4x32_10(make_uint4(d >> 1, sg, (uint32_t)u, s_abs), A.key);
                ws = (d & 1) ? W.z : W.x;
                wacc = (d & 1) ? W.w : W.y;
            } else {
                const uint4 W = philox4x32_10(make_uint4(d, sg, (uint32_t)u, s_abs), A.key);
                ws = W.x;
                wacc = W.y;
                wwt = W.z;
            }
            const double Enew = -fm_log(u01(ws), T);
            if (kModel == FM_UBCM) {
                // (kv + 0*Enew) orders the use of the gathered kv after the RNG/log work above,
                // so the gather latency hides behind it; exact since Enew is finite and kv >= 0
                const double kvd = __dadd_rn(kv, __dmul_rn(Enew, 0.0));
                const double X = landed ? __dmul_rn(ku, kvd) : 1.0;  // dummy for restarted lanes
                const double D = __dadd_rn(1.0, X);
                const double hn = fm_log1p(X, T);
                if (landed) {  // accept iff u < (X/D) / (xq/dq), cross-multiplied (R10)
                    acc = __dmul_rn(__dmul_rn(u01(w_land), xq), D) < __dmul_rn(X, dq);
                    xq = X;
                    dq = D;
                    h = hn;
                }
            } else {
                const double kvd = __dadd_rn(kv, __dmul_rn(Enew, 0.0));  // see UBCM
                const double z = landed ? __dmul_rn(ku, kvd) : 1.0;  // dummy for restarted lanes
                const double t = __dmul_rn(yu, yv);
                const double Dp = __dadd_rn(__dsub_rn(1.0, t), z);
                const double hn = fm_log1p(__dmul_rn(z, iomT), T);
                if (landed) {
                    acc = __dmul_rn(__dmul_rn(u01(w_land), xq), Dp) < __dmul_rn(z, dq);
                    xq = z;
                    dq = __dadd_rn(omT, z);
                    h = hn;
                    if (acc) {  // Eq. 5 weight, log t = log y_u + log y_v (R8)
                        const double lu = fm_log(u01(w_wt), T);
                        const double G = floor(__ddiv_rn(lu, __dadd_rn(lyu, lyv)));
                        if (G <= 2147483646.0) {
                            w = 1 + (int32_t)G;
                        } else {
                            w = INT32_MAX;
                            wsat = true;
                        }
                    }
                }
            }
            E = Enew;
        }
        if (landed) {
            if (acc) {
                const int2 ev = make_int2(min(id_u, id_v), max(id_u, id_v));
                if (cnt < cap) {
                    A.edges[slot + cnt] = ev;
                    if (kModel == FM_ECM) A.weights[slot + cnt] = w;
                } else if (!A.rerun_base && cnt < 2 * cap) {  // spill: one extra region of `cap` edges
                    if (sp == -1) {
                        const unsigned long long o = atomicAdd(A.spill_counter, (unsigned long long)cap);
                        sp = (int64_t)(o + cap) <= A.spill_cap ? (int64_t)o : -2;
                    }
                    if (sp >= 0) {
                        A.spill_e[sp + cnt - cap] = ev;
                        if (kModel == FM_ECM) A.spill_w[sp + cnt - cap] = w;
                    }
                }
                cnt++;
                n_acc++;
            }
        }
    }
    if (A.rerun_base) return;
    const unsigned dr = __reduce_add_sync(0xffffffffu, n_draw);
    const unsigned la = __reduce_add_sync(0xffffffffu, n_land);
    const unsigned ac = __reduce_add_sync(0xffffffffu, n_acc);
    const bool anysat = __any_sync(0xffffffffu, wsat);
    if (lane == 0) {
        atomicAdd(&A.counters[0], (unsigned long long)dr);
        atomicAdd(&A.counters[1], (unsigned long long)la);
        atomicAdd(&A.counters[2], (unsigned long long)ac);
        if (anysat) atomicOr(A.flags, kFlagWeightSat);
    }
}

__device__ __forceinline__ bool task_overflowed(int64_t cnt, int64_t cap, int64_t sp)
{
    return cnt > cap && (cnt > 2 * cap || sp < 0);
}

__global__ void __launch_bounds__(256) k_overflow(int64_t n_tasks, int64_t n_chunks, const int64_t *__restrict__ chunk_cap,
                                                  const int64_t *__restrict__ counts,
                                                  const int64_t *__restrict__ spill_off, unsigned long long *n_overflow,
                                                  int64_t *__restrict__ overflow_list)
{
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n_tasks) return;
    const int64_t c = t % n_chunks;
    if (task_overflowed(counts[t], chunk_cap[c + 1] - chunk_cap[c], spill_off[t])) {
        const unsigned long long k = atomicAdd(n_overflow, 1ull);
        overflow_list[k] = t;
    }
}

// Gather: block b handles tasks [256 b, 256 b + 256): their metadata is staged in shared memory
// by one coalesced pass, then each warp copies 32 of the tasks (slot, then spill part),
// 4 elements per lane in flight.  Overflowed tasks are skipped (re-run into the final array).
constexpr int kCopyThreads = 256;
__global__ void __launch_bounds__(kCopyThreads) k_compact(int64_t n_tasks, int64_t n_chunks, int64_t cap_per_sample,
                                                          const int64_t *__restrict__ chunk_cap,
                                                          const int64_t *__restrict__ counts,
                                                          const int64_t *__restrict__ dest,
                                                          const int64_t *__restrict__ spill_off,
                                                          const int2 *__restrict__ se, const int32_t *__restrict__ sw,
                                                          const int2 *__restrict__ spe, const int32_t *__restrict__ spw,
                                                          int2 *__restrict__ oe, int32_t *__restrict__ ow)
{
    __shared__ int64_t s_src[kCopyThreads], s_dst[kCopyThreads], s_sp[kCopyThreads];
    __shared__ int32_t s_cnt[kCopyThreads], s_cap[kCopyThreads];
    const int64_t t0 = (int64_t)blockIdx.x * kCopyThreads;
    {
        const int64_t t = t0 + threadIdx.x;
        int32_t cn = 0, cp = 0;
        int64_t src = 0, dst = 0, sp = -1;
        if (t < n_tasks) {
            const int64_t s = t / n_chunks, c = t - s * n_chunks;
            const int64_t cap = chunk_cap[c + 1] - chunk_cap[c];
            const int64_t cnt = counts[t];
            sp = spill_off[t];
            cn = task_overflowed(cnt, cap, sp) ? 0 : (int32_t)cnt;
            cp = (int32_t)cap;
            src = s * cap_per_sample + chunk_cap[c];
            dst = dest[t];
        }
        s_src[threadIdx.x] = src;
        s_dst[threadIdx.x] = dst;
        s_sp[threadIdx.x] = sp;
        s_cnt[threadIdx.x] = cn;
        s_cap[threadIdx.x] = cp;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int k = wid; k < kCopyThreads; k += kCopyThreads / 32) {
        const int32_t cnt = s_cnt[k], cap = s_cap[k];
        if (cnt == 0) continue;
        const int64_t src = s_src[k], dst = s_dst[k], sp = s_sp[k];
        const int32_t n1 = min(cnt, cap);
        for (int32_t i0 = 0; i0 < n1; i0 += 128) {
            int2 v[4];
#pragma unroll
            for (int j = 0; j < 4; j++) {
                const int32_t i = i0 + j * 32 + lane;
                if (i < n1) v[j] = se[src + i];
            }
#pragma unroll
            for (int j = 0; j < 4; j++) {
                const int32_t i = i0 + j * 32 + lane;
                if (i < n1) oe[dst + i] = v[j];
            }
            if (ow) {
                int32_t x[4];
#pragma unroll
                for (int j = 0; j < 4; j++) {
                    const int32_t i = i0 + j * 32 + lane;
                    if (i < n1) x[j] = sw[src + i];
                }
#pragma unroll
                for (int j = 0; j < 4; j++) {
                    const int32_t i = i0 + j * 32 + lane;
                    if (i < n1) ow[dst + i] = x[j];
                }
            }
        }
        for (int32_t i = cap + lane; i < cnt; i += 32) {  // spilled tail
            oe[dst + i] = spe[sp + i - cap];
            if (ow) ow[dst + i] = spw[sp + i - cap];
        }
    }
}

__global__ void k_offsets(int64_t n_samples, int64_t n_chunks, const int64_t *__restrict__ dest,
                          int64_t *__restrict__ offsets)
{
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s <= n_samples) offsets[s] = dest[s * n_chunks];
}

// diagnostics: fn 0 = fm_log(x), 1 = fm_log1p(x), 2 = -fm_log(u01(k)) with k = (uint32)x
__global__ void __launch_bounds__(256) k_debug_eval(int fn, int64_t n, const double *__restrict__ in,
                                                    double *__restrict__ out)
{
    load_logtab();
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double x = in[i];
    double y;
    const SmemLogTab T;
    if (fn == 0) y = fm_log(x, T);
    else if (fn == 1) y = fm_log1p(x, T);
    else y = -fm_log(u01((uint32_t)x), T);
    out[i] = y;
}

// host: the log table, computed once in long double (logc = -log(invc) to ~2^-64 relative)
LogTable make_log_table()
{
    LogTable T;
    for (int i = 0; i < kLogTable; i++) {
        long double c;
        if (i < 80) c = 0.6875L + ((long double)i + 0.5L) / 256.0L;  // z in [0.6875, 1), width 1/256
        else c = 1.0L + ((long double)(i - 80) + 0.5L) / 128.0L;     // z in [1, 1.375), width 1/128
        if (i == 79 || i == 80) c = 1.0L;                             // the two intervals touching 1
        const double invc = (double)(1.0L / c);
        const long double L = -logl((long double)invc);
        const double hi = (double)(roundl(L * 0x1p43L) * 0x1p-43L);  // multiple of 2^-43
        T.ic[i] = make_double2(invc, hi);
        T.logc_lo[i] = (double)(L - (long double)hi);
    }
    return T;
}

std::mutex g_tab_mu;
bool g_tab_done[64] = {false};

}  // namespace

cudaError_t ensure_log_table(cudaStream_t st)
{
    (void)st;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lk(g_tab_mu);
    if (dev < 64 && g_tab_done[dev]) return cudaSuccess;
    static const LogTable T = make_log_table();
    e = cudaMemcpyToSymbol(g_logtab, &T, sizeof(T));
    if (e == cudaSuccess && dev < 64) g_tab_done[dev] = true;
    return e;
}

// the sampler is instantiated for several register budgets (min resident blocks per SM);
// FM_SAMPLE_MINB selects one at run time (tuning), default per model
template <int kModel, int kMinB>
static cudaError_t launch_sample_t(const SampleArgs &a, cudaStream_t st)
{
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_sample<kModel, kMinB>, kThreads, 0);
    int64_t blocks = (int64_t)sms * (per > 0 ? per : 1);
    const int64_t need = (a.n_tasks + kThreads - 1) / kThreads;  // at most one task per lane at start
    if (need < blocks) blocks = need;
    count_launch();
    k_sample<kModel, kMinB><<<(unsigned)blocks, kThreads, 0, st>>>(a);
    return cudaGetLastError();
}

template <int kModel>
static cudaError_t launch_sample_m(int minb, const SampleArgs &a, cudaStream_t st)
{
    switch (minb) {
    case 1: return launch_sample_t<kModel, 1>(a, st);
    case 2: return launch_sample_t<kModel, 2>(a, st);
    case 4: return launch_sample_t<kModel, 4>(a, st);
    default: return launch_sample_t<kModel, 3>(a, st);
    }
}

cudaError_t launch_sample(int model, const SampleArgs &a, cudaStream_t st)
{
    if (a.n_tasks <= 0) return cudaSuccess;
    cudaError_t e = ensure_log_table(st);
    if (e != cudaSuccess) return e;
    e = cudaMemsetAsync(a.task_counter, 0, sizeof(unsigned long long), st);
    if (e != cudaSuccess) return e;
    if (a.spill_counter && !a.rerun_base) {
        e = cudaMemsetAsync(a.spill_counter, 0, sizeof(unsigned long long), st);
        if (e != cudaSuccess) return e;
    }
    const char *ev = getenv("FM_SAMPLE_MINB");
    const int minb = ev && *ev ? atoi(ev) : (model == FM_UBCM ? 3 : 2);
    return model == FM_UBCM ? launch_sample_m<FM_UBCM>(minb, a, st) : launch_sample_m<FM_ECM>(minb, a, st);
}

cudaError_t launch_overflow(int64_t n_tasks, int64_t n_chunks, const int64_t *chunk_cap, const int64_t *counts,
                            const int64_t *spill_off, unsigned long long *n_overflow, int64_t *overflow_list,
                            cudaStream_t st)
{
    if (n_tasks <= 0) return cudaSuccess;
    count_launch();
    k_overflow<<<(unsigned)((n_tasks + 255) / 256), 256, 0, st>>>(n_tasks, n_chunks, chunk_cap, counts, spill_off,
                                                                 n_overflow, overflow_list);
    return cudaGetLastError();
}

cudaError_t launch_compact(int64_t total, int64_t n_tasks, int64_t n_chunks, int64_t cap_per_sample,
                           const int64_t *chunk_cap, const int64_t *counts, const int64_t *dest,
                           const int64_t *spill_off, const int2 *scratch_e, const int32_t *scratch_w,
                           const int2 *spill_e, const int32_t *spill_w, int2 *out_e, int32_t *out_w, cudaStream_t st)
{
    if (n_tasks <= 0 || total <= 0) return cudaSuccess;
    count_launch();
    k_compact<<<(unsigned)((n_tasks + kCopyThreads - 1) / kCopyThreads), kCopyThreads, 0, st>>>(
        n_tasks, n_chunks, cap_per_sample, chunk_cap, counts, dest, spill_off, scratch_e, scratch_w, spill_e, spill_w,
        out_e, out_w);
    return cudaGetLastError();
}

cudaError_t launch_offsets(int64_t n_samples, int64_t n_chunks, const int64_t *dest, int64_t *offsets, cudaStream_t st)
{
    count_launch();
    k_offsets<<<(unsigned)((n_samples + 1 + 255) / 256), 256, 0, st>>>(n_samples, n_chunks, dest, offsets);
    return cudaGetLastError();
}

cudaError_t launch_debug_eval(int fn, int64_t n, const double *in, double *out, cudaStream_t st)
{
    cudaError_t e = ensure_log_table(st);
    if (e != cudaSuccess) return e;
    if (n <= 0) return cudaSuccess;
    count_launch();
    k_debug_eval<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(fn, n, in, out);
    return cudaGetLastError();
}

}  // namespace fm
