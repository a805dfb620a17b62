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

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <mutex>

#include "fm_internal.cuh"
#include "fm_math.cuh"
#include "fm_plan_kernels.cuh"

namespace fm {

__device__ LogTable g_logtab;
#ifdef FM_TRACE
// per-warp timeline of the last sampler launch (instrumentation build, scripts/trace_run.py):
// start, first time the task queue was exhausted for the warp, end (globaltimer ns), iterations,
// iterations after exhaustion, SM id
__device__ unsigned long long g_trace[4096][6];
__device__ __forceinline__ unsigned long long gtimer()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ unsigned smid()
{
    unsigned r;
    asm volatile("mov.u32 %0, %smid;" : "=r"(r));
    return r;
}
#endif

namespace {

#ifndef FM_SAMPLE_THREADS
#define FM_SAMPLE_THREADS 256
#endif
#ifndef FM_SAMPLE_MINB_UBCM
#define FM_SAMPLE_MINB_UBCM 3
#endif
#ifndef FM_SAMPLE_MINB_ECM
#define FM_SAMPLE_MINB_ECM 3
#endif
#ifndef FM_SAMPLE_MINB_RANKOUT  // UBCM rank-out path (N >= 2^21: DRAM-latency-bound gathers)
#define FM_SAMPLE_MINB_RANKOUT 4
#endif
constexpr int kThreads = FM_SAMPLE_THREADS;  // threads per block of the sampler
constexpr int kBatch = 64;  // tasks per warp batch

// per-block copy of the log table: (invc, logc) pairs, one 16-byte lookup (8 conflict-free
// copies, one per bank group, measured no faster: the lookups are not the bottleneck)
struct LogSmem {
    double2 ic[kLogTable];
};
__shared__ __align__(16) LogSmem s_log;
struct SmemLogTab {
    const LogConsts &lc;  // in the kernel's parameter bank: constant-bank operands, no register copies
    uint32_t base;        // 32-bit shared address of s_log (opaque: one register, no per-use address math)
    __device__ __forceinline__ void entry(int i, double &invc, double &logc) const
    {
        asm("ld.shared.v2.f64 {%0,%1}, [%2];" : "=d"(invc), "=d"(logc) : "r"(base + ((uint32_t)i << 4)));
    }
    __device__ __forceinline__ const LogConsts &C() const { return lc; }
};

// fill s_log; returns this lane's column address, produced after the barrier (so no table read
// is scheduled before the table is complete)
__device__ __forceinline__ uint32_t load_logtab()
{
    for (int j = threadIdx.x; j < kLogTable; j += blockDim.x) s_log.ic[j] = g_logtab.ic[j];
    __syncthreads();
    uint32_t base = (uint32_t)__cvta_generic_to_shared(&s_log);
    asm volatile("mov.b32 %0, %0;" : "+r"(base));
    return base;
}

// kC independent chains (lane-chunk tasks) per thread, interleaved for instruction-level
// parallelism (instantiated with kC = 1: two chains measured slower, their registers cost more
// occupancy than their ILP gains).
// kStats: statistics mode (fm_sample_degrees): degree / strength sums instead of edge lists.
// kGather (UBCM): 0 = kappa and id from two arrays, 1 = one 16-byte (kappa, id) record, 2 = kappa
// only: the scratch edge holds (row id, candidate RANK) and the compaction maps the rank to its id
// (the id gather leaves the latency-bound chain for the bandwidth-bound copy).
// kOrdered: bipartite / directed output (row id, candidate id) as is (R16).
// kCheck (FM_DEBUG_CHECKS=1): every landed candidate checks the contract p <= q (1 + 2^-50)
// (DESIGN R13) and flags kErrBound -- the call then fails with FM_ERR_BOUND.
template <int kModel, int kMinBlocks, int kC, bool kStats, bool kRefresh, int kGather, bool kOrdered, bool kCheck>
__global__ void __launch_bounds__(kThreads, kMinBlocks) k_sample(const SampleArgs A)
{
    extern __shared__ __align__(16) unsigned char s_dyn[];  // per-chain prefetch slots
    // rarely used per-chain task state lives in shared memory (registers are the occupancy limit)
    __shared__ int64_t s_task[kThreads * kC];   // current task id, -1 none
    __shared__ int64_t s_spill[kThreads * kC];  // its spill region: -1 none, -2 failed
    // 64-bit per-thread draw / accepted counters: the 32-bit registers below are added here at
    // every task end (a statistics call over many samples passes 2^32 per warp)
    __shared__ unsigned long long s_ndraw[kThreads], s_nacc[kThreads];
    // UBCM: the last < 4 accepted edges of each lane's slot, so that the slot is written in whole
    // 32-byte sectors (structure of arrays: conflict-free)
    __shared__ int2 s_eb[kModel == FM_UBCM ? 4 : 1][kThreads];
    const bool buf4 = kModel == FM_UBCM && A.buf4 && !A.rerun_base && !kStats;
    // ECM: the scratch holds one 16-byte (src, dst, w, 0) record per edge, written two per sector
    // (the lane's previous record waits in shared memory); the compaction splits the records into
    // the edge and weight arrays (separate 8- and 4-byte stores wrote two partial sectors per edge)
    __shared__ int4 s_er[kModel == FM_ECM ? kThreads : 1];
    const bool aos = kModel == FM_ECM && A.buf4 && !A.rerun_base && !kStats;
    const SmemLogTab T{A.lc, load_logtab()};
    const int lane = threadIdx.x & 31;
    const uint32_t lt = (1u << lane) - 1u;
    const int64_t n_tasks = A.n_tasks_dev ? (int64_t)*A.n_tasks_dev : A.n_tasks;

    // ---- warp batch of task ids [bpos, bend); lane 0 holds the start of the next batch ----
    unsigned long long next_batch = 0;
    if (lane == 0) next_batch = atomicAdd(A.task_counter, (unsigned long long)kBatch);
    int64_t bpos = 0, bend = 0;
    bool warp_done = false;
    // ---- per-chain task state ----
    int2 *eb[kC];  // the task's output slot (scratch, or the final list when re-running)
    int32_t g[kC], g_end[kC], cnt[kC], cap[kC];
    uint32_t s_abs[kC];
    // ---- per-chain segment state ----
    bool act[kC];
    int32_t u[kC], b[kC], cur[kC], id_u[kC], excl[kC];
    uint32_t row_acc[kC];          // statistics mode: accepted edges of the current segment
    unsigned long long row_w[kC];  //                  and their weight sum (ECM)
    uint32_t sg[kC], d[kC], wacc[kC], wwt[kC];
    double xq[kC], dq[kC], h[kC], rh[kC], ku[kC], E[kC], yu[kC], lyu[kC], omT[kC], iomT[kC];
#pragma unroll
    for (int c = 0; c < kC; c++) {
        s_task[threadIdx.x * kC + c] = -1;
        s_spill[threadIdx.x * kC + c] = -1;
        eb[c] = A.edges;
        g[c] = g_end[c] = cnt[c] = cap[c] = 0;
        s_abs[c] = 0;
        act[c] = false;
        u[c] = b[c] = cur[c] = id_u[c] = 0;
        excl[c] = -1;
        row_acc[c] = 0;
        row_w[c] = 0;
        sg[c] = d[c] = wacc[c] = wwt[c] = 0;
        xq[c] = 0.0; dq[c] = 1.0; h[c] = 0.0; rh[c] = 0.0; ku[c] = 0.0; E[c] = 0.0;
        yu[c] = 0.0; lyu[c] = 0.0; omT[c] = 1.0; iomT[c] = 1.0;
    }
    // draws; landed = draws - segments and accepted = edges are derived by the host (every
    // segment ends with exactly one terminal draw); statistics mode counts accepted edges
    uint32_t n_draw = 0, n_acc = 0;
    s_ndraw[threadIdx.x] = 0;
    s_nacc[threadIdx.x] = 0;
    bool wsat = false, bad_bound = false;

    // segment g[c] of chain c's task becomes current (64/96-byte record; the record of the next
    // segment is prefetched into this chain's shared-memory slot with cp.async)
    // this thread's prefetch slots: 32-bit shared addresses (no generic-address arithmetic)
    // structure of arrays: 16-byte part k of thread t's slot at (k * kThreads + t) * 16, so the
    // 8 lanes of a 16-byte shared access touch 8 consecutive 16-byte words (conflict-free)
    static_assert(kC == 1, "prefetch slot layout assumes one chain per thread");
    constexpr int kPart = 16 * kThreads;
    uint32_t slot0 = (uint32_t)__cvta_generic_to_shared(s_dyn) + threadIdx.x * 16;
    asm volatile("mov.b32 %0, %0;" : "+r"(slot0));  // opaque: held in a register, not recomputed per use
    auto start_seg = [&](const int c, const bool prefetched) {
        const uint32_t my_next = slot0;
        int4 p0, p3;
        double2 p1, p2, p4, p5;
        if (prefetched) {
            // the slot address passes through the wait: the loads below cannot move above it
            uint32_t sa = my_next;
            asm volatile("cp.async.wait_all;\n" : "+r"(sa)::"memory");
            asm("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(p0.x), "=r"(p0.y), "=r"(p0.z), "=r"(p0.w) : "r"(sa));
            asm("ld.shared.v2.f64 {%0,%1}, [%2+%3];" : "=d"(p1.x), "=d"(p1.y) : "r"(sa), "n"(kPart));
            asm("ld.shared.v2.f64 {%0,%1}, [%2+%3];" : "=d"(p2.x), "=d"(p2.y) : "r"(sa), "n"(2 * kPart));
            asm("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4+%5];"
                : "=r"(p3.x), "=r"(p3.y), "=r"(p3.z), "=r"(p3.w) : "r"(sa), "n"(3 * kPart));
            if (kModel == FM_ECM) {
                asm("ld.shared.v2.f64 {%0,%1}, [%2+%3];" : "=d"(p4.x), "=d"(p4.y) : "r"(sa), "n"(4 * kPart));
                asm("ld.shared.v2.f64 {%0,%1}, [%2+%3];" : "=d"(p5.x), "=d"(p5.y) : "r"(sa), "n"(5 * kPart));
            }
        } else {
            const SegRec *r = reinterpret_cast<const SegRec *>(A.rec + (size_t)g[c] * kRecStride(kModel));
            p0 = *reinterpret_cast<const int4 *>(r);
            p1 = *reinterpret_cast<const double2 *>(&r->h0);
            p2 = *reinterpret_cast<const double2 *>(&r->d0);
            p3 = *reinterpret_cast<const int4 *>(&r->id_u);
            if (kModel == FM_ECM) {
                p4 = *reinterpret_cast<const double2 *>(&r->yu);
                p5 = *reinterpret_cast<const double2 *>(&r->omT);
            }
        }
        u[c] = p0.x;
        cur[c] = p0.y - 1;  // virtual previous position a-1 (R3)
        b[c] = p0.z;
        sg[c] = (uint32_t)p0.w;
        h[c] = p1.x;
        xq[c] = p1.y;
        dq[c] = p2.x;
        ku[c] = p2.y;
        id_u[c] = p3.x;
        excl[c] = p3.y;  // directed: u's own in-copy (R16), else -1
        rh[c] = __hiloint2double(p3.w, p3.z);
        if (kModel == FM_ECM) {
            yu[c] = p4.x;
            lyu[c] = p4.y;
            omT[c] = p5.x;
            iomT[c] = p5.y;
        }
        d[c] = 0;
        g[c]++;
        act[c] = true;
        if (g[c] < g_end[c]) {
            const unsigned char *src = A.rec + (size_t)g[c] * kRecStride(kModel);
            constexpr int parts = kModel == FM_ECM ? 6 : 4;
#pragma unroll
            for (int k = 0; k < parts; k++)
                asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(my_next + kPart * k), "l"(src + 16 * k)
                             : "memory");
            asm volatile("cp.async.commit_group;\n" ::: "memory");
        }
    };
    auto U01 = [](uint32_t k) { return kModel == FM_UBCM ? u01(k) : u01_cvt(k); };
    // u01 of the skip word, and the accept/weight words, of chain c's draw d[c] (R1, R2)
    auto draw_u = [&](const int c) {
        uint32_t ws;
        if (kModel == FM_UBCM) {
            const uint4 W = philox4x32_10(make_uint4(d[c] >> 1, sg[c], (uint32_t)u[c], s_abs[c]), A.key);
            ws = (d[c] & 1) ? W.z : W.x;
            wacc[c] = (d[c] & 1) ? W.w : W.y;
        } else {
            const uint4 W = philox4x32_10(make_uint4(d[c], sg[c], (uint32_t)u[c], s_abs[c]), A.key);
            ws = W.x;
            wacc[c] = W.y;
            wwt[c] = W.z;
        }
        return U01(ws);
    };

#ifdef FM_TRACE
    const unsigned long long tr_t0 = gtimer();
    unsigned long long tr_done = 0, tr_it = 0, tr_it_done = 0;
#endif
    for (;;) {
#ifdef FM_TRACE
        tr_it++;
        if (warp_done) {
            tr_it_done++;
            if (!tr_done) tr_done = gtimer();
        }
#endif
        // ---- 1. task management (only when a chain of the warp has no segment left; a single
        //      vote otherwise): such chains take the next task ids of the warp's batch (the next
        //      batch is requested as soon as one is opened) ----
        bool fresh[kC];
        bool need_any = false;
#pragma unroll
        for (int c = 0; c < kC; c++) {
            fresh[c] = false;
            need_any = need_any || !act[c];
        }
        if (__any_sync(0xffffffffu, need_any)) {
#pragma unroll
        for (int c = 0; c < kC; c++) {
            const bool needc = !act[c];
            const int ci = threadIdx.x * kC + c;
            if (needc) {
                const int64_t tk = s_task[ci];
                if (tk >= 0) {
                    if (buf4) {  // the slot's last partial sector
                        const int32_t n1 = min(cnt[c], cap[c]);
                        for (int j = 0; j < (n1 & 3); j++) {
                            eb[c][(n1 & ~3) + j] = s_eb[j][threadIdx.x];
                        }
                    }
                    if (aos) {
                        const int32_t n1 = min(cnt[c], cap[c]);
                        if (n1 & 1) reinterpret_cast<int4 *>(A.edges)[(eb[c] - A.edges) + n1 - 1] = s_er[threadIdx.x];
                    }
                    if (!A.rerun_base && !kStats) {
                        A.counts[tk] = cnt[c];
                        A.spill_off[tk] = s_spill[ci];
                    }
                    s_task[ci] = -1;
                    s_ndraw[threadIdx.x] += n_draw;
                    s_nacc[threadIdx.x] += n_acc;
                    n_draw = n_acc = 0;
                }
            }
            const uint32_t nc = __ballot_sync(0xffffffffu, needc && !warp_done);
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
                if (needc && !warp_done && my < n_tasks) {
                    int64_t t = A.task_list ? A.task_list[my] : my;
                    if (A.il_s[0] > 0 && !A.task_list) {  // chunk-major queue -> canonical task index
                        const int kq = my < A.tm.t_split ? 0 : 1;
                        const int64_t m = kq ? my - A.tm.t_split : my, ns = A.il_s[kq];
                        const int64_t cq = m / ns;
                        t = (kq ? A.tm.t_split : 0) + (m - cq * ns) * A.tm.n_chunks[kq] + cq;
                    }
                    int64_t s, ch;
                    int kk;
                    task_decode(A.tm, t, s, ch, kk);
                    s_task[ci] = t;
                    g[c] = (int32_t)A.tm.seg[kk][ch];
                    g_end[c] = (int32_t)A.tm.seg[kk][ch + 1];
                    if (A.rerun_base) {
                        const int64_t sl = A.rerun_base[t];
                        eb[c] = A.edges + sl;
                        cap[c] = (int32_t)max((int64_t)0, min((int64_t)INT32_MAX, A.out_cap - sl));  // bounded by the list
                    } else {
                        eb[c] = A.edges + (s * A.tm.cap_per_sample + A.tm.cap[kk][ch]);
                        cap[c] = (int32_t)(A.tm.cap[kk][ch + 1] - A.tm.cap[kk][ch]);
                    }
                    s_abs[c] = A.first_sample + (uint32_t)s;
                    cnt[c] = 0;
                    s_spill[ci] = -1;
                    if (g[c] < g_end[c]) {
                        start_seg(c, false);
                        fresh[c] = true;
                    }
                }
                if (bpos >= n_tasks) warp_done = true;
            }
        }
        bool any_act = false;
#pragma unroll
        for (int c = 0; c < kC; c++) any_act = any_act || act[c];
        if (!__any_sync(0xffffffffu, any_act)) {
            if (warp_done) break;
            continue;
        }
        }
        // ---- 2. a freshly fetched task consumes no draw this iteration: like a restarted chain,
        //      it only computes E of its draw 0 in the convergent block 4+5 ----
        // ---- 3. consume one draw per chain ----
        bool landed[kC];
        uint32_t w_land[kC], w_wt[kC];
        double kv[kC], yv[kC], lyv[kC], ymn[kC];
        int32_t id_v[kC];
        double idd[kC];  // the record word holding the id (low half), see the ECM block below
#pragma unroll
        for (int c = 0; c < kC; c++) {
            landed[c] = false;
            w_land[c] = w_wt[c] = 0;
            // kv and id_v are left undefined unless the draw lands: a defined "else" value makes
            // the compiler copy the gathered register at the branch merge, i.e. wait for the
            // gather there instead of at its first use (ncu: long-scoreboard stall).  ECM keeps
            // them defined: undefined (or gathered after the merge) they cost a register spill
            // at 24 warps/SM and measured slower
            if (kModel == FM_ECM) {
                kv[c] = yv[c] = lyv[c] = 0.0;
                id_v[c] = 0;
                idd[c] = 0.0;
                ymn[c] = 0.0;
            }
            if (act[c] && !fresh[c]) {
                n_draw++;
                const double R = div_markstein(E[c], h[c], rh[c]);  // = E / h, IEEE
                // R < lim (lim = b-1-cur >= 0 an integer) <=> R < 2^31 and floor(R) < lim, with
                // floor(R) the low word of RZ(R + 2^52) (exact for 0 <= R < 2^52): no I2F / F2I
                const double Rt = __dadd_rz(R, 0x1p52);
                const int32_t fl = __double2loint(Rt);
                const bool step = R < 2147483648.0 && fl < b[c] - 1 - cur[c];
                if (!step) {  // terminal draw (R5)
                    if (kStats && row_acc[c] && A.deg_row) {  // statistics mode: flush the row node's sums
                        atomicAdd(&A.deg_row[id_u[c]], (unsigned long long)row_acc[c]);
                        if (kModel == FM_ECM) atomicAdd(&A.str_row[id_u[c]], row_w[c]);
                        row_acc[c] = 0;
                        row_w[c] = 0;
                    }
                    if (g[c] < g_end[c]) start_seg(c, true);
                    else act[c] = false;
                } else {
                    cur[c] = cur[c] + 1 + fl;  // floor(R)
                    // ECM: one 32-byte record per candidate (Plan::cand); id needed only if accepted
                    if (kModel == FM_ECM) {
                        const double2 v0 = __ldg(A.cand + 2 * (uint32_t)cur[c]);
                        const double2 v1 = __ldg(A.cand + 2 * (uint32_t)cur[c] + 1);
                        kv[c] = v0.x;
                        yv[c] = v0.y;
                        lyv[c] = v1.x;
                        idd[c] = v1.y;
                        if (kRefresh) ymn[c] = __ldg(A.ymax_c + cur[c] + 1);
                    } else if (kGather == 2) {  // UBCM: κ only, the id is mapped in the compaction
                        kv[c] = A.kappa_s[cur[c]];
                    } else if (kGather == 1) {  // UBCM, large N: one 16-byte record (κ, π): one DRAM access
                        const double2 v0 = __ldg(A.cand + (uint32_t)cur[c]);
                        kv[c] = v0.x;
                        idd[c] = v0.y;
                    } else {  // UBCM, L2-resident arrays: two plain gathers (measured no slower)
                        kv[c] = A.kappa_s[cur[c]];
                        id_v[c] = A.perm[cur[c]];
                    }
                    // directed: the row's own in-copy is skipped with p = 0, bound kept (R16)
                    landed[c] = cur[c] != excl[c];
                    w_land[c] = wacc[c];
                    w_wt[c] = wwt[c];
                    d[c]++;
                }
            }
        }
        // ---- 4+5. per chain, one straight-line block: RNG + E of the next draw (overlaps the
        //      k[cur] gather) and the p/q test of the landed candidate (restarted chains
        //      evaluate a dummy X = 1 and keep their h0, x0, d0) ----
        bool acc[kC];
        int32_t w[kC];
#pragma unroll
        for (int c = 0; c < kC; c++) {
            acc[c] = false;
            w[c] = 1;
            if (act[c]) {
                const double us = draw_u(c);
                // (kv + 0*us) orders the use of the gathered kv after the Philox rounds above, so
                // the gather latency hides behind them while the two logarithms below (E of the
                // next draw, log1p of this candidate) stay independent; exact since us in (0,1)
                // (kv is read only if landed: the ?: evaluates the selected operand only)
                const double Enew = -fm_log(us, T);
                const double ord = us;  // (ordering after E of the next draw instead measured no faster)
                if (kModel == FM_UBCM) {
                    double ordu = ord;
                    if (kGather == 1)  // the record's unused high id word read here (see the ECM block)
                        ordu = __dadd_rn(ord, __hiloint2double(__double2hiint(idd[c]), 0));
                    const double X = landed[c] ? __dmul_rn(ku[c], __dadd_rn(kv[c], __dmul_rn(ordu, 0.0))) : 1.0;
                    const double D = __dadd_rn(1.0, X);
                    const double hn = fm_log1p(X, T);
                    if (landed[c]) {  // accept iff u < (X/D) / (xq/dq), cross-multiplied (R10)
                        if (kCheck && __dmul_rn(X, dq[c]) > __dmul_rn(__dmul_rn(xq[c], D), 1.0 + 0x1p-50))
                            bad_bound = true;  // p > q (1 + 2^-50): the bound is violated
                        acc[c] = __dmul_rn(__dmul_rn(U01(w_land[c]), xq[c]), D) < __dmul_rn(X, dq[c]);
                        xq[c] = X;
                        dq[c] = D;
                        h[c] = hn;
                        rh[c] = __drcp_rn(hn);
                    }
                } else {
                    // (us + hid) * 0: hid = the record's unused high id word (zero) as a double, "read"
                    // here where the gather is awaited anyway -- left dead, its register was reused
                    // right after the gather and the write-after-write wait on the in-flight load
                    // stalled every warp before Philox (15 % of the ECM kernel's stall samples)
                    const double hid = __hiloint2double(__double2hiint(idd[c]), 0);
                    const double z = landed[c] ? __dmul_rn(ku[c], __dadd_rn(kv[c], __dmul_rn(__dadd_rn(ord, hid), 0.0)))
                                               : 1.0;
                    // (yv + 0*us), like kv: the gathered y is used only after the Philox rounds (the
                    // plain product was scheduled first and stalled every warp on the gather:
                    // 20 % of the ECM kernel's stall samples)
                    const double t = __dmul_rn(yu[c], __dadd_rn(yv[c], __dmul_rn(ord, 0.0)));
                    const double Dp = __dadd_rn(__dsub_rn(1.0, t), z);
                    // the bound for the candidates still ahead: per segment 1 - T = omT, or (kRefresh,
                    // R17) per reached candidate 1 - y_u Ymax[cur+1]
                    double omb = omT[c], iomb = iomT[c];
                    if (kRefresh && landed[c]) {
                        omb = __dsub_rn(1.0, __dmul_rn(yu[c], __dadd_rn(ymn[c], __dmul_rn(ord, 0.0))));  // (ordered too)
                        iomb = __drcp_rn(omb);
                    }
                    const double hn = fm_log1p(__dmul_rn(z, iomb), T);
                    if (landed[c]) {
                        if (kCheck && __dmul_rn(z, dq[c]) > __dmul_rn(__dmul_rn(xq[c], Dp), 1.0 + 0x1p-50))
                            bad_bound = true;  // p > q_hat (1 + 2^-50)
                        acc[c] = __dmul_rn(__dmul_rn(U01(w_land[c]), xq[c]), Dp) < __dmul_rn(z, dq[c]);
                        xq[c] = z;
                        dq[c] = __dadd_rn(omb, z);
                        h[c] = hn;
                        rh[c] = __drcp_rn(hn);
                        if (acc[c]) {  // Eq. 5 weight, log t = log y_u + log y_v (R8)
                            const double lu = fm_log(U01(w_wt[c]), T);
                            const double G = floor(__ddiv_rn(lu, __dadd_rn(lyu[c], lyv[c])));
                            if (G <= 2147483646.0) {
                                w[c] = 1 + (int32_t)G;
                            } else {
                                w[c] = INT32_MAX;
                                wsat = true;
                            }
                        }
                    }
                }
                E[c] = Enew;
            }
        }
        // ---- 6. append accepted edges to the tasks' slots, in draw order ----
#pragma unroll
        for (int c = 0; c < kC; c++) {
            if (kModel == FM_ECM || kGather == 1) id_v[c] = __double2loint(idd[c]);
            if (kStats && acc[c]) {  // statistics mode (NEXT-3): degrees/strengths, no edge list
                if (A.deg_row) {
                    row_acc[c]++;
                    atomicAdd(&A.deg_col[id_v[c]], 1ull);
                    if (kModel == FM_ECM) {
                        row_w[c] += (unsigned long long)w[c];
                        atomicAdd(&A.str_col[id_v[c]], (unsigned long long)w[c]);
                    }
                }
                // rich club: the edge lies within the top-m nodes iff its larger rank cur < m
                if (A.rank_hist) atomicAdd(&A.rank_hist[cur[c]], 1ull);
                n_acc++;
            } else if (acc[c]) {
                const int2 ev = kGather == 2 ? make_int2(id_u[c], cur[c])  // (row id, candidate rank)
                                : kOrdered  ? make_int2(id_u[c], id_v[c])
                                            : make_int2(min(id_u[c], id_v[c]), max(id_u[c], id_v[c]));
                if (cnt[c] < cap[c]) {
                    if (buf4) {
                        const int k = cnt[c] & 3;
                        if (k < 3) {
                            s_eb[k][threadIdx.x] = ev;
                        } else {  // a whole sector: edges cnt-3 .. cnt
                            const int2 e0 = s_eb[0][threadIdx.x], e1 = s_eb[1][threadIdx.x], e2 = s_eb[2][threadIdx.x];
                            // two 16-byte stores to one sector (one 256-bit STG.256 measured 1 % slower)
                            int4 *q = reinterpret_cast<int4 *>(eb[c] + (cnt[c] - 3));
                            if (kGather == 2) {  // large N: evict-first, the L2 keeps the kappa gather target (-0.7 %)
                                __stcs(q, make_int4(e0.x, e0.y, e1.x, e1.y));
                                __stcs(q + 1, make_int4(e2.x, e2.y, ev.x, ev.y));
                            } else {
                                q[0] = make_int4(e0.x, e0.y, e1.x, e1.y);
                                q[1] = make_int4(e2.x, e2.y, ev.x, ev.y);
                            }
                        }
                    } else if (aos) {
                        const int4 rec = make_int4(ev.x, ev.y, w[c], 0);
                        if ((cnt[c] & 1) == 0) {
                            s_er[threadIdx.x] = rec;
                        } else {  // records cnt-1, cnt: one sector
                            int4 *q = reinterpret_cast<int4 *>(A.edges) + ((eb[c] - A.edges) + cnt[c] - 1);
                            q[0] = s_er[threadIdx.x];
                            q[1] = rec;
                        }
                    } else {
                        eb[c][cnt[c]] = ev;
                        if (kModel == FM_ECM) A.weights[(eb[c] - A.edges) + cnt[c]] = w[c];
                    }
                } else if (!A.rerun_base && cnt[c] < 2 * cap[c]) {  // spill: one extra region of `cap`
                    const int ci = threadIdx.x * kC + c;
                    int64_t sp = s_spill[ci];
                    if (sp == -1) {
                        const unsigned long long o = atomicAdd(A.spill_counter, (unsigned long long)cap[c]);
                        sp = (int64_t)(o + cap[c]) <= A.spill_cap ? (int64_t)o : -2;
                        s_spill[ci] = sp;
                    }
                    if (sp >= 0) {
                        A.spill_e[sp + cnt[c] - cap[c]] = ev;
                        if (kModel == FM_ECM) A.spill_w[sp + cnt[c] - cap[c]] = w[c];
                    }
                }
                cnt[c]++;
            }
        }
    }
#ifdef FM_TRACE
    if (lane == 0 && !A.rerun_base) {
        const int wi = blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5);
        if (wi < 4096) {
            g_trace[wi][0] = tr_t0;
            g_trace[wi][1] = tr_done;
            g_trace[wi][2] = gtimer();
            g_trace[wi][3] = tr_it;
            g_trace[wi][4] = tr_it_done;
            g_trace[wi][5] = smid();
        }
    }
#endif
    if (kCheck && __any_sync(0xffffffffu, bad_bound) && lane == 0) atomicOr(A.flags, kErrBound);
    if (A.rerun_base) return;
    unsigned long long dr = s_ndraw[threadIdx.x] + n_draw, ac = s_nacc[threadIdx.x] + n_acc;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        dr += __shfl_xor_sync(0xffffffffu, dr, o);
        ac += __shfl_xor_sync(0xffffffffu, ac, o);
    }
    const bool anysat = __any_sync(0xffffffffu, wsat);
    if (lane == 0) {
        atomicAdd(&A.counters[0], dr);
        if (kStats) atomicAdd(&A.counters[2], ac);
        if (anysat) atomicOr(A.flags, kFlagWeightSat);
    }
}

__device__ __forceinline__ bool task_overflowed(int64_t cnt, int64_t cap, int64_t sp)
{
    return cnt > cap && (cnt > 2 * cap || sp < 0);
}

__global__ void __launch_bounds__(256) k_overflow(int64_t n_tasks, const TaskMap tm, const int64_t *__restrict__ counts,
                                                  const int64_t *__restrict__ spill_off, unsigned long long *n_overflow,
                                                  int64_t *__restrict__ overflow_list)
{
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n_tasks) return;
    int64_t s, c;
    int k;
    task_decode(tm, t, s, c, k);
    if (task_overflowed(counts[t], tm.cap[k][c + 1] - tm.cap[k][c], spill_off[t])) {
        const unsigned long long o = atomicAdd(n_overflow, 1ull);
        overflow_list[o] = t;
    }
}

// Gather: block b handles tasks [256 b, 256 b + 256): their metadata is staged in shared memory
// by one coalesced pass, then each warp copies 32 of the tasks (slot, then spill part),
// 4 elements per lane in flight.  Overflowed tasks are skipped (re-run into the final array).
constexpr int kCopyThreads = 256;
#ifndef FM_COPY_UNROLL
#define FM_COPY_UNROLL 4
#endif
constexpr int kCU = FM_COPY_UNROLL;  // elements per lane in flight
template <bool kMap, bool kRec>
__global__ void __launch_bounds__(kCopyThreads) k_compact(int64_t n_tasks, const TaskMap tm,
                                                          const int64_t *__restrict__ counts,
                                                          const int64_t *__restrict__ dest,
                                                          const int64_t *__restrict__ spill_off,
                                                          const int2 *__restrict__ se, const int32_t *__restrict__ sw,
                                                          const int2 *__restrict__ spe, const int32_t *__restrict__ spw,
                                                          int2 *__restrict__ oe, int32_t *__restrict__ ow,
                                                          int64_t out_cap, const int32_t *__restrict__ rank_map,
                                                          int ordered)
{
    // rank_map: the scratch holds (row id, candidate rank): map the rank to its id and orient
    auto fin = [&](int2 v) -> int2 {
        if (!kMap) return v;
        const int32_t id = __ldg(rank_map + v.y);
        return ordered ? make_int2(v.x, id) : make_int2(min(v.x, id), max(v.x, id));
    };
    __shared__ int64_t s_src[kCopyThreads], s_dst[kCopyThreads], s_sp[kCopyThreads];
    __shared__ int32_t s_cnt[kCopyThreads], s_cap[kCopyThreads];
    const int64_t t0 = (int64_t)blockIdx.x * kCopyThreads;
    {
        const int64_t t = t0 + threadIdx.x;
        int32_t cn = 0, cp = 0;
        int64_t src = 0, dst = 0, sp = -1;
        if (t < n_tasks) {
            int64_t s, c;
            int k;
            task_decode(tm, t, s, c, k);
            const int64_t cap = tm.cap[k][c + 1] - tm.cap[k][c];
            const int64_t cnt = counts[t];
            sp = spill_off[t];
            dst = dest[t];
            // tasks that would land beyond the list are dropped: the host sees the total and redoes the write
            cn = task_overflowed(cnt, cap, sp) || dst + cnt > out_cap ? 0 : (int32_t)cnt;
            cp = (int32_t)cap;
            src = s * tm.cap_per_sample + tm.cap[k][c];
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
        if (kRec) {  // ECM 16-byte records (src, dst, w, 0) -> edge and weight arrays
            const int4 *sr = reinterpret_cast<const int4 *>(se);
            for (int32_t i0 = 0; i0 < n1; i0 += 32 * kCU) {
                int4 v[kCU];
#pragma unroll
                for (int j = 0; j < kCU; j++) {
                    const int32_t i = i0 + j * 32 + lane;
                    if (i < n1) v[j] = sr[src + i];
                }
#pragma unroll
                for (int j = 0; j < kCU; j++) {
                    const int32_t i = i0 + j * 32 + lane;
                    if (i < n1) {
                        oe[dst + i] = make_int2(v[j].x, v[j].y);
                        ow[dst + i] = v[j].z;
                    }
                }
            }
        }
        for (int32_t i0 = 0; i0 < (kRec ? 0 : n1); i0 += 32 * kCU) {
            int2 v[kCU];
#pragma unroll
            for (int j = 0; j < kCU; j++) {
                const int32_t i = i0 + j * 32 + lane;
                if (i < n1) v[j] = kMap ? __ldcs(se + src + i) : se[src + i];  // (map: keep L2 for rank_map)
            }
            if (kMap) {
#pragma unroll
                for (int j = 0; j < kCU; j++) {
                    const int32_t i = i0 + j * 32 + lane;
                    if (i < n1) v[j] = fin(v[j]);
                }
            }
#pragma unroll
            for (int j = 0; j < kCU; j++) {
                const int32_t i = i0 + j * 32 + lane;
                if (i < n1) {
                    if (kMap) __stcs(oe + dst + i, v[j]);
                    else oe[dst + i] = v[j];
                }
            }
            if (ow) {
                int32_t x[kCU];
#pragma unroll
                for (int j = 0; j < kCU; j++) {
                    const int32_t i = i0 + j * 32 + lane;
                    if (i < n1) x[j] = sw[src + i];
                }
#pragma unroll
                for (int j = 0; j < kCU; j++) {
                    const int32_t i = i0 + j * 32 + lane;
                    if (i < n1) ow[dst + i] = x[j];
                }
            }
        }
        for (int32_t i = cap + lane; i < cnt; i += 32) {  // spilled tail
            oe[dst + i] = fin(spe[sp + i - cap]);
            if (ow) ow[dst + i] = spw[sp + i - cap];
        }
    }
}

__global__ void k_offsets(int64_t n_samples, const TaskMap tm, const int64_t *__restrict__ dest,
                          int64_t *__restrict__ offsets)
{
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s > n_samples) return;
    const int64_t t0 = s <= tm.s_split ? s * tm.n_chunks[0] : tm.t_split + (s - tm.s_split) * tm.n_chunks[1];
    offsets[s] = dest[t0];  // dest[n_tasks] is the total
}

__global__ void k_add_u64(const uint64_t *__restrict__ in, uint64_t *__restrict__ out, int64_t n)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] += in[i];
}

// diagnostics: fn 0 = fm_log(x), 1 = fm_log1p(x), 2 = -fm_log(u01(k)) with k = (uint32)x,
// 3 = in[2i] / in[2i+1] by div_markstein with the reciprocal the sampler uses
__global__ void __launch_bounds__(256) k_debug_eval(int fn, int64_t n, const double *__restrict__ in,
                                                    double *__restrict__ out, const LogConsts lc)
{
    const SmemLogTab T{lc, load_logtab()};
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    if (fn == 3) {
        const double b = in[2 * i + 1];
        out[i] = div_markstein(in[2 * i], b, __drcp_rn(b));
        return;
    }
    const double x = in[i];
    double y;
    if (fn == 0) y = fm_log(x, T);
    else if (fn == 1) y = fm_log1p(x, T);
    else y = -fm_log(u01((uint32_t)x), T);
    out[i] = y;
}

// host: the log table, computed once in long double (logc = RN(-log(invc)))
LogTable make_log_table()
{
    LogTable T;
    for (int i = 0; i < kLogTable; i++) {
        long double c;
        if (i < 80) c = 0.6875L + ((long double)i + 0.5L) / 256.0L;  // z in [0.6875, 1), width 1/256
        else c = 1.0L + ((long double)(i - 80) + 0.5L) / 128.0L;     // z in [1, 1.375), width 1/128
        if (i == 79 || i == 80) c = 1.0L;                             // the two intervals touching 1
        const double invc = (double)(1.0L / c);
        T.ic[i] = make_double2(invc, (double)(-logl((long double)invc)));
    }
    return T;
}

std::mutex g_tab_mu;
bool g_tab_done[64] = {false};

}  // namespace

#ifdef FM_TRACE
void dump_trace()
{
    static unsigned long long h[4096][6];
    if (cudaMemcpyFromSymbol(h, g_trace, sizeof(h)) != cudaSuccess) return;
    const char *path = getenv("FM_TRACE_FILE");
    FILE *f = fopen(path ? path : "/tmp/fm_trace.bin", "wb");
    if (f) {
        fwrite(h, sizeof(h), 1, f);
        fclose(f);
    }
    static unsigned long long z[4096][6];
    cudaMemcpyToSymbol(g_trace, z, sizeof(z));
}
#endif

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

// one instantiation per (model, statistics mode, ECM bound refresh, UBCM gather record, output
// orientation); kMinB = 3 blocks per SM
template <int kModel, int kMinB, int kC, bool kStats, bool kRefresh, int kGather, bool kOrdered, bool kCheck>
static cudaError_t launch_sample_t(const SampleArgs &a, cudaStream_t st)
{
    auto kern = k_sample<kModel, kMinB, kC, kStats, kRefresh, kGather, kOrdered, kCheck>;
    int dev = 0, sms = 0, per = 0;
    cudaError_t err = cudaGetDevice(&dev);
    if (err == cudaSuccess) err = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (err != cudaSuccess) return err;
    const size_t dyn = (size_t)kThreads * kC * (kModel == FM_ECM ? 96 : 64);
    // function attributes are per device: set once per (instantiation, device), thread-safe
    static std::mutex attr_mu;
    static bool attr_set[kMaxDevices] = {};
    std::lock_guard<std::mutex> attr_lk(attr_mu);
    if (dev >= kMaxDevices) return cudaErrorInvalidDevice;
    if (!attr_set[dev]) {
        err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
        if (err != cudaSuccess) return err;
        // shared-memory carveout (percent of the unified L1/shared capacity): the driver's default
        // picked 135 KB of shared memory for 3 x 27 KB of need; 40 % leaves more L1 for the kappa /
        // perm gathers (UBCM kernel -1 %; 0 % starves occupancy: +70 %).  FM_SAMPLE_CARVEOUT
        // overrides (-1 = driver default)
        // (raised to what kMinB blocks need: static + dynamic shared memory + 1 KB reserved each)
        const char *cv = getenv("FM_SAMPLE_CARVEOUT");
        int carve = cv && *cv ? atoi(cv) : 40;
        cudaFuncAttributes fa;
        if (carve >= 0 && cudaFuncGetAttributes(&fa, kern) == cudaSuccess) {
            const size_t need = (size_t)kMinB * (fa.sharedSizeBytes + dyn + 1024);
            const int pct = (int)((need * 100 + 228 * 1024 - 1) / (228 * 1024));
            carve = std::max(carve, std::min(pct, 100));
        }
        if (carve >= 0) {
            err = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, carve);
            if (err != cudaSuccess) return err;
        }
        attr_set[dev] = true;
    }
    err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, kThreads, dyn);
    if (err != cudaSuccess) return err;
    int64_t blocks = (int64_t)sms * (per > 0 ? per : 1);
    const int64_t need = (a.n_tasks + kThreads * kC - 1) / (kThreads * kC);  // <= one task per chain at start
    if (need < blocks) blocks = need;
    count_launch();
    kern<<<(unsigned)blocks, kThreads, dyn, st>>>(a);
    return cudaGetLastError();
}

template <int kModel, bool kStats, bool kRefresh, int kGather, bool kCheck>
static cudaError_t launch_sample_c(const SampleArgs &a, cudaStream_t st)
{
    constexpr int kMinB = kModel == FM_ECM ? FM_SAMPLE_MINB_ECM
                          : kGather == 2   ? FM_SAMPLE_MINB_RANKOUT : FM_SAMPLE_MINB_UBCM;
    // statistics mode writes no pairs: its orientation is irrelevant
    if constexpr (!kStats)
        if (kGather != 2 && a.ordered)
            return launch_sample_t<kModel, kMinB, 1, kStats, kRefresh, kGather, true, kCheck>(a, st);
    return launch_sample_t<kModel, kMinB, 1, kStats, kRefresh, kGather, false, kCheck>(a, st);
}

template <int kModel, bool kStats, bool kRefresh, int kGather>
static cudaError_t launch_sample_o(const SampleArgs &a, cudaStream_t st)
{
    return a.check ? launch_sample_c<kModel, kStats, kRefresh, kGather, true>(a, st)
                   : launch_sample_c<kModel, kStats, kRefresh, kGather, false>(a, st);
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
    // one chain per thread, 3 blocks of 256 per SM (kC = 2, 2 or 4 blocks per SM measured slower)
    const bool stats = a.deg_row != nullptr || a.rank_hist != nullptr;
    if (model == FM_UBCM) {
        if (a.rank_out && !stats && !a.rerun_base) return launch_sample_o<FM_UBCM, false, false, 2>(a, st);
        if (a.cand) return stats ? launch_sample_o<FM_UBCM, true, false, 1>(a, st)
                                 : launch_sample_o<FM_UBCM, false, false, 1>(a, st);
        return stats ? launch_sample_o<FM_UBCM, true, false, 0>(a, st)
                     : launch_sample_o<FM_UBCM, false, false, 0>(a, st);
    }
    if (stats) return launch_sample_o<FM_ECM, true, false, 0>(a, st);
    return a.ymax_c ? launch_sample_o<FM_ECM, false, true, 0>(a, st)
                    : launch_sample_o<FM_ECM, false, false, 0>(a, st);
}

cudaError_t launch_overflow(int64_t n_tasks, const TaskMap &tm, const int64_t *counts, const int64_t *spill_off,
                            unsigned long long *n_overflow, int64_t *overflow_list, cudaStream_t st)
{
    if (n_tasks <= 0) return cudaSuccess;
    count_launch();
    k_overflow<<<(unsigned)((n_tasks + 255) / 256), 256, 0, st>>>(n_tasks, tm, counts, spill_off, n_overflow,
                                                                 overflow_list);
    return cudaGetLastError();
}

cudaError_t launch_compact(int64_t out_cap, int64_t n_tasks, const TaskMap &tm, const int64_t *counts, const int64_t *dest,
                           const int64_t *spill_off, const int2 *scratch_e, const int32_t *scratch_w,
                           const int2 *spill_e, const int32_t *spill_w, int2 *out_e, int32_t *out_w,
                           const int32_t *rank_map, int ordered, int ecm_rec, cudaStream_t st)
{
    if (n_tasks <= 0 || out_cap <= 0) return cudaSuccess;
    count_launch();
    const unsigned grid = (unsigned)((n_tasks + kCopyThreads - 1) / kCopyThreads);
    if (rank_map)
        k_compact<true, false><<<grid, kCopyThreads, 0, st>>>(n_tasks, tm, counts, dest, spill_off, scratch_e,
                                                              scratch_w, spill_e, spill_w, out_e, out_w, out_cap,
                                                              rank_map, ordered);
    else if (ecm_rec)
        k_compact<false, true><<<grid, kCopyThreads, 0, st>>>(n_tasks, tm, counts, dest, spill_off, scratch_e,
                                                              scratch_w, spill_e, spill_w, out_e, out_w, out_cap,
                                                              rank_map, ordered);
    else
        k_compact<false, false><<<grid, kCopyThreads, 0, st>>>(n_tasks, tm, counts, dest, spill_off, scratch_e,
                                                               scratch_w, spill_e, spill_w, out_e, out_w, out_cap,
                                                               rank_map, ordered);
    return cudaGetLastError();
}

cudaError_t launch_offsets(int64_t n_samples, const TaskMap &tm, const int64_t *dest, int64_t *offsets, cudaStream_t st)
{
    count_launch();
    k_offsets<<<(unsigned)((n_samples + 1 + 255) / 256), 256, 0, st>>>(n_samples, tm, dest, offsets);
    return cudaGetLastError();
}

cudaError_t launch_add_u64(const uint64_t *in, uint64_t *out, int64_t n, cudaStream_t st)
{
    if (n <= 0) return cudaSuccess;
    count_launch();
    k_add_u64<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(in, out, n);
    return cudaGetLastError();
}

cudaError_t launch_debug_eval(int fn, int64_t n, const double *in, double *out, cudaStream_t st)
{
    cudaError_t e = ensure_log_table(st);
    if (e != cudaSuccess) return e;
    if (n <= 0) return cudaSuccess;
    count_launch();
    k_debug_eval<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(fn, n, in, out, log_consts());
    return cudaGetLastError();
}

}  // namespace fm
