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
#include <type_traits>

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

// block shape of the sampler: 24 warps per SM at <= 80 registers as 2 blocks of 384 threads (r02 A/B
// against 3 x 256: config 5 -0.4 %, config 2 -1.6 %, ECM +-0: one log / range table and barrier
// less per SM; 28 and 30 warps per SM -- 128 x 7, 224 x 4, 192 x 5 -- measured +0.3 ... +33 %)
#ifndef FM_SAMPLE_THREADS
#define FM_SAMPLE_THREADS 384
#endif
#ifndef FM_SAMPLE_MINB_UBCM
#define FM_SAMPLE_MINB_UBCM 2
#endif
#ifndef FM_SAMPLE_MINB_ECM
#define FM_SAMPLE_MINB_ECM 2
#endif
#ifndef FM_SAMPLE_THREADS_RANKOUT  // the rank-out path keeps 4 x 256 threads at <= 64 registers
#define FM_SAMPLE_THREADS_RANKOUT 256
#endif
#ifndef FM_SAMPLE_MINB_RANKOUT  // UBCM rank-out path (N >= 2^21: DRAM-latency-bound gathers)
#define FM_SAMPLE_MINB_RANKOUT 4
#endif
constexpr int kThreads = FM_SAMPLE_THREADS;  // threads per block of the sampler
constexpr int kThreadsRankOut = FM_SAMPLE_THREADS_RANKOUT;
constexpr int kFuseThreadsC = 768;  // fused launch: one block per SM, 23 sampler warps + 1 copier (24 warps at 80 registers fill the register file)
// block size of an instantiation: the fused write runs one block per SM, the rank-out path its own shape
__host__ __device__ constexpr int sampler_threads(bool fuse, int gather) { return fuse ? kFuseThreadsC : gather == 2 ? kThreadsRankOut : kThreads; }
constexpr int kBatch = kQueueBatch;  // tasks per warp batch

// one sample range of the task map (TaskMap) for the sampler's shared-memory table
struct RangeRec {
    const int64_t *seg, *cap;
    int64_t n_chunks;
    double inv_chunks;
    int64_t s0, t0, il_s;
    double inv_il;  // 1 / il_s
};

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

// ------------------------------------------------------------------------------------------
// v3 fused write (a6 without the compaction pass), warp-specialised.  In a fused launch every
// block has kThreads/32 - 1 SAMPLER warps and one COPIER warp.  Sampler warps claim the task
// queue in batches of kBatch consecutive canonical tasks (every task of a batch runs on a lane of
// the claiming warp) and register each batch in their block's ring (shared memory).  A lane that
// finishes a task adds (1 task, its edge count) to its batch's packed counter; the lane that
// finishes a batch's last task publishes the batch's edge count in the batch's global status word
// (decoupled look-back: 2 flag bits + 62-bit value; batch 0 publishes its inclusive prefix).  The
// copier warp takes the finished batches of its block, forms each one's output offset by
// look-back over the preceding batches (resumable: an unfinished predecessor is revisited
// later), publishes the inclusive prefix, copies the batch's edges from the scratch slots --
// written by its own block moments earlier, in the L2 -- into the final list with streaming
// stores, discards the batch's scratch lines from the L2 (discard.global.L2: no write-back), and
// frees the ring entry.  A sampler warp with no free ring entry leaves its idle lanes idle.
// Deadlock-free: finished-batch counts are published by sampler lanes, so a look-back waits only
// on unfinished batches, and those run on sampler warps that never wait.
constexpr uint64_t kGrpAgg = 1ull << 62, kGrpInc = 2ull << 62, kGrpVal = (1ull << 62) - 1;
constexpr int kBRing = 128;             // ring entries per block (one bit each in 64-bit masks)
constexpr int kPackShift = 40;          // packed batch counter: finished tasks << 40 | edges
#ifndef FM_COPY_JOBS
#define FM_COPY_JOBS 8
#endif
#ifndef FM_COPY_JOBS_RANKOUT
#define FM_COPY_JOBS_RANKOUT 4
#endif

// The status words carry only their own value (no data is published through them: a copier
// copies its own block's batches, ordered by CTA-scope fences), so relaxed gpu-scope accesses
// suffice -- an acquire load would invalidate the SM's whole L1 (CCTL.IVALL) at every poll.
__device__ __forceinline__ uint64_t ld_status(const unsigned long long *p)
{
    uint64_t v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_status(unsigned long long *p, uint64_t v)
{
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void discard_l2_line(const void *p)
{
    asm volatile("discard.global.L2 [%0], 128;" ::"l"(p) : "memory");
}

// fused-write instrumentation (FM_FUSE_STATS builds): copies, copy cycles, polls without progress,
// entries finished but blocked per poll, ring-full claim failures, sampler idle iterations
#ifdef FM_FUSE_STATS
__device__ unsigned long long g_fstats[8];
#define FSTAT(i, v) atomicAdd(&g_fstats[i], (unsigned long long)(v))
#else
#define FSTAT(i, v) ((void)0)
#endif

// a task of the sub-batch being copied (per-copier table in shared memory)
struct __align__(16) CopyDesc {
    long long src, dst;  // slot start (scratch element index), final position
    long long sp;        // spill region (-1 none)
    int cnt, cap, jexcl, pad;
};

// the block's ring of claimed batches and the copier's staging buffer (shared memory); the
// non-fused kernels get a minimal instance (no static shared memory for a copier they do not have)
template <int NR, int NS>
struct RingT {
    unsigned long long packed[NR];  // finished tasks << kPackShift | their edges
    long long b[NR];                // batch id, -1 free
    long long lb_j[NR];             // resumable look-back: next predecessor to read (-2: none yet)
    unsigned long long lb_pre[NR];  //   and the sum collected so far
    unsigned long long free_mask[NR > 64 ? NR / 64 : 1];  // free entries
    unsigned exited;                // sampler warps that have left the loop
    unsigned long long mbar[2];     // the copier's bulk-load barriers (one per staging buffer)
    CopyDesc desc[NR < 32 ? 1 : 32];  // the copier's sub-batch table (register-copy path)
};
using BlockRing = RingT<kBRing, 0>;

// Copy the finished batch b (tasks [b kb, ...)) to the final list at `prefix`; write each task's
// final offset.  Warp-synchronous.
template <int kGather>
__device__ __forceinline__ void batch_copy(const SampleArgs &A, int64_t b, int64_t prefix, int64_t agg, int kb,
                                           CopyDesc *desc)
{
    const int lane = threadIdx.x & 31;
    constexpr int kCopyJobs = kGather == 2 ? FM_COPY_JOBS_RANKOUT : FM_COPY_JOBS;
    const int64_t T = A.n_tasks;
    const int64_t t0 = b * kb, t1 = min(T, t0 + kb);
    if (t1 == T && lane == 0) A.dest[T] = prefix + agg;
    int64_t run = prefix;
#ifdef FM_FUSE_STATS
    long long ph0 = clock64(), ph_desc = 0, ph_jobs = 0;
#endif
    for (int64_t tb = t0; tb < t1; tb += 32) {
        const int64_t t = tb + lane;
        int64_t cnt = 0, src = 0, sp = -1, cap = 0;
        if (t < t1) {
            int64_t s_, c_;
            int k_;
            task_decode(A.tm, t, s_, c_, k_);
            cap = FM_TM_SEL(A.tm, cap, k_)[c_ + 1] - FM_TM_SEL(A.tm, cap, k_)[c_];
            src = s_ * A.tm.cap_per_sample + FM_TM_SEL(A.tm, cap, k_)[c_];
            cnt = A.counts[t];
            sp = A.spill_off[t];
        }
        int64_t incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int64_t v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        const int64_t dst = run + incl - cnt;
        if (t < t1) A.dest[t] = dst;
        run += __shfl_sync(0xffffffffu, incl, 31);
        // not copied: tasks whose data is incomplete (slot and spill overflowed: re-run after the
        // kernel) and tasks beyond the list's capacity (the host then redoes the call)
        const bool skip = (cnt > cap && (cnt > 2 * cap || sp < 0)) || dst + cnt > A.out_cap;
        const int64_t ncp = skip ? 0 : cnt;
        // jobs: 64 consecutive elements of one task, two per lane (16-byte loads: slots and spill
        // regions start at multiples of 4 elements)
        const int32_t nj = (int32_t)((ncp + 63) >> 6);
        int32_t jincl = nj;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int32_t v = __shfl_up_sync(0xffffffffu, jincl, o);
            if (lane >= o) jincl += v;
        }
        const int32_t jexcl = jincl - nj;
        const int32_t njobs = __shfl_sync(0xffffffffu, jincl, 31);
        __syncwarp();
        desc[lane].src = src;
        desc[lane].dst = dst;
        desc[lane].sp = sp;
        desc[lane].cnt = (int32_t)ncp;
        desc[lane].cap = (int32_t)cap;
        desc[lane].jexcl = jexcl;
        __syncwarp();
#ifdef FM_FUSE_STATS
        const long long ph1 = clock64();
        ph_desc += ph1 - ph0;
#endif
        for (int32_t j0 = 0; j0 < njobs; j0 += kCopyJobs) {
#ifdef FM_FUSE_STATS
            if (lane == 0) FSTAT(5, 1);
#endif
            int4 v[kCopyJobs];
            int64_t od[kCopyJobs];
            int nv[kCopyJobs];
#pragma unroll
            for (int q = 0; q < kCopyJobs; q++) {
                nv[q] = 0;
                od[q] = 0;
                const int32_t j = j0 + q;
                if (j >= njobs) continue;  // warp-uniform
                // the task holding job j: job prefixes increase strictly over the tasks with jobs,
                // so it is the last such lane whose first job is <= j; its descriptor from the table
                const int kk = 31 - __clz(__ballot_sync(0xffffffffu, jexcl <= j && nj > 0));
                const CopyDesc &D = desc[kk];
                const int64_t e = (int64_t)(j - D.jexcl) * 64 + 2 * lane;
                const int64_t c_k = D.cnt, cap_k = D.cap, src_k = D.src, sp_k = D.sp, dst_k = D.dst;
                if (e < c_k) {
                    const int2 *q2 = e < cap_k ? A.edges + src_k + e : A.spill_e + sp_k + (e - cap_k);
                    v[q] = *reinterpret_cast<const int4 *>(q2);
                    nv[q] = e + 1 < c_k ? 2 : 1;
                    od[q] = dst_k + e;
                }
            }
            // every load of the round is issued before the first store (a compiler barrier: the
            // loads would otherwise be sunk next to their stores, one latency each)
            asm volatile("" ::: "memory");
#ifdef FM_FUSE_STATS
            const long long pl = clock64();
#endif
#pragma unroll
            for (int q = 0; q < kCopyJobs; q++) {
                if (nv[q] == 0) continue;
                int2 e0 = make_int2(v[q].x, v[q].y), e1 = make_int2(v[q].z, v[q].w);
                if (kGather == 2) {  // UBCM large N: (row id, candidate rank) -> (min id, max id)
                    const int32_t i0 = __ldg(A.rank_map + e0.y);
                    e0 = make_int2(min(e0.x, i0), max(e0.x, i0));
                    if (nv[q] == 2) {
                        const int32_t i1 = __ldg(A.rank_map + e1.y);
                        e1 = make_int2(min(e1.x, i1), max(e1.x, i1));
                    }
                }
                if (nv[q] == 2 && (od[q] & 1) == 0) {
                    __stcs(reinterpret_cast<int4 *>(A.out_e + od[q]), make_int4(e0.x, e0.y, e1.x, e1.y));
                } else {
                    __stcs(A.out_e + od[q], e0);
                    if (nv[q] == 2) __stcs(A.out_e + od[q] + 1, e1);
                }
            }
#ifdef FM_FUSE_STATS
            if (lane == 0) FSTAT(4, clock64() - pl);
#endif
        }
#ifdef FM_FUSE_STATS
        {
            const long long ph2 = clock64();
            ph_jobs += ph2 - ph1;
            ph0 = ph2;
        }
#endif
    }
#ifdef FM_FUSE_STATS
    if (lane == 0) {
        FSTAT(6, ph_desc);
        FSTAT(7, ph_jobs);
    }
#endif
    // hand the batch's scratch lines back without a write-back: only whole 128-byte lines inside
    // its slots (which no other task shares), after every lane's loads of them have completed
    // (their values were stored above)
    __syncwarp();
    if (A.discard) {
        const char *base = reinterpret_cast<const char *>(A.edges);
        int64_t s_first, c_first, s_last, c_last;
        int k_first, k_last;
        task_decode(A.tm, t0, s_first, c_first, k_first);
        task_decode(A.tm, t1 - 1, s_last, c_last, k_last);
        for (int64_t s_ = s_first; s_ <= s_last; s_++) {
            // the batch's tasks of sample s_ are consecutive chunks of one chunking: their slots
            // form one contiguous range
            const int kc = s_ == s_first ? k_first : s_ == s_last ? k_last : sample_range(A.tm, s_);
            const int64_t lo_c = s_ == s_first ? c_first : 0;
            const int64_t hi_c = s_ == s_last ? c_last + 1 : FM_TM_SEL(A.tm, n_chunks, kc);
            const size_t a = (size_t)(s_ * A.tm.cap_per_sample + FM_TM_SEL(A.tm, cap, kc)[lo_c]) * sizeof(int2);
            const size_t z = (size_t)(s_ * A.tm.cap_per_sample + FM_TM_SEL(A.tm, cap, kc)[hi_c]) * sizeof(int2);
            const size_t la = (a + 127) & ~(size_t)127, lz = z & ~(size_t)127;
            for (size_t l = la + (size_t)lane * 128; l < lz; l += 32 * 128) discard_l2_line(base + l);
        }
    }
}

// ---- bulk asynchronous copies (TMA engine) for the copier: the data never passes through
// registers, so the copier issues ~1 instruction per task instead of ~1 per 16 bytes (measured:
// a register-copying warp next to 21 issue-bound sampler warps moved ~1 GB/s) ----
__device__ __forceinline__ void mbar_init(uint32_t mbar, unsigned count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(mbar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect(uint32_t mbar, unsigned bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t mbar, unsigned parity)
{
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(mbar),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst_smem, const void *src, unsigned bytes, uint32_t mbar)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst_smem),
                 "l"(src), "r"(bytes), "r"(mbar)
                 : "memory");
}
__device__ __forceinline__ void bulk_s2g(void *dst, uint32_t src_smem, unsigned bytes)
{
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(src_smem), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }

// ---- the pipelined copy: sub-batches of 32 tasks (one per lane) alternate between two staging
// buffers, so the bulk loads of one sub-batch overlap the stores of the previous one ----
constexpr int kStageBuf = 40960;  // bytes per staging buffer (two buffers)
struct SubDesc {
    long long dst, src;  // final position, slot start (elements)
    long long sp;        // spill region of a spilled task (copied by the warp), else -1
    int ncp, cap;        // elements to copy, slot capacity
    unsigned off;        // staging offset (bytes, 16-byte aligned)
};

// Descriptors of the sub-batch [tb, min(tb + 32, t1)) whose output starts at `run` (advanced past
// it); writes the tasks' final offsets.  Returns the sub-batch's staged bytes (> kStageBuf: it
// does not fit one buffer).
__device__ __forceinline__ unsigned sub_prep(const SampleArgs &A, int64_t tb, int64_t t1, int64_t &run, SubDesc &d)
{
    const int lane = threadIdx.x & 31;
    const int64_t t = tb + lane;
    int64_t cnt = 0, src = 0, sp = -1, cap = 0;
    if (t < t1) {
        int64_t s_, c_;
        int k_;
        task_decode(A.tm, t, s_, c_, k_);
        cap = FM_TM_SEL(A.tm, cap, k_)[c_ + 1] - FM_TM_SEL(A.tm, cap, k_)[c_];
        src = s_ * A.tm.cap_per_sample + FM_TM_SEL(A.tm, cap, k_)[c_];
        cnt = A.counts[t];
        sp = A.spill_off[t];
    }
    int64_t incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int64_t v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
    }
    const int64_t dst = run + incl - cnt;
    if (t < t1) A.dest[t] = dst;
    run += __shfl_sync(0xffffffffu, incl, 31);
    // not copied: incomplete tasks (slot and spill overflowed: re-run after the kernel) and tasks
    // beyond the list's capacity (the host then redoes the call); spilled tasks (rare) are copied
    // by the warp itself (sub_finish)
    const bool skip = (cnt > cap && (cnt > 2 * cap || sp < 0)) || dst + cnt > A.out_cap;
    const int64_t ncp = skip ? 0 : cnt;
    const unsigned need = ncp > cap ? 0u : (unsigned)(((ncp + 1) & ~int64_t(1)) * 8);
    unsigned inc = need;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned v = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += v;
    }
    d.dst = dst;
    d.src = src;
    d.sp = ncp > cap ? sp : -1;
    d.ncp = (int)ncp;
    d.cap = (int)cap;
    d.off = inc - need;
    return __shfl_sync(0xffffffffu, inc, 31);
}

// spilled tasks of a sub-batch (slot + spill region, rare): plain warp copy
__device__ __forceinline__ void sub_copy_spilled(const SampleArgs &A, const SubDesc &d, bool all)
{
    const int lane = threadIdx.x & 31;
    unsigned spl = __ballot_sync(0xffffffffu, d.ncp > 0 && (all || d.sp >= 0));
    while (spl) {
        const int k = __ffs(spl) - 1;
        spl &= spl - 1;
        const long long d_k = __shfl_sync(0xffffffffu, d.dst, k);
        const int c_k = __shfl_sync(0xffffffffu, d.ncp, k), cap_k = __shfl_sync(0xffffffffu, d.cap, k);
        const long long sp_k = __shfl_sync(0xffffffffu, d.sp, k), src_k = __shfl_sync(0xffffffffu, d.src, k);
        for (int e = lane; e < c_k; e += 32)
            __stcs(A.out_e + d_k + e, e < cap_k ? A.edges[src_k + e] : A.spill_e[sp_k + e - cap_k]);
    }
}
__device__ __forceinline__ void sub_finish_nowait(const SampleArgs &A, const SubDesc &d) { sub_copy_spilled(A, d, false); }
__device__ __forceinline__ void sub_copy_plain(const SampleArgs &A, const SubDesc &d) { sub_copy_spilled(A, d, true); }

// Bulk-load the sub-batch's slots into the staging buffer (one instruction per task).
__device__ __forceinline__ void sub_issue(const SampleArgs &A, const SubDesc &d, uint32_t buf, uint32_t mbar,
                                          unsigned total)
{
    const int lane = threadIdx.x & 31;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (lane == 0) mbar_arrive_expect(mbar, total);
    __syncwarp();
    if (d.ncp > 0 && d.sp < 0)
        bulk_g2s(buf + d.off, reinterpret_cast<const char *>(A.edges) + (size_t)d.src * 8,
                 (unsigned)((d.ncp + 1) & ~1) * 8, mbar);
}

// Wait for the sub-batch's loads, discard its scratch lines, store it: aligned final positions by
// one bulk store per task, odd ones by the warp (pairs re-aligned through shared memory).
__device__ __forceinline__ void sub_finish(const SampleArgs &A, const SubDesc &d, uint32_t buf, uint32_t mbar,
                                           unsigned &phase)
{
    const int lane = threadIdx.x & 31;
    mbar_wait(mbar, phase & 1);
    phase++;
    const bool staged = d.ncp > 0 && d.sp < 0;
    if (staged && A.discard) {
        const char *base = reinterpret_cast<const char *>(A.edges);
        const size_t a = (size_t)d.src * 8, z = a + (size_t)d.cap * 8;
        for (size_t l = (a + 127) & ~(size_t)127; l + 128 <= z; l += 128) discard_l2_line(base + l);
    }
    const bool even = (d.dst & 1) == 0;
    if (staged && even) {
        const unsigned nb = (unsigned)(d.ncp & ~1) * 8;
        if (nb) bulk_s2g(A.out_e + d.dst, buf + d.off, nb);
        if (d.ncp & 1) {
            int2 e;
            asm volatile("ld.shared.v2.b32 {%0,%1}, [%2];" : "=r"(e.x), "=r"(e.y) : "r"(buf + d.off + (unsigned)(d.ncp - 1) * 8));
            __stcs(A.out_e + d.dst + d.ncp - 1, e);
        }
    }
    bulk_commit();
    unsigned odd = __ballot_sync(0xffffffffu, staged && !even);
    while (odd) {
        const int k = __ffs(odd) - 1;
        odd &= odd - 1;
        const long long d_k = __shfl_sync(0xffffffffu, d.dst, k);
        const int c_k = __shfl_sync(0xffffffffu, d.ncp, k);
        const unsigned o_k = __shfl_sync(0xffffffffu, d.off, k);
        for (int e0 = 2 * lane; e0 < c_k + 1; e0 += 64) {
            if (e0 == 0) {  // element 0 alone; pairs (e0 - 1, e0) after it are 16-byte aligned
                int2 e;
                asm volatile("ld.shared.v2.b32 {%0,%1}, [%2];" : "=r"(e.x), "=r"(e.y) : "r"(buf + o_k));
                __stcs(A.out_e + d_k, e);
                continue;
            }
            int2 x0, x1;
            asm volatile("ld.shared.v2.b32 {%0,%1}, [%2];" : "=r"(x0.x), "=r"(x0.y) : "r"(buf + o_k + (unsigned)(e0 - 1) * 8));
            if (e0 < c_k) {
                asm volatile("ld.shared.v2.b32 {%0,%1}, [%2];" : "=r"(x1.x), "=r"(x1.y) : "r"(buf + o_k + (unsigned)e0 * 8));
                __stcs(reinterpret_cast<int4 *>(A.out_e + d_k + e0 - 1), make_int4(x0.x, x0.y, x1.x, x1.y));
            } else {
                __stcs(A.out_e + d_k + e0 - 1, x0);
            }
        }
    }
    sub_copy_spilled(A, d, false);  // spilled tasks (slot + spill region): plain warp copy
}

// The copier warp of a fused block: resolve and copy the block's finished batches until every
// sampler warp of the block has left and the ring is empty.  A poll costs one status load per
// finished entry, all in parallel (lane l owns entries l and l + 32): the word of the predecessor
// its look-back is suspended on.  Only entries whose word has become non-zero walk further.
template <int kGather>
__device__ __forceinline__ void copier_loop(const SampleArgs &A, BlockRing &Rg, int n_samplers, int kb, uint32_t stage)
{
    const int lane = threadIdx.x & 31;
    // pipeline state: the sub-batch whose loads are in flight (finished after the next one is issued)
    unsigned ph[2] = {0, 0};
    const uint32_t mb[2] = {(uint32_t)__cvta_generic_to_shared(&Rg.mbar[0]),
                            (uint32_t)__cvta_generic_to_shared(&Rg.mbar[1])};
    SubDesc pd;
    pd.ncp = 0;
    bool pending = false;
    unsigned ptot = 0;
    int pbuf = 0, nbuf = 0;
    auto flush = [&]() {
        if (!pending) return;
        if (ptot) {
            sub_finish(A, pd, stage + (uint32_t)pbuf * kStageBuf, mb[pbuf], ph[pbuf]);
        } else {  // nothing staged (spilled tasks only)
            SubDesc z = pd;
            sub_finish_nowait(A, z);
        }
        pending = false;
    };
    auto copy_batch = [&](int64_t b, int64_t prefix, int64_t agg) {
        const int64_t T = A.n_tasks;
        const int64_t t0 = b * kb, t1 = min(T, t0 + kb);
        if (t1 == T && lane == 0) A.dest[T] = prefix + agg;
        int64_t run = prefix;
        for (int64_t tb = t0; tb < t1; tb += 32) {
            SubDesc d;
            const unsigned tot = sub_prep(A, tb, t1, run, d);
            if (tot <= (unsigned)kStageBuf) {
                const int x = nbuf;
                // buffer x's previous stores must have read it: at most the other buffer's group pending
                asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                __syncwarp();
                if (tot) sub_issue(A, d, stage + (uint32_t)x * kStageBuf, mb[x], tot);
                flush();
                pd = d;
                ptot = tot;
                pbuf = x;
                pending = true;
                nbuf ^= 1;
            } else {  // (rare) a sub-batch larger than a buffer: plain warp copy
                flush();
                sub_copy_plain(A, d);
            }
        }
    };
    for (;;) {
        bool did = false;
        bool any_entry = false;
        for (int half = 0; half < kBRing / 32; half++) {  // (lane l: entries l, l + 32, ...)
            const int el = half * 32 + lane;
            const long long be = *(volatile long long *)&Rg.b[el];
            const unsigned long long pk = *(volatile unsigned long long *)&Rg.packed[el];
            any_entry = any_entry || be >= 0;
            const int n_in = be >= 0 ? (int)min((int64_t)kb, A.n_tasks - (int64_t)be * kb) : 0;
            const bool fin = be >= 0 && (int)(pk >> kPackShift) == n_in;
            // per finished entry: one load of the predecessor it waits on (batch 0 waits on none)
            bool go = false;
            if (fin) {
                if (be == 0) {
                    go = true;
                } else {
                    const long long jw = Rg.lb_j[el] < -1 ? be - 1 : Rg.lb_j[el];
                    go = (ld_status(A.grp_state + jw) & ~kGrpVal) != 0;
                }
            }
            unsigned ready = __ballot_sync(0xffffffffu, go);
#ifdef FM_FUSE_STATS
            const unsigned blocked = __ballot_sync(0xffffffffu, fin && !go);
            if (lane == 0) FSTAT(3, __popc(blocked));
#else
            (void)fin;
#endif
            while (ready) {
                const int el0 = __ffs(ready) - 1;
                const int e = half * 32 + el0;
                ready &= ready - 1;
                const int64_t b = __shfl_sync(0xffffffffu, be, el0);
                const int64_t agg = (int64_t)(__shfl_sync(0xffffffffu, pk, el0) & ((1ull << kPackShift) - 1));
                // look-back, 32 predecessors per step (one status word per lane): the nearest INC in
                // the window ends it; an unfinished batch above it suspends it (resumed from there)
                int64_t prefix = -1;
                if (b == 0) {
                    prefix = 0;
                } else {
                    int64_t j = Rg.lb_j[e] < -1 ? b - 1 : Rg.lb_j[e];  // highest predecessor not summed
                    uint64_t pre = Rg.lb_j[e] < -1 ? 0 : Rg.lb_pre[e];
                    for (;;) {
                        const int64_t jj = j - lane;
                        const uint64_t v = jj >= 0 ? ld_status(A.grp_state + jj) : kGrpInc;
                        const uint64_t f = v & ~kGrpVal;
                        const unsigned inc = __ballot_sync(0xffffffffu, f == kGrpInc);
                        const unsigned zero = __ballot_sync(0xffffffffu, f == 0);
                        const int li = inc ? __ffs(inc) - 1 : 32;    // nearest INC
                        const int lz = zero ? __ffs(zero) - 1 : 32;  // nearest unfinished
                        const int upto = min(li, lz);
                        uint64_t part = (lane < upto || (lane == li && li < lz)) ? (v & kGrpVal) : 0;
#pragma unroll
                        for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
                        pre += part;
                        if (li < lz) {
                            prefix = (int64_t)pre;
                            break;
                        }
                        j -= upto;
                        if (lz < 32) {  // suspended on predecessor j
                            if (lane == 0) {
                                Rg.lb_j[e] = j;
                                Rg.lb_pre[e] = pre;
                            }
                            break;
                        }
                    }
                    if (prefix >= 0 && lane == 0) st_status(A.grp_state + b, kGrpInc | (uint64_t)(prefix + agg));
                }
                if (prefix < 0) continue;
                __threadfence_block();  // (acquire: the batch's slot data after its finished count)
#ifdef FM_FUSE_STATS
                const long long c0 = clock64();
#endif
#ifdef FM_FUSE_NOCOPY  // timing experiment only: the copier resolves but does not copy
                if (false)
#endif
                if (kGather == 2)  // rank-out: the ids are mapped on the way (through registers)
                    batch_copy<kGather>(A, b, prefix, agg, kb, Rg.desc);
                else
                    copy_batch(b, prefix, agg);
#ifdef FM_FUSE_STATS
                if (lane == 0) {
                    FSTAT(0, 1);
                    FSTAT(1, clock64() - c0);
                }
#endif
                if (lane == 0) {  // free the entry: counter reset before the id, both before the free bit
                    Rg.lb_j[e] = -2;
                    *(volatile unsigned long long *)&Rg.packed[e] = 0;
                    __threadfence_block();
                    *(volatile long long *)&Rg.b[e] = -1;
                    __threadfence_block();
                    atomicOr(&Rg.free_mask[e >> 6], 1ull << (e & 63));
                }
                did = true;
            }
            __syncwarp();
        }
        if (!did) {
            flush();  // (idle: complete the sub-batch in flight)
            const unsigned ex = *(volatile unsigned *)&Rg.exited;
            if (ex == (unsigned)n_samplers && !__any_sync(0xffffffffu, any_entry)) {
                asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // (writes complete)
                break;
            }
            if (lane == 0) FSTAT(2, 1);
            __nanosleep(500);
        }
    }
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
// kFuse: v3 fused write (UBCM edge lists; the launch's a.fuse): the block's last warp is a copier.
template <int kModel, int kMinBlocks, int kC, bool kStats, bool kRefresh, int kGather, bool kOrdered, bool kCheck,
          bool kFuse>
__global__ void __launch_bounds__(sampler_threads(kFuse, kGather), kFuse ? 1 : kMinBlocks) k_sample(const __grid_constant__ SampleArgs A)
{
    // block size: several blocks per SM, or one fused block per SM
    constexpr int kT = sampler_threads(kFuse, kGather);
    extern __shared__ __align__(16) unsigned char s_dyn[];  // per-chain prefetch slots
    // rarely used per-chain task state lives in shared memory (registers are the occupancy limit)
    __shared__ int64_t s_task[kT * kC];   // current task id, -1 none
    __shared__ int64_t s_spill[kT * kC];  // its spill region: -1 none, -2 failed
    // 64-bit per-thread draw / accepted counters: the 32-bit registers below are added here at
    // every task end (a statistics call over many samples passes 2^32 per warp)
    __shared__ unsigned long long s_ndraw[kT / 32], s_nacc[kT / 32];  // per warp
    // UBCM: the last < 4 accepted edges of each lane's slot, so that the slot is written in whole
    // 32-byte sectors (structure of arrays: conflict-free)
    __shared__ int2 s_eb[kModel == FM_UBCM ? 4 : 1][kT];
    const bool buf4 = kModel == FM_UBCM && A.buf4 && !A.rerun_base && !kStats;
    // ECM: the scratch holds one 16-byte (src, dst, w, 0) record per edge, written two per sector
    // (the lane's previous record waits in shared memory); the compaction splits the records into
    // the edge and weight arrays (separate 8- and 4-byte stores wrote two partial sectors per edge)
    __shared__ int4 s_er[kModel == FM_ECM ? kT : 1];
    const bool aos = kModel == FM_ECM && A.buf4 && !A.rerun_base && !kStats;
    // v3 fused write (UBCM edge lists): the block's last warp copies the finished batches of its
    // sampler warps to the final list
    static_assert(!kFuse || (kModel == FM_UBCM && !kStats), "fused write: UBCM edge lists only");
    constexpr bool fuse = kFuse;
    using Ring = std::conditional_t<kFuse, BlockRing, RingT<1, 16>>;
    __shared__ Ring s_ring[1];
    __shared__ unsigned char s_tslot[kFuse ? kT : 1];
    Ring &R = s_ring[0];
    if constexpr (kFuse) {
        if (threadIdx.x < kBRing) {
            R.b[threadIdx.x] = -1;
            R.packed[threadIdx.x] = 0;
            R.lb_j[threadIdx.x] = -2;
            if (threadIdx.x < kBRing / 64) R.free_mask[threadIdx.x] = ~0ull;
            if (threadIdx.x == 0) {
                R.exited = 0;
                mbar_init((uint32_t)__cvta_generic_to_shared(&R.mbar[0]), 1);
                mbar_init((uint32_t)__cvta_generic_to_shared(&R.mbar[1]), 1);
                asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            }
        }
    }
    // the task map's three sample ranges as a table indexed by the range
    __shared__ RangeRec s_rng[kRanges];
    if (threadIdx.x == 0) {
#pragma unroll
        for (int r = 0; r < kRanges; r++) {
            s_rng[r].seg = A.tm.seg[r];
            s_rng[r].cap = A.tm.cap[r];
            s_rng[r].n_chunks = A.tm.n_chunks[r];
            s_rng[r].inv_chunks = A.tm.inv_chunks[r];
            s_rng[r].s0 = A.tm.s0[r];
            s_rng[r].t0 = A.tm.t0[r];
            s_rng[r].il_s = A.il_s[r];
            s_rng[r].inv_il = A.il_s[r] > 0 ? 1.0 / (double)A.il_s[r] : 0.0;
        }
    }
    const SmemLogTab T{A.lc, load_logtab()};  // (block barrier inside)
    if constexpr (kFuse) {
        if ((threadIdx.x >> 5) == 0) {  // the block's copier warp
            // the staging buffer: dynamic shared memory after the sampler warps' prefetch slots
            copier_loop<kGather>(A, R, kT / 32 - 1, kBatch,
                                 ((uint32_t)__cvta_generic_to_shared(s_dyn) + (uint32_t)(kT * kC * 64) + 127u) & ~127u);
            return;
        }
    }
    const int lane = threadIdx.x & 31;
    const uint32_t lt = (1u << lane) - 1u;
    const int64_t n_tasks = A.n_tasks_dev ? (int64_t)*A.n_tasks_dev : A.n_tasks;

    // ---- warp batch of task ids [bpos, bend); lane 0 holds the start of the next batch ----
    unsigned long long next_batch = 0;  // (prefetched claim; the fused write claims at open time)
    if (!kFuse && lane == 0) next_batch = atomicAdd(A.task_counter, (unsigned long long)kBatch);
    int64_t bpos = 0, bend = 0;
    int cur_slot = 0;  // fused write: ring entry of the batch [bpos, bend)
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
    if ((threadIdx.x & 31) == 0) {
        s_ndraw[threadIdx.x >> 5] = 0;
        s_nacc[threadIdx.x >> 5] = 0;
    }
    bool wsat = false, bad_bound = false;

    // segment g[c] of chain c's task becomes current (64/96-byte record; the record of the next
    // segment is prefetched into this chain's shared-memory slot with cp.async)
    // this thread's prefetch slots: 32-bit shared addresses (no generic-address arithmetic)
    // structure of arrays: 16-byte part k of thread t's slot at (k * kThreads + t) * 16, so the
    // 8 lanes of a 16-byte shared access touch 8 consecutive 16-byte words (conflict-free)
    static_assert(kC == 1, "prefetch slot layout assumes one chain per thread");
    constexpr int kPart = 16 * kT;
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
                // (.cg: the records stream past the L1, which stays with the kappa gathers -- config 4 -0.9 %,
                // config 5 -0.3 % against .ca)
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(my_next + kPart * k), "l"(src + 16 * k)
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
                        if (kFuse && fuse) {  // v3: the task is finished: count it in its batch
                            const int sl = s_tslot[threadIdx.x];
                            // the slot's edges (its last partial sector above), spill and count are
                            // written: order them before the count the copier warp reads (CTA scope)
                            __threadfence_block();
                            const unsigned long long old =
                                atomicAdd(&R.packed[sl], (1ull << kPackShift) | (unsigned long long)cnt[c]);
                            const int64_t bb = R.b[sl];
                            if ((int64_t)(old >> kPackShift) + 1 == min((int64_t)kBatch, n_tasks - bb * kBatch)) {
                                // the batch's last task: publish its edge count (batch 0: its prefix)
                                const uint64_t agg = (old & ((1ull << kPackShift) - 1)) + (uint64_t)cnt[c];
                                st_status(A.grp_state + bb, (bb == 0 ? kGrpInc : kGrpAgg) | agg);
                            }
                        }
                    }
                    s_task[ci] = -1;
#ifndef FM_THREAD_COUNTERS
                    atomicAdd(&s_ndraw[threadIdx.x >> 5], (unsigned long long)n_draw);
                    if (kStats) atomicAdd(&s_nacc[threadIdx.x >> 5], (unsigned long long)n_acc);
                    n_draw = n_acc = 0;
#endif
                }
            }
            const uint32_t nc = __ballot_sync(0xffffffffu, needc && !warp_done);
            if (nc) {
                const int k = __popc(nc), rank = __popc(nc & lt);
                const int64_t avail = bend - bpos;
                int64_t my;
                int myslot = 0;
                if (k <= avail) {
                    my = bpos + rank;
                    bpos += k;
                    myslot = cur_slot;
                } else {
                    int64_t nb;
                    int ns = 0;
                    if constexpr (kFuse) {
                        // fused write: reserve a free entry of the block's ring first, then claim the
                        // batch (no prefetched claims: every claimed batch is running, so a look-back
                        // never waits on a batch that cannot start); no entry: the idle lanes wait
                        int got = -1;
                        long long nbl = 0;
                        if (lane == 0) {
                            // (start the search at this warp's own word: less contention)
                            const int w0 = ((threadIdx.x >> 5) * (kBRing / 64)) / (kT / 32);
                            for (int wq = 0; wq < kBRing / 64 && got < 0; wq++) {
                                const int w = (w0 + wq) % (kBRing / 64);
                                unsigned long long m = *(volatile unsigned long long *)&R.free_mask[w];
                                while (m) {
                                    const int e = __ffsll((long long)m) - 1;
                                    const unsigned long long old = atomicAnd(&R.free_mask[w], ~(1ull << e));
                                    if (old & (1ull << e)) {  // (its counter is already 0)
                                        got = w * 64 + e;
                                        break;
                                    }
                                    m = old & ~(1ull << e);
                                }
                            }
                            if (got >= 0) {
                                nbl = (long long)atomicAdd(A.task_counter, (unsigned long long)kBatch);
                                if (nbl < n_tasks) *(volatile long long *)&R.b[got] = nbl / kBatch;
                                else atomicOr(&R.free_mask[got >> 6], 1ull << (got & 63));  // the queue is empty
                            }
                        }
                        ns = __shfl_sync(0xffffffffu, got, 0);
                        nb = __shfl_sync(0xffffffffu, nbl, 0);
                    } else {
                        nb = (int64_t)__shfl_sync(0xffffffffu, next_batch, 0);
                    }
                    if (ns >= 0) {
                        my = rank < avail ? bpos + rank : nb + (rank - avail);
                        myslot = rank < avail ? cur_slot : ns;
                        cur_slot = ns;
                        bpos = nb + (k - avail);
                        bend = nb + kBatch;
                        if (!kFuse && lane == 0) next_batch = atomicAdd(A.task_counter, (unsigned long long)kBatch);
                    } else {
                        my = rank < avail ? bpos + rank : -1;
                        myslot = cur_slot;
                        bpos = bend;

                    }
                }
                if (needc && !warp_done && my >= 0 && my < n_tasks) {
                    if (kFuse) s_tslot[threadIdx.x] = (unsigned char)myslot;
                    int64_t t = A.task_list ? A.task_list[my] : my;
                    // the task's range record from the block's shared-memory table (one LDS per
                    // field: selecting among the three ranges' parameters cost ~40 instructions)
                    // (queue index and task index lie in the same range: the chunk-major order permutes
                    // the tasks of each range among themselves)
                    const RangeRec &Q = s_rng[task_range(A.tm, t)];
                    int64_t s, ch;
                    if (Q.il_s > 0 && !A.task_list) {
                        // chunk-major queue: position m of the range = chunk ch of its sample s
                        // (m = ch ns + s; fp64 quotient estimate, no 64-bit division); canonical task
                        // index t = t0 + s n_chunks + ch
                        divmod_est(my - Q.t0, Q.il_s, Q.inv_il, ch, s);
                        t = Q.t0 + s * Q.n_chunks + ch;
                    } else {
                        divmod_est(t - Q.t0, Q.n_chunks, Q.inv_chunks, s, ch);
                    }
                    s += Q.s0;
                    const int64_t *seg_k = Q.seg, *cap_k = Q.cap;
                    s_task[ci] = t;
                    g[c] = (int32_t)seg_k[ch];
                    g_end[c] = (int32_t)seg_k[ch + 1];
                    if (A.rerun_base) {
                        const int64_t sl = A.rerun_base[t] + A.out_base;
                        eb[c] = A.edges + sl;
                        cap[c] = (int32_t)max((int64_t)0, min((int64_t)INT32_MAX, A.out_cap - sl));  // bounded by the list
                    } else {
                        const int64_t c0 = cap_k[ch];
                        eb[c] = A.edges + (s * A.tm.cap_per_sample + c0);
                        cap[c] = (int32_t)(cap_k[ch + 1] - c0);
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
            // a task without segments (an empty last lane-chunk) fetched in this very round has not
            // recorded its end yet (count, spill, batch bookkeeping happen at the lane's next fetch
            // round): one more round before the warp leaves -- its counts were left unwritten when
            // the queue ended with such tasks (found by tests/test_gpu_fuzz.py)
            bool pend = false;
#pragma unroll
            for (int c = 0; c < kC; c++) pend = pend || s_task[threadIdx.x * kC + c] >= 0;
            if (warp_done && !__any_sync(0xffffffffu, pend)) break;
            if (kFuse && fuse) {  // (ring full: the copier is behind)
                __nanosleep(256);
            }
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
                        kv[c] = A.kappa_s[cur[c]];  // (ld.global.cg / .nc measured +-0 on config 4)
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
                            if (kGather == 2 && !kFuse) {  // large N: evict-first, the L2 keeps the kappa gather target (-0.7 %)
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
        const int wi = blockIdx.x * (kT / 32) + (threadIdx.x >> 5);
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
    if (kFuse && fuse) {  // after the warp's last task end
        __syncwarp();
        __threadfence_block();
        if (lane == 0) atomicAdd(&R.exited, 1u);
    }
    if (kCheck && __any_sync(0xffffffffu, bad_bound) && lane == 0) atomicOr(A.flags, kErrBound);
    if (A.rerun_base) return;
    unsigned long long dr = n_draw, ac = n_acc;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        dr += __shfl_xor_sync(0xffffffffu, dr, o);
        ac += __shfl_xor_sync(0xffffffffu, ac, o);
    }
    __syncwarp();
    dr += s_ndraw[threadIdx.x >> 5];
    ac += s_nacc[threadIdx.x >> 5];
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

// (128 threads at <= 32 registers, like k_offsets: they fit next to the resident sampler blocks)
__global__ void __launch_bounds__(128, 16) k_overflow(int64_t n_tasks, const TaskMap tm, const int64_t *__restrict__ counts,
                                                      const int64_t *__restrict__ spill_off, unsigned long long *n_overflow,
                                                      int64_t *__restrict__ overflow_list)
{
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n_tasks) return;
    int64_t s, c;
    int k;
    task_decode(tm, t, s, c, k);
    if (task_overflowed(counts[t], FM_TM_SEL(tm, cap, k)[c + 1] - FM_TM_SEL(tm, cap, k)[c], spill_off[t])) {
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
                                                          int ordered, const int64_t *__restrict__ out_base)
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
            const int64_t cap = FM_TM_SEL(tm, cap, k)[c + 1] - FM_TM_SEL(tm, cap, k)[c];
            const int64_t cnt = counts[t];
            sp = spill_off[t];
            dst = dest[t] + (out_base ? *out_base : 0);  // (+ the edges of the preceding sample groups)
            // tasks that would land beyond the list are dropped: the host sees the total and redoes the write
            cn = task_overflowed(cnt, cap, sp) || dst + cnt > out_cap ? 0 : (int32_t)cnt;
            cp = (int32_t)cap;
            src = s * tm.cap_per_sample + FM_TM_SEL(tm, cap, k)[c];
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

// Compaction with a small footprint (128 threads, <= 32 registers, 48 KB of shared memory): one
// such block fits into the 4096 registers per SM that three 256-thread sampler blocks at 80
// registers leave free (the sampler's shared-memory carveout leaves it room), so the compaction
// of sample group g runs NEXT TO the persistent sampler of group g + 1 on every SM (DESIGN.md
// 12.3: HBM is ~10 % busy under the sampler).  With so few registers -- and with the SM's
// load/store path busy with the sampler's gathers -- the bytes in flight go through the TMA
// engine: each warp copies 32 consecutive tasks (lane l holds task l's slot, final position and
// count); per round the next tasks whose slots fit one 6 KB staging buffer are loaded by ONE
// cp.async.bulk per task (issued by the task's own lane, completing on the buffer's mbarrier),
// double-buffered, and the warp stores a landed round task by task with aligned 16-byte stores
// (a task at an odd final position: its first edge alone, then pairs re-aligned through shared
// memory).  Slots must be 32-byte aligned (Plan::slots_aligned).  *out_base (device) is added to
// every final position: the edges of the preceding sample groups.
constexpr int kC2Threads = 128, kC2Buf = 6144;
constexpr int kC2Smem = (kC2Threads / 32) * (2 * kC2Buf + 16);  // bytes per block (dynamic)
#ifdef FM_C2_STATS  // instrumentation build: blocks and block time per SM, first start / last end
__device__ unsigned long long g_c2[256][2];
__device__ unsigned long long g_c2t[2] = {~0ull, 0ull};
#endif
template <bool kMap, bool kRec>
__global__ void __launch_bounds__(kC2Threads, 16) k_compact2(int64_t n_tasks, const TaskMap tm,
                                                             const int64_t *__restrict__ counts,
                                                             const int64_t *__restrict__ dest,
                                                             const int64_t *__restrict__ spill_off,
                                                             const int4 *__restrict__ se4, const int2 *__restrict__ spe,
                                                             const int32_t *__restrict__ spw, int2 *__restrict__ oe,
                                                             int32_t *__restrict__ ow, int64_t out_cap,
                                                             const int32_t *__restrict__ rank_map, int ordered,
                                                             const int64_t *__restrict__ out_base)
{
    extern __shared__ __align__(128) unsigned char s_c2[];
#ifdef FM_C2_STATS
    unsigned long long c2_t0 = 0;
    {
        asm volatile("mov.u64 %0, %globaltimer;" : "=l"(c2_t0));
        if (threadIdx.x == 0) atomicMin(&g_c2t[0], c2_t0);
    }
#endif
    const int lane = threadIdx.x & 31;
    const int64_t t0 = ((int64_t)blockIdx.x * (kC2Threads / 32) + (threadIdx.x >> 5)) * 32;
    if (t0 >= n_tasks) return;  // (warp-uniform; the kernel has no block barrier)
    // this warp's two staging buffers and their mbarriers
    const uint32_t buf0 = (uint32_t)__cvta_generic_to_shared(s_c2) + (threadIdx.x >> 5) * (2 * kC2Buf + 16);
    const uint32_t mb0 = buf0 + 2 * kC2Buf;
    if (lane == 0) {
        mbar_init(mb0, 1);
        mbar_init(mb0 + 8, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    const int64_t t = t0 + lane;
    const int64_t base = out_base ? *out_base : 0;
    int64_t src = 0, dst = base;
    int32_t n1 = 0;
    bool spilled = false;
    if (t < n_tasks) {
        int64_t s, c;
        int kr;
        task_decode(tm, t, s, c, kr);
        const int64_t *capp = FM_TM_SEL(tm, cap, kr);
        const int64_t c0 = capp[c];
        const int64_t cap = capp[c + 1] - c0;
        const int64_t cnt = counts[t];
        dst = dest[t] + base;
        // tasks that would land beyond the list are dropped: the host sees the total and redoes the write
        const bool drop = task_overflowed(cnt, cap, spill_off[t]) || dst + cnt > out_cap;
        n1 = drop ? 0 : (int32_t)min(cnt, cap);
        spilled = !drop && cnt > cap;
        src = s * tm.cap_per_sample + c0;
    }
    // staged bytes of the task's slot part: whole 16-byte units (a slot is a multiple of 32 bytes)
    const uint32_t bytes = kRec ? (uint32_t)n1 * 16u : (uint32_t)((n1 + 1) & ~1) * 8u;
    const char *gsrc = reinterpret_cast<const char *>(se4) + (size_t)src * (kRec ? 16 : 8);
    __syncwarp();
    // store the staged task (final position d, n elements, staged at shared address sa), warp-wide
    auto store_task = [&](int64_t d, int32_t n, uint32_t sa) {
        if (kRec) {
            for (int32_t e = lane; e < n; e += 32) {
                int4 v;
                asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(sa + e * 16));
                __stcs(oe + d + e, make_int2(v.x, v.y));
                __stcs(ow + d + e, v.z);
            }
            return;
        }
        // pairs (e, e + 1) at even final positions: e = odd + 2 lane, ... (odd: element 0 alone first)
        const int32_t odd = (int32_t)(d & 1);
        if (odd && lane == 0) {
            int2 v;
            asm volatile("ld.shared.v2.b32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(sa));
            if (kMap) {
                v.y = __ldg(rank_map + v.y);
                if (!ordered) v = make_int2(min(v.x, v.y), max(v.x, v.y));
            }
            __stcs(oe + d, v);
        }
        for (int32_t e = odd + 2 * lane; e < n; e += 64) {
            int4 v;
            if (odd) {
                asm volatile("ld.shared.v2.b32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(sa + e * 8));
                if (e + 1 < n) asm volatile("ld.shared.v2.b32 {%0,%1}, [%2];" : "=r"(v.z), "=r"(v.w) : "r"(sa + e * 8 + 8));
            } else {
                asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(sa + e * 8));
            }
            if (kMap) {  // (row id, candidate rank) -> the candidate's id, oriented
                v.y = __ldg(rank_map + v.y);
                if (e + 1 < n) v.w = __ldg(rank_map + v.w);
                if (!ordered) v = make_int4(min(v.x, v.y), max(v.x, v.y), min(v.z, v.w), max(v.z, v.w));
            }
            if (e + 1 < n) __stcs(reinterpret_cast<int4 *>(oe + d + e), v);
            else __stcs(oe + d + e, make_int2(v.x, v.y));
        }
    };
    // (rare) a slot part larger than a staging buffer: plain warp copy
    {
        unsigned big = __ballot_sync(0xffffffffu, n1 > 0 && bytes > (uint32_t)kC2Buf);
        while (big) {
            const int k = __ffs(big) - 1;
            big &= big - 1;
            const int64_t d_k = __shfl_sync(0xffffffffu, dst, k), s_k = __shfl_sync(0xffffffffu, src, k);
            const int32_t n_k = __shfl_sync(0xffffffffu, n1, k);
            for (int32_t e = lane; e < n_k; e += 32) {
                if (kRec) {
                    const int4 v = se4[s_k + e];
                    oe[d_k + e] = make_int2(v.x, v.y);
                    ow[d_k + e] = v.z;
                } else {
                    int2 v = reinterpret_cast<const int2 *>(se4)[s_k + e];
                    if (kMap) {
                        v.y = __ldg(rank_map + v.y);
                        if (!ordered) v = make_int2(min(v.x, v.y), max(v.x, v.y));
                    }
                    oe[d_k + e] = v;
                }
            }
        }
    }
    bool pending = n1 > 0 && bytes <= (uint32_t)kC2Buf;
    // two-stage pipeline over rounds: round r's loads are issued into buffer r & 1, then round r - 1
    // (the other buffer) is awaited and stored
    bool p_mine = false;     // this lane's task is in the round in flight
    uint32_t p_off = 0;      //   at this offset of its buffer
    int p_buf = 0, r = 0;
    bool p_any = false;
    unsigned ph = 0;         // bit b: phase parity of buffer b's mbarrier
    for (;;) {
        const bool any = __any_sync(0xffffffffu, pending);
        if (!any && !p_any) break;
        bool mine = false;
        uint32_t off = 0;
        const int b = r & 1;
        if (any) {
            // this round: the pending tasks, in lane order, whose staging ranges fit the buffer
            const uint32_t sz = pending ? bytes : 0u;
            uint32_t inc = sz;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t v = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += v;
            }
            off = inc - sz;
            mine = pending && inc <= (uint32_t)kC2Buf;  // (the first pending task always fits)
            const uint32_t total = __reduce_add_sync(0xffffffffu, mine ? sz : 0u);
            // buffer b was last read by the stores of round r - 2 (generic proxy): order the
            // async-proxy writes after them
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive_expect(mb0 + 8 * b, total);
            __syncwarp();
            if (mine) bulk_g2s(buf0 + b * kC2Buf + off, gsrc, bytes, mb0 + 8 * b);
            pending = pending && !mine;
        }
        if (p_any) {  // finish the previous round
            mbar_wait(mb0 + 8 * p_buf, (ph >> p_buf) & 1u);
            ph ^= 1u << p_buf;
            unsigned m = __ballot_sync(0xffffffffu, p_mine);
            while (m) {
                const int k = __ffs(m) - 1;
                m &= m - 1;
                store_task(__shfl_sync(0xffffffffu, dst, k), __shfl_sync(0xffffffffu, n1, k),
                           buf0 + p_buf * kC2Buf + __shfl_sync(0xffffffffu, p_off, k));
            }
            __syncwarp();
        }
        p_any = any;
        p_mine = mine;
        p_off = off;
        p_buf = b;
        r++;
    }
#ifdef FM_C2_STATS
    if (threadIdx.x == 0) {
        unsigned long long t1;
        unsigned sm;
        asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t1));
        asm volatile("mov.u32 %0, %smid;" : "=r"(sm));
        atomicAdd(&g_c2[sm][0], 1ull);
        atomicAdd(&g_c2[sm][1], t1 - c2_t0);
        atomicMax(&g_c2t[1], t1);
    }
#endif
    // spilled tails (rare): the task's lane re-reads its metadata, the warp copies
    unsigned m = __ballot_sync(0xffffffffu, spilled);
    while (m) {
        const int k = __ffs(m) - 1;
        m &= m - 1;
        const int64_t tk = t0 + k;
        int64_t s, c;
        int kr;
        task_decode(tm, tk, s, c, kr);
        const int64_t *capp = FM_TM_SEL(tm, cap, kr);
        const int64_t cap = capp[c + 1] - capp[c];
        const int64_t cnt = counts[tk], sp = spill_off[tk];
        const int64_t d_k = dest[tk] + base;
        for (int64_t i = cap + lane; i < cnt; i += 32) {
            int2 ev = spe[sp + i - cap];
            if (kMap) {
                const int32_t id = __ldg(rank_map + ev.y);
                ev = ordered ? make_int2(ev.x, id) : make_int2(min(ev.x, id), max(ev.x, id));
            }
            oe[d_k + i] = ev;
            if (kRec) ow[d_k + i] = spw[sp + i - cap];
        }
    }
}

// per-sample offsets of a sample group: offsets[s] = base + dest[first task of sample s], and the
// running total for the next group, base_next = base + dest[n_tasks]
__global__ void __launch_bounds__(128, 16) k_offsets(int64_t n_samples, const TaskMap tm, const int64_t *__restrict__ dest,
                                                     int64_t *__restrict__ offsets, const int64_t *__restrict__ base_in,
                                                     int64_t *base_out, int64_t *base_out_host)
{
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s > n_samples) return;
    const int64_t base = base_in ? *base_in : 0;
    const int64_t v = base + dest[sample_first_task(tm, s)];  // dest[n_tasks] is the group's total
    offsets[s] = v;
    if (s == n_samples && base_out) *base_out = v;
    // (mapped page-locked host word: the host learns the group's end without a copy-engine transfer,
    // which would queue behind the D2H copies of the preceding groups' edges)
    if (s == n_samples && base_out_host) *(volatile int64_t *)base_out_host = v;
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

void fuse_stats_dump()
{
#ifdef FM_C2_STATS
    {
        static unsigned long long h[256][2], ht[2];
        if (cudaMemcpyFromSymbol(h, g_c2, sizeof(h)) == cudaSuccess && cudaMemcpyFromSymbol(ht, g_c2t, sizeof(ht)) == cudaSuccess) {
            unsigned long long nb = 0, tt = 0, mn = ~0ull, mx = 0;
            int used = 0;
            for (int i = 0; i < 256; i++) {
                nb += h[i][0];
                tt += h[i][1];
                if (h[i][0]) {
                    used++;
                    mn = h[i][0] < mn ? h[i][0] : mn;
                    mx = h[i][0] > mx ? h[i][0] : mx;
                }
            }
            fprintf(stderr, "[c2] blocks %llu on %d SMs (min %llu max %llu per SM), mean block time %.1f us, span %.3f ms\n", nb, used,
                    mn, mx, nb ? 1e-3 * (double)tt / (double)nb : 0.0, 1e-6 * (double)(ht[1] - ht[0]));
            static unsigned long long z[256][2], zt[2] = {~0ull, 0ull};
            cudaMemcpyToSymbol(g_c2, z, sizeof(z));
            cudaMemcpyToSymbol(g_c2t, zt, sizeof(zt));
        }
    }
#endif
#ifdef FM_FUSE_STATS
    unsigned long long h[8];
    if (cudaMemcpyFromSymbol(h, g_fstats, sizeof(h)) != cudaSuccess) return;
    fprintf(stderr, "[fuse] copies %llu copy_cycles/copy %.0f idle_polls %llu blocked_entries %llu ring_full %llu "
                    "all_idle_iters %llu desc_cycles/copy %.0f job_cycles/copy %.0f\n", h[0], h[0] ? (double)h[1] / h[0] : 0.0,
            h[2], h[3], h[4], h[5], h[0] ? (double)h[6] / h[0] : 0.0, h[0] ? (double)h[7] / h[0] : 0.0);
    static unsigned long long z[8];
    cudaMemcpyToSymbol(g_fstats, z, sizeof(z));
#endif
}

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
template <int kModel, int kMinB, int kC, bool kStats, bool kRefresh, int kGather, bool kOrdered, bool kCheck,
          bool kFuse>
static cudaError_t launch_sample_t(const SampleArgs &a, cudaStream_t st)
{
    auto kern = k_sample<kModel, kMinB, kC, kStats, kRefresh, kGather, kOrdered, kCheck, kFuse>;
    constexpr int kT = sampler_threads(kFuse, kGather);
    int dev = 0, sms = 0, per = 0;
    cudaError_t err = cudaGetDevice(&dev);
    if (err == cudaSuccess) err = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (err != cudaSuccess) return err;
    const size_t dyn = (size_t)kT * kC * (kModel == FM_ECM ? 96 : 64) + (kFuse ? 2 * kStageBuf + 128 : 0);
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
            // (FM_SAMPLE_GROUPS set: + one co-resident small-footprint compaction block of the pipelined
            // sample groups; the driver rounds the preference down as long as the sampler fits, so in
            // practice only FM_SAMPLE_CARVEOUT=100 makes that room)
            const size_t need = (size_t)(kFuse ? 1 : kMinB) * (fa.sharedSizeBytes + dyn + 1024) +
                                (getenv("FM_SAMPLE_GROUPS") ? kC2Smem + 2048 : 0);
            const int pct = (int)((need * 100 + 228 * 1024 - 1) / (228 * 1024));
            carve = std::max(carve, std::min(pct, 100));
        }
        if (carve >= 0) {
            err = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, carve);
            if (err != cudaSuccess) return err;
        }
        attr_set[dev] = true;
    }
    err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, kT, dyn);
    if (err != cudaSuccess) return err;
    int64_t blocks = (int64_t)sms * (per > 0 ? per : 1);
    const int64_t need = (a.n_tasks + kT * kC - 1) / (kT * kC);  // <= one task per chain at start
    if (need < blocks) blocks = need;
    count_launch();
    kern<<<(unsigned)blocks, kT, dyn, st>>>(a);
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
            return launch_sample_t<kModel, kMinB, 1, kStats, kRefresh, kGather, true, kCheck, false>(a, st);
    if constexpr (kModel == FM_UBCM && !kStats)
        if (a.fuse && !a.rerun_base && !a.ordered)
            return launch_sample_t<kModel, kMinB, 1, kStats, kRefresh, kGather, false, kCheck, true>(a, st);
    return launch_sample_t<kModel, kMinB, 1, kStats, kRefresh, kGather, false, kCheck, false>(a, st);
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
    if (!a.counters_zeroed) {
        e = cudaMemsetAsync(a.task_counter, 0, sizeof(unsigned long long), st);
        if (e != cudaSuccess) return e;
    }
    if (a.spill_counter && !a.rerun_base && !a.counters_zeroed) {
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
    k_overflow<<<(unsigned)((n_tasks + 127) / 128), 128, 0, st>>>(n_tasks, tm, counts, spill_off, n_overflow,
                                                                 overflow_list);
    return cudaGetLastError();
}

cudaError_t launch_compact(int64_t out_cap, int64_t n_tasks, const TaskMap &tm, const int64_t *counts, const int64_t *dest,
                           const int64_t *spill_off, const int2 *scratch_e, const int32_t *scratch_w,
                           const int2 *spill_e, const int32_t *spill_w, int2 *out_e, int32_t *out_w,
                           const int32_t *rank_map, int ordered, int ecm_rec, int small, const int64_t *out_base,
                           cudaStream_t st)
{
    if (n_tasks <= 0 || out_cap <= 0) return cudaSuccess;
    count_launch();
    if (small) {
        // small-footprint kernel (aligned slots; UBCM pairs or ECM records): co-resident with the sampler
        const unsigned grid = (unsigned)((n_tasks + kC2Threads - 1) / kC2Threads);
        const int4 *se4 = reinterpret_cast<const int4 *>(scratch_e);
        auto go = [&](auto kern) -> cudaError_t {
            cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kC2Smem);
            if (e != cudaSuccess) return e;
            kern<<<grid, kC2Threads, kC2Smem, st>>>(n_tasks, tm, counts, dest, spill_off, se4, spill_e, spill_w, out_e, out_w,
                                                    out_cap, rank_map, ordered, out_base);
            return cudaGetLastError();
        };
        if (rank_map) return go(k_compact2<true, false>);
        if (ecm_rec) return go(k_compact2<false, true>);
        return go(k_compact2<false, false>);
    }
    const unsigned grid = (unsigned)((n_tasks + kCopyThreads - 1) / kCopyThreads);
    if (rank_map) {
        // the rank -> id gathers like a large L1: 25 % carveout (15-25 %: config 4 write 1.07 -> 1.04 ms;
        // 0 % and 100 %: 2.3-2.6 ms); FM_COMPACT_CARVEOUT overrides
        const char *cv = getenv("FM_COMPACT_CARVEOUT");
        cudaFuncSetAttribute(k_compact<true, false>, cudaFuncAttributePreferredSharedMemoryCarveout,
                             cv && *cv ? atoi(cv) : 25);
    }
    if (rank_map)
        k_compact<true, false><<<grid, kCopyThreads, 0, st>>>(n_tasks, tm, counts, dest, spill_off, scratch_e,
                                                              scratch_w, spill_e, spill_w, out_e, out_w, out_cap,
                                                              rank_map, ordered, out_base);
    else if (ecm_rec)
        k_compact<false, true><<<grid, kCopyThreads, 0, st>>>(n_tasks, tm, counts, dest, spill_off, scratch_e,
                                                              scratch_w, spill_e, spill_w, out_e, out_w, out_cap,
                                                              rank_map, ordered, out_base);
    else
        k_compact<false, false><<<grid, kCopyThreads, 0, st>>>(n_tasks, tm, counts, dest, spill_off, scratch_e,
                                                               scratch_w, spill_e, spill_w, out_e, out_w, out_cap,
                                                               rank_map, ordered, out_base);
    return cudaGetLastError();
}

cudaError_t launch_offsets(int64_t n_samples, const TaskMap &tm, const int64_t *dest, int64_t *offsets,
                           const int64_t *base_in, int64_t *base_out, int64_t *base_out_host, cudaStream_t st)
{
    count_launch();
    k_offsets<<<(unsigned)((n_samples + 1 + 127) / 128), 128, 0, st>>>(n_samples, tm, dest, offsets, base_in, base_out,
                                                                      base_out_host);
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
