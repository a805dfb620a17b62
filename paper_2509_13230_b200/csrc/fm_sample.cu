// fm_sample.cu -- a5 (the chain) and a6 (count -> scan -> write) on sm_100a.
//
// Work decomposition: one warp per task = (sample s, chunk c); a chunk is a run of plan
// segments in canonical order with ~equal estimated draws.  Inside the warp every lane runs
// one segment's chain at a time (lane-per-chain, lock-step one draw per iteration); a lane
// whose segment ends takes the next unclaimed segment of the chunk (warp-uniform cursor via
// __ballot_sync), so lanes stay busy until the chunk is exhausted.  Accepted edges of an
// iteration are compacted with ballot/popc and stored contiguously (coalesced 8-byte
// stores) into the chunk's scratch slot; the slot order is deterministic (iteration, lane).
//
// Decision arithmetic: the exact operation sequence of DESIGN.md 3.5 with RN intrinsics
// (no contraction), CUDA libdevice log/log1p (<= 1 ulp; the only difference from the oracle).
#include <float.h>

#include "fm_internal.cuh"
#include "fm_plan_kernels.cuh"

namespace fm {
namespace {

constexpr int kWarpsPerBlock = 4;

template <int kModel>
__global__ void __launch_bounds__(kWarpsPerBlock * 32) k_sample(const SampleArgs A)
{
    const int lane = threadIdx.x & 31;
    int64_t task = (int64_t)blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
    if (task >= A.n_tasks) return;  // warp-uniform
    if (A.task_list) task = A.task_list[task];
    const int64_t s = task / A.n_chunks;
    const int64_t c = task - s * A.n_chunks;
    const int64_t g1 = A.chunk_seg[c + 1];
    int64_t next_g = A.chunk_seg[c];
    int64_t base, cap;
    if (A.rerun_base) {
        base = A.rerun_base[task];
        cap = INT64_MAX;
    } else {
        base = task * A.cap;
        cap = A.cap;
    }
    const uint32_t s_abs = A.first_sample + (uint32_t)s;
    const uint32_t lt = (1u << lane) - 1u;

    bool has = false;
    int32_t u = 0, b = 0, cur = 0, id_u = 0;
    uint32_t sigma = 0, d = 0;
    double q = 0.0, h = 0.0, ku = 0.0, yu = 0.0, omT = 1.0;
    uint32_t n_draw = 0, n_land = 0, n_acc = 0;
    bool wsat = false;
    int64_t out_n = 0;

    for (;;) {
        // ---- refill: lanes without a segment claim the next ones, in lane order ----
        const uint32_t need = __ballot_sync(0xffffffffu, !has);
        if (need && next_g < g1) {
            const int64_t g = next_g + __popc(need & lt);
            if (!has && g < g1) {
                const int4 sg = A.seg[g];
                u = sg.x;
                cur = sg.y - 1;  // virtual previous position a-1 (R3)
                b = sg.z;
                sigma = (uint32_t)sg.w;
                q = A.seg_q0[g];
                h = A.seg_h0[g];
                ku = A.kappa_s[u];
                id_u = A.perm[u];
                if (kModel == FM_ECM) {
                    yu = A.y_s[u];
                    omT = A.seg_omT[g];
                }
                d = 0;
                has = true;
            }
            next_g += __popc(need);
            if (next_g > g1) next_g = g1;
        }
        if (!__any_sync(0xffffffffu, has)) break;

        bool acc = false;
        int32_t id_v = 0, w = 1;
        if (has) {
            uint32_t w_skip, w_acc, w_wt = 0;
            if (kModel == FM_UBCM) {
                const uint4 W = philox4x32_10(make_uint4(d >> 1, sigma, (uint32_t)u, s_abs), A.k0, A.k1);
                w_skip = (d & 1) ? W.z : W.x;
                w_acc = (d & 1) ? W.w : W.y;
            } else {
                const uint4 W = philox4x32_10(make_uint4(d, sigma, (uint32_t)u, s_abs), A.k0, A.k1);
                w_skip = W.x;
                w_acc = W.y;
                w_wt = W.z;
            }
            n_draw++;
            const double E = -log(u01(w_skip));
            const double R = __ddiv_rn(E, h);
            if (!(R < (double)(b - 1 - cur))) {
                has = false;  // terminal draw: end of this segment's candidate list (R5)
            } else {
                cur = cur + 1 + (int32_t)R;  // R >= 0: truncation == floor
                n_land++;
                const double kv = A.kappa_s[cur];
                if (kModel == FM_UBCM) {
                    const double X = __dmul_rn(ku, kv);
                    const double p = __ddiv_rn(X, __dadd_rn(1.0, X));
                    acc = __dmul_rn(u01(w_acc), q) < p;
                    q = p;
                    h = log1p(X);
                } else {
                    const double z = __dmul_rn(ku, kv);
                    const double t = __dmul_rn(yu, A.y_s[cur]);
                    const double p = __ddiv_rn(z, __dadd_rn(__dsub_rn(1.0, t), z));
                    acc = __dmul_rn(u01(w_acc), q) < p;
                    if (acc) {
                        const double G = floor(__ddiv_rn(log(u01(w_wt)), log(t)));
                        if (G <= 2147483646.0) {
                            w = 1 + (int32_t)G;
                        } else {
                            w = INT32_MAX;
                            wsat = true;
                        }
                    }
                    q = __ddiv_rn(z, __dadd_rn(omT, z));
                    h = log1p(__ddiv_rn(z, omT));
                }
                d++;
                if (acc) {
                    id_v = A.perm[cur];
                    n_acc++;
                }
            }
        }
        // ---- emit: warp-compacted contiguous stores ----
        const uint32_t am = __ballot_sync(0xffffffffu, acc);
        if (am) {
            if (acc) {
                const int64_t pos = out_n + __popc(am & lt);
                if (pos < cap) {
                    A.edges[base + pos] = make_int2(min(id_u, id_v), max(id_u, id_v));
                    if (kModel == FM_ECM) A.weights[base + pos] = w;
                }
            }
            out_n += __popc(am);
        }
    }
    if (A.rerun_base) return;
    const unsigned dr = __reduce_add_sync(0xffffffffu, n_draw);
    const unsigned la = __reduce_add_sync(0xffffffffu, n_land);
    const unsigned ac = __reduce_add_sync(0xffffffffu, n_acc);
    const bool anysat = __any_sync(0xffffffffu, wsat);
    if (lane == 0) {
        A.counts[task] = out_n;
        atomicAdd(&A.counters[0], (unsigned long long)dr);
        atomicAdd(&A.counters[1], (unsigned long long)la);
        atomicAdd(&A.counters[2], (unsigned long long)ac);
        if (anysat) atomicOr(A.flags, kFlagWeightSat);
    }
}

__global__ void __launch_bounds__(256) k_overflow(int64_t n_tasks, int64_t cap, const int64_t *__restrict__ counts,
                                                  unsigned long long *n_overflow, int64_t *__restrict__ overflow_list)
{
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < n_tasks && counts[t] > cap) {
        const unsigned long long k = atomicAdd(n_overflow, 1ull);
        overflow_list[k] = t;
    }
}

// one block per task: copy the task's scratch slot to its final position (overflowed tasks
// are skipped; they are re-run straight into the final array, with identical results)
__global__ void __launch_bounds__(256) k_compact(int64_t n_tasks, int64_t cap, const int64_t *__restrict__ counts,
                                                 const int64_t *__restrict__ dest, const int2 *__restrict__ se,
                                                 const int32_t *__restrict__ sw, int2 *__restrict__ oe,
                                                 int32_t *__restrict__ ow)
{
    for (int64_t t = blockIdx.x; t < n_tasks; t += gridDim.x) {
        const int64_t cnt = counts[t];
        if (cnt > cap) continue;
        const int64_t src = t * cap;
        const int64_t dst = dest[t];
        for (int64_t i = threadIdx.x; i < cnt; i += blockDim.x) {
            oe[dst + i] = se[src + i];
            if (ow) ow[dst + i] = sw[src + i];
        }
    }
}

__global__ void k_offsets(int64_t n_samples, int64_t n_chunks, const int64_t *__restrict__ dest,
                          int64_t *__restrict__ offsets)
{
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s <= n_samples) offsets[s] = dest[s * n_chunks];
}

}  // namespace

cudaError_t launch_sample(int model, const SampleArgs &a, cudaStream_t st)
{
    if (a.n_tasks <= 0) return cudaSuccess;
    const int64_t blocks = (a.n_tasks + kWarpsPerBlock - 1) / kWarpsPerBlock;
    count_launch();
    if (model == FM_UBCM)
        k_sample<FM_UBCM><<<(unsigned)blocks, kWarpsPerBlock * 32, 0, st>>>(a);
    else
        k_sample<FM_ECM><<<(unsigned)blocks, kWarpsPerBlock * 32, 0, st>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_overflow(int64_t n_tasks, int64_t cap, const int64_t *counts, unsigned long long *n_overflow,
                            int64_t *overflow_list, cudaStream_t st)
{
    if (n_tasks <= 0) return cudaSuccess;
    count_launch();
    k_overflow<<<(unsigned)((n_tasks + 255) / 256), 256, 0, st>>>(n_tasks, cap, counts, n_overflow, overflow_list);
    return cudaGetLastError();
}

cudaError_t launch_compact(int64_t n_tasks, int64_t cap, const int64_t *counts, const int64_t *dest,
                           const int2 *scratch_e, const int32_t *scratch_w, int2 *out_e, int32_t *out_w,
                           cudaStream_t st)
{
    if (n_tasks <= 0) return cudaSuccess;
    const int64_t grid = n_tasks < 1048576 ? n_tasks : 1048576;
    count_launch();
    k_compact<<<(unsigned)grid, 256, 0, st>>>(n_tasks, cap, counts, dest, scratch_e, scratch_w, out_e, out_w);
    return cudaGetLastError();
}

cudaError_t launch_offsets(int64_t n_samples, int64_t n_chunks, const int64_t *dest, int64_t *offsets, cudaStream_t st)
{
    count_launch();
    k_offsets<<<(unsigned)((n_samples + 1 + 255) / 256), 256, 0, st>>>(n_samples, n_chunks, dest, offsets);
    return cudaGetLastError();
}

}  // namespace fm
