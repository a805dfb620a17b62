// fm_plan.cu -- a1 (validate + key), a2 gathers, a3 (beta_min suffix max), a4 (planner).
// Every floating-point operation on the planner path is an explicit round-to-nearest
// intrinsic in the order of DESIGN.md section 3.4, so the plan is bit-identical to the
// oracle's (compiled with --fmad=false as a second guard).
#include <float.h>

#include "fm_internal.cuh"
#include "fm_plan_kernels.cuh"

namespace fm {

// ------------------------------------------------------------------------------------------
// a1: validate (x finite >= 0; ECM y in [0,1); kappa^2 finite) and build the radix key
// ~bits(kappa) (kappa = x or x*y; -0.0 normalised to +0.0).
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_validate_key(int model, int64_t n, const double *__restrict__ x,
                                                      const double *__restrict__ y, uint64_t *__restrict__ keys,
                                                      int32_t *__restrict__ ids, PlanScalars *sc,
                                                      unsigned int *__restrict__ hist)
{
    // also: the radix digit histograms of all 8 byte positions (fm_sort.cu consumes them).
    // Grid-stride (a bounded grid): each block accumulates in shared memory and flushes its
    // 8 x 256 counts and its key OR/AND once.
    __shared__ unsigned int h[8][256];
    __shared__ unsigned long long s_or, s_and;
    __shared__ int s_bad;
    for (int p = 0; p < 8; p++) h[p][threadIdx.x] = 0;
    if (threadIdx.x == 0) {
        s_or = 0;
        s_and = ~0ull;
        s_bad = 0;
    }
    __syncthreads();
    uint64_t kor = 0, kand = ~0ull;
    bool bad = false;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double xi = x[i];
        bool ok = isfinite(xi) && xi >= 0.0;
        double kappa = xi;
        if (model == FM_ECM) {
            const double yi = y[i];
            ok = ok && isfinite(yi) && yi >= 0.0 && yi < 1.0;
            kappa = __dmul_rn(xi, yi);
        }
        kappa = __dadd_rn(kappa, 0.0);  // -0.0 -> +0.0
        const double k2 = __dmul_rn(kappa, kappa);
        ok = ok && isfinite(__dmul_rn(k2, k2));  // R10's cross products stay finite
        const uint64_t key = ~(uint64_t)__double_as_longlong(kappa);
        keys[i] = key;
        ids[i] = (int32_t)i;
        kor |= key;
        kand &= key;
        bad = bad || !ok;
#pragma unroll
        for (int p = 0; p < 8; p++) atomicAdd(&h[p][(key >> (8 * p)) & 0xFF], 1u);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        kor |= __shfl_xor_sync(0xffffffffu, kor, o);
        kand &= __shfl_xor_sync(0xffffffffu, kand, o);
    }
    const bool anybad = __any_sync(0xffffffffu, bad);
    if ((threadIdx.x & 31) == 0) {
        atomicOr(&s_or, (unsigned long long)kor);
        atomicAnd(&s_and, (unsigned long long)kand);
        if (anybad) s_bad = 1;
    }
    __syncthreads();
    for (int p = 0; p < 8; p++)
        if (h[p][threadIdx.x]) atomicAdd(&hist[p * 256 + threadIdx.x], h[p][threadIdx.x]);
    if (threadIdx.x == 0) {
        atomicOr(&sc->key_or, s_or);
        atomicAnd(&sc->key_and, s_and);
        if (s_bad) atomicOr(&sc->flags, kErrInvalid);
    }
}

// a2 epilogue: rank-space arrays from the sorted keys
__global__ void __launch_bounds__(256) k_gather_sorted(int model, int64_t n, const uint64_t *__restrict__ skeys,
                                                       const double *__restrict__ y, const int32_t *__restrict__ perm,
                                                       double *__restrict__ kappa_s, double *__restrict__ y_s,
                                                       double *__restrict__ ly_s)
{
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    kappa_s[r] = __longlong_as_double((long long)~skeys[r]);
    if (model == FM_ECM) {
        const double yr = y[perm[r]];
        y_s[r] = yr;
        ly_s[r] = log(yr);  // R8: log t = log y_i + log y_j
    }
}

// a4 step 1-2: F and the fixed-point keys
__global__ void k_set_F(int64_t n, int L, const double *kappa_s, PlanScalars *sc)
{
    int e = 0;
    const double k0 = kappa_s[0];
    if (k0 > 0.0) frexp(k0, &e);
    sc->F = 61 - e - L;
}

__global__ void __launch_bounds__(256) k_kfx(int64_t n, int L, const double *__restrict__ kappa_s,
                                             PlanScalars *__restrict__ sc, uint64_t *__restrict__ kfx)
{
    const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n) return;
    int e = 0;
    const double k0 = kappa_s[0];
    if (k0 > 0.0) frexp(k0, &e);
    const int F = 61 - e - L;
    if (v == 0) sc->F = F;
    kfx[v] = (uint64_t)floor(ldexp(kappa_s[v], F));
}

// first candidate of row u: undirected j > u; bipartite / directed every - node
__device__ __forceinline__ int64_t row_c0(int kind, int64_t u) { return kind == FM_UNDIRECTED ? u + 1 : 0; }

// a4 step 3-4 (per row): r_u, sat_u, Wtot_u, m_u.  Rows: kappa_s/y_s (n); candidates: ckappa/ymax (nc).
__global__ void __launch_bounds__(256) k_rows(int model, int kind, int64_t n, int64_t nc, int64_t S,
                                              const double *__restrict__ kappa_s, const double *__restrict__ y_s,
                                              const double *__restrict__ ckappa, const double *__restrict__ ymax,
                                              const uint64_t *__restrict__ P, PlanScalars *sc, RowInfo *__restrict__ rows,
                                              int64_t *__restrict__ row_m)
{
    const int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    long long work = 0, wseg = 0;
    if (u < n) {
        const int64_t c0 = row_c0(kind, u);
        if (c0 < nc) {
            const int F = sc->F;
            double r = kappa_s[u];
            if (model == FM_ECM) r = __ddiv_rn(kappa_s[u], __dsub_rn(1.0, __dmul_rn(y_s[u], ymax[c0])));
            int64_t sat;
            if (__dmul_rn(r, ckappa[c0]) < 1.0) {
                sat = c0;
            } else {  // smallest v in [c0, nc] with v == nc or r*ckappa[v] < 1 (monotone predicate)
                int64_t lo = c0 + 1, hi = nc;
                while (lo < hi) {
                    const int64_t mid = lo + ((hi - lo) >> 1);
                    if (__dmul_rn(r, ckappa[mid]) < 1.0) hi = mid; else lo = mid + 1;
                }
                sat = lo;
            }
            const int64_t WN = plan_W(P, F, c0, r, sat, nc);
            const int64_t Wt = WN + kUnit;
            const int64_t m = (Wt + S * kUnit - 1) / (S * kUnit);
            rows[u].r = r;
            rows[u].sat = sat;
            rows[u].wtot = Wt;
            row_m[u] = m;
            work = WN + m * kUnit;
            // bound of one segment's work: Wtot (unsplit) or ceil(Wtot/m) + 2 units + 2 (DESIGN 7.2)
            wseg = m == 1 ? Wt : (Wt + m - 1) / m + 2 * kUnit + 2;
        } else {
            row_m[u] = 0;  // no candidates (the last undirected row): no segment, no draw
        }
    }
    // block reduce of work (int64): one pair of global atomics per block (a per-warp pair made
    // the 1e7-row plan wait ~0.5 ms on two contended addresses)
    __shared__ long long s_work[8], s_wseg[8];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        work += __shfl_xor_sync(0xffffffffu, work, o);
        wseg = max(wseg, __shfl_xor_sync(0xffffffffu, wseg, o));
    }
    if ((threadIdx.x & 31) == 0) {
        s_work[threadIdx.x >> 5] = work;
        s_wseg[threadIdx.x >> 5] = wseg;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        long long tw = 0, tm = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); w++) {
            tw += s_work[w];
            tm = max(tm, s_wseg[w]);
        }
        if (tw) {
            atomicAdd((unsigned long long *)&sc->total_work, (unsigned long long)tw);
            atomicMax(&sc->wmax, tm);
        }
    }
}

// cut k of row u (1 <= k < m): smallest v in [c0+1, nc-1] with W_u(v) >= floor(k Wtot / m), nc-1 if none
__device__ __forceinline__ int64_t plan_cut(const uint64_t *P, int F, int64_t nc, int64_t c0, const RowInfo &ri,
                                            int64_t m, int64_t k)
{
    const int64_t q = ri.wtot / m, rm = ri.wtot - q * m;
    const int64_t theta = k * q + (k * rm) / m;  // == floor(k * Wtot / m) exactly
    int64_t lo = c0 + 1, hi = nc - 1;
    while (lo < hi) {
        const int64_t mid = lo + ((hi - lo) >> 1);
        if (plan_W(P, F, c0, ri.r, ri.sat, mid) >= theta) hi = mid; else lo = mid + 1;
    }
    return lo;
}

// a4 step 5-6 (per segment): (u, a, b, sigma), initial bound (x0, d0, h0, omT), work estimate,
// written straight into the sampler's packed record (SegRec)
#ifndef FM_EMIT_MINB
#define FM_EMIT_MINB 6  // 42 registers: config-4 plan 1.99 -> 1.95 ms (5: 1.96, 8 spills: 2.07)
#endif
__global__ void __launch_bounds__(256, FM_EMIT_MINB) k_emit(int model, int kind, int64_t n, int64_t nc, int64_t n_seg,
                                              const double *__restrict__ kappa_s, const double *__restrict__ y_s,
                                              const double *__restrict__ ly_s, const int32_t *__restrict__ perm,
                                              const int32_t *__restrict__ excl, const double *__restrict__ ckappa,
                                              const double *__restrict__ ymax, const uint64_t *__restrict__ P,
                                              PlanScalars *sc, const RowInfo *__restrict__ rows,
                                              const int64_t *__restrict__ row_seg,
                                              const int64_t *__restrict__ seg_row_x, unsigned char *__restrict__ rec,
                                              int64_t *__restrict__ seg_work)
{
    __shared__ __align__(16) SegRec s_rec[256];  // the block's records, written out coalesced
    __shared__ int64_t s_u0;
    const int64_t g0 = (int64_t)blockIdx.x * blockDim.x;
    const int64_t g = g0 + threadIdx.x;
    const int nb = (int)min((int64_t)blockDim.x, n_seg - g0);  // records of this block
    // row u of segment g: largest u with row_seg[u] <= g.  Every row that has candidates has >= 1
    // segment (rows with candidates: n-1 undirected, all n otherwise).  Large plans: the number of
    // row starts at or before g, minus one (seg_row_x = exclusive scan of the row-start flags);
    // small plans (seg_row_x NULL, fewer launches): u(g) in [g - extra, g], the block's first row
    // u0 found once, then u(g) in [u0, u0 + (g - g0)]
    const int64_t rows_w = kind == FM_UNDIRECTED ? n - 1 : n;
    if (!seg_row_x) {
        const int64_t extra = n_seg - rows_w;
        if (threadIdx.x == 0) {
            int64_t lo = g0 - extra > 0 ? g0 - extra : 0, hi = g0 < rows_w - 1 ? g0 : rows_w - 1;
            while (lo < hi) {
                const int64_t mid = lo + ((hi - lo + 1) >> 1);
                if (row_seg[mid] <= g0) lo = mid; else hi = mid - 1;
            }
            s_u0 = lo;
        }
        __syncthreads();
    }
    if (g < n_seg) {
        const int F = sc->F;
        int64_t u;
        if (seg_row_x) {
            u = seg_row_x[g + 1] - 1;
        } else {
            int64_t lo = s_u0, hi = s_u0 + (g - g0) < rows_w - 1 ? s_u0 + (g - g0) : rows_w - 1;
            while (lo < hi) {
                const int64_t mid = lo + ((hi - lo + 1) >> 1);
                if (row_seg[mid] <= g) lo = mid; else hi = mid - 1;
            }
            u = lo;
        }
        const int64_t c0 = row_c0(kind, u);
        const int64_t sigma = g - row_seg[u];
        const int64_t m = row_seg[u + 1] - row_seg[u];
        const RowInfo ri = rows[u];
        int64_t a, b;
        a = sigma == 0 ? c0 : plan_cut(P, F, nc, c0, ri, m, sigma);
        b = sigma == m - 1 ? nc : plan_cut(P, F, nc, c0, ri, m, sigma + 1);
        if (!(a < b) || !(a >= c0)) atomicOr(&sc->flags, kErrState);
        SegRec r;
        r.u = (int)u;
        r.a = (int)a;
        r.b = (int)b;
        r.sigma = (int)sigma;
        // bound at the virtual previous position a-1 (R3); a bipartite row start uses candidate 0 (R16)
        const int64_t bp = a > 0 ? a - 1 : 0;
        const double ku = kappa_s[u];
        const double kq = __dmul_rn(ku, ckappa[bp]);
        r.x0 = kq;
        r.ku = ku;
        r.id_u = perm[u];
        r.excl = excl ? excl[u] : -1;
        if (model == FM_UBCM) {
            r.omT = 1.0;
            r.iomT = 1.0;
            r.d0 = __dadd_rn(1.0, kq);
            r.h0 = log1p(kq);
            r.yu = 0.0;
            r.ly_u = 0.0;
        } else {
            const double T = __dmul_rn(y_s[u], ymax[a]);
            const double omT = __dsub_rn(1.0, T);
            const double iomT = __ddiv_rn(1.0, omT);
            r.omT = omT;
            r.iomT = iomT;
            r.d0 = __dadd_rn(omT, kq);
            r.h0 = log1p(__dmul_rn(kq, iomT));
            r.yu = y_s[u];
            r.ly_u = ly_s[u];
        }
        r.rh0 = __drcp_rn(r.h0);
        s_rec[threadIdx.x] = r;
        const int64_t wa = sigma == 0 ? 0 : plan_W(P, F, c0, ri.r, ri.sat, a);
        const int64_t wb = plan_W(P, F, c0, ri.r, ri.sat, b);
        seg_work[g] = wb - wa + kUnit;
    }
    __syncthreads();
    // 16-byte words of the block's records, consecutive threads -> consecutive addresses
    // (the record stride is kRecStride(model): UBCM stores the first 4 of the 6 parts)
    const int4 *src = reinterpret_cast<const int4 *>(s_rec);
    const int words = kRecStride(model) / 16;
    int4 *dst = reinterpret_cast<int4 *>(rec + g0 * kRecStride(model));
    constexpr int kWords = (int)(sizeof(SegRec) / 16);
    for (int i = threadIdx.x; i < nb * words; i += blockDim.x) dst[i] = src[(i / words) * kWords + i % words];
}

// row-start flags for k_emit's segment -> row map: flag[row_seg[u]] = 1 for rows with segments
__global__ void k_row_starts(int64_t n, const int64_t *__restrict__ row_seg, int64_t *__restrict__ flag)
{
    const int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (u < n && row_seg[u + 1] > row_seg[u]) flag[row_seg[u]] = 1;
}

// directed (R16): excl[u] = candidate rank of row u's own node (inverse of the candidate order)
__global__ void k_rank_of(int64_t nc, const int32_t *__restrict__ cperm, int32_t *__restrict__ crank)
{
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r < nc) crank[cperm[r]] = (int32_t)r;
}
__global__ void k_excl(int64_t n, const int32_t *__restrict__ perm, const int32_t *__restrict__ crank,
                       int32_t *__restrict__ excl)
{
    const int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (u < n) excl[u] = crank[perm[u]];
}

// chunking: lane-chunk c starts at the first segment whose work prefix reaches c * target;
// its scratch slot holds floor(1.25 * est_draws) + 16 edges (edges <= draws)
__global__ void __launch_bounds__(256) k_chunks(int64_t n_seg, int64_t n_chunks, int64_t target,
                                                const int64_t *__restrict__ work_pre, int64_t *__restrict__ chunk_seg,
                                                int64_t *__restrict__ chunk_cap)
{
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= n_chunks) return;
    auto start = [&](int64_t cc) -> int64_t {
        if (cc >= n_chunks) return n_seg;
        const int64_t th = cc * target;
        int64_t lo = 0, hi = n_seg;  // smallest g with work_pre[g] >= th
        while (lo < hi) {
            const int64_t mid = lo + ((hi - lo) >> 1);
            if (work_pre[mid] >= th) hi = mid; else lo = mid + 1;
        }
        return lo;
    };
    const int64_t g0 = start(c), g1 = start(c + 1);
    chunk_seg[c] = g0;
    if (c == n_chunks - 1) chunk_seg[n_chunks] = n_seg;
    const int64_t w = work_pre[g1] - work_pre[g0];
    chunk_cap[c] = ((((w + (w >> 2)) >> kG) + 16) + 3) & ~int64_t(3);  // whole 32-byte sectors of edges
}

// the sampler's per-candidate gather record (Plan::cand)
__global__ void __launch_bounds__(256) k_pack_cand(int model, int64_t nc, const double *__restrict__ ckappa,
                                                   const int32_t *__restrict__ cperm, const double *__restrict__ cy,
                                                   const double *__restrict__ cly, double2 *__restrict__ cand)
{
    const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= nc) return;
    const double id = __hiloint2double(0, cperm[v]);
    if (model == FM_ECM) {
        cand[2 * v] = make_double2(ckappa[v], cy[v]);
        cand[2 * v + 1] = make_double2(cly[v], id);
    } else {
        cand[v] = make_double2(ckappa[v], id);
    }
}

// test hook (FM_DEBUG_SCRATCH_CAP): every lane-chunk gets the same tiny slot -> forces re-runs
__global__ void k_fill_caps(int64_t *chunk_cap, int64_t n_chunks, int64_t cap)
{
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c <= n_chunks) chunk_cap[c] = c * cap;
}

}  // namespace fm

namespace fm {
// test hook (FM_DEBUG_BAD_BOUND, fm_capi.cu): every segment record's initial bound numerator x0
// scaled by f (q0 = x0 / d0 shrinks below p of the first candidates: a contract violation)
__global__ void k_debug_scale_bound(unsigned char *rec, int64_t n_seg, int stride, double f)
{
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= n_seg) return;
    SegRec *r = reinterpret_cast<SegRec *>(rec + (size_t)g * stride);
    r->x0 = __dmul_rn(r->x0, f);
}
}  // namespace fm
