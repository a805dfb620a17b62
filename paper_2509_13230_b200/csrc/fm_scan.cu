// fm_scan.cu -- device scans used by the planner and the output writer (a4, a6).
// Reduce-then-scan in three launches: per-tile reduction, one-block scan of tile partials,
// per-tile scan seeded by its partial.  Tiles are 256 threads x 8 contiguous items.
#include "fm_internal.cuh"

namespace fm {
namespace {

constexpr int kThreads = 256;
constexpr int kItems = 8;
constexpr int kTile = kThreads * kItems;

struct SumU64 {
    using T = uint64_t;
    __device__ static T id() { return 0; }
    __device__ static T op(T a, T b) { return a + b; }
};
struct MaxF64 {
    using T = double;
    __device__ static T id() { return 0.0; }  // inputs are >= 0 (y in [0,1))
    __device__ static T op(T a, T b) { return fmax(a, b); }
};

// logical index i -> physical index (reverse scans walk the array from the end)
template <bool kRev>
__device__ __forceinline__ int64_t phys(int64_t i, int64_t n) { return kRev ? n - 1 - i : i; }

template <typename Op, int kT = kThreads>
__device__ __forceinline__ typename Op::T block_exclusive(typename Op::T v, typename Op::T *total)
{
    using T = typename Op::T;
    __shared__ T warp_tot[kT / 32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    T inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc = Op::op(t, inc);
    }
    if (lane == 31) warp_tot[wid] = inc;
    __syncthreads();
    T wpre = Op::id(), all = Op::id();
#pragma unroll
    for (int w = 0; w < kT / 32; w++) {
        if (w < wid) wpre = Op::op(wpre, warp_tot[w]);
        all = Op::op(all, warp_tot[w]);
    }
    T exc = __shfl_up_sync(0xffffffffu, inc, 1);
    if (lane == 0) exc = Op::id();
    __syncthreads();
    *total = all;
    return Op::op(wpre, exc);
}

template <typename Op, bool kRev>
__global__ void __launch_bounds__(kThreads) k_tile_reduce(const typename Op::T *in, int64_t n,
                                                          typename Op::T *partial)
{
    using T = typename Op::T;
    const int64_t base = (int64_t)blockIdx.x * kTile + (int64_t)threadIdx.x * kItems;
    T acc = Op::id();
#pragma unroll
    for (int k = 0; k < kItems; k++) {
        const int64_t i = base + k;
        if (i < n) acc = Op::op(acc, in[phys<kRev>(i, n)]);
    }
    T tot;
    block_exclusive<Op>(acc, &tot);
    if (threadIdx.x == 0) partial[blockIdx.x] = tot;
}

// one block: exclusive scan of partial[0..nb) in place
template <typename Op>
__global__ void __launch_bounds__(kThreads) k_partials(typename Op::T *partial, int64_t nb)
{
    using T = typename Op::T;
    T carry = Op::id();
    for (int64_t b0 = 0; b0 < nb; b0 += kTile) {
        T v[kItems];
        T acc = Op::id();
#pragma unroll
        for (int k = 0; k < kItems; k++) {
            const int64_t i = b0 + (int64_t)threadIdx.x * kItems + k;
            v[k] = i < nb ? partial[i] : Op::id();
            acc = Op::op(acc, v[k]);
        }
        T tot;
        T pre = Op::op(carry, block_exclusive<Op>(acc, &tot));
#pragma unroll
        for (int k = 0; k < kItems; k++) {
            const int64_t i = b0 + (int64_t)threadIdx.x * kItems + k;
            if (i < nb) partial[i] = pre;
            pre = Op::op(pre, v[k]);
        }
        carry = Op::op(carry, tot);
        __syncthreads();
    }
}

// kInclusive=false: out[i] = op(in[0..i)), out[n] = total.  true: out[i] = op(in[0..i]).
template <typename Op, bool kRev, bool kInclusive>
__global__ void __launch_bounds__(kThreads) k_tile_scan(const typename Op::T *in, typename Op::T *out, int64_t n,
                                                        const typename Op::T *partial, int64_t nb)
{
    using T = typename Op::T;
    const int64_t base = (int64_t)blockIdx.x * kTile + (int64_t)threadIdx.x * kItems;
    T v[kItems];
    T acc = Op::id();
#pragma unroll
    for (int k = 0; k < kItems; k++) {
        const int64_t i = base + k;
        v[k] = i < n ? in[phys<kRev>(i, n)] : Op::id();
        acc = Op::op(acc, v[k]);
    }
    T tot;
    T pre = Op::op(partial[blockIdx.x], block_exclusive<Op>(acc, &tot));
#pragma unroll
    for (int k = 0; k < kItems; k++) {
        const int64_t i = base + k;
        if (kInclusive) pre = Op::op(pre, v[k]);
        if (i < n) out[phys<kRev>(i, n)] = pre;
        if (!kInclusive) pre = Op::op(pre, v[k]);
    }
    if (!kInclusive && blockIdx.x == nb - 1 && threadIdx.x == kThreads - 1) out[n] = pre;
}

template <typename Op, bool kRev, bool kInclusive>
cudaError_t run_scan(const typename Op::T *in, typename Op::T *out, int64_t n, void *tmp, size_t tmp_bytes,
                     cudaStream_t st)
{
    using T = typename Op::T;
    if (n <= 0) return cudaSuccess;
    const int64_t nb = (n + kTile - 1) / kTile;
    if (tmp_bytes < sizeof(T) * (size_t)nb) return cudaErrorInvalidValue;
    T *partial = (T *)tmp;
    count_launch();
    k_tile_reduce<Op, kRev><<<(unsigned)nb, kThreads, 0, st>>>(in, n, partial);
    count_launch();
    k_partials<Op><<<1, kThreads, 0, st>>>(partial, nb);
    count_launch();
    k_tile_scan<Op, kRev, kInclusive><<<(unsigned)nb, kThreads, 0, st>>>(in, out, n, partial, nb);
    return cudaGetLastError();
}

__global__ void k_set_f64(double *p, double v) { *p = v; }

// Single-pass exclusive sum (decoupled look-back): tiles in ticket order publish their
// aggregate, then their inclusive prefix (64-bit status word: 2 flag bits + 62-bit value; all
// sums here are non-negative and < 2^62).  status[] and the ticket counter start at zero.
constexpr uint64_t kFlagAgg = 1ull << 62, kFlagInc = 2ull << 62, kValMask = (1ull << 62) - 1;

// kT = 128 with <= 32 registers (kMinB = 16) is the small-footprint variant: one such block fits
// next to three resident sampler blocks per SM (the pipelined sample groups).
template <int kT, int kMinB, int kIt>
__global__ void __launch_bounds__(kT, kMinB) k_scan_lb(const uint64_t *in, uint64_t *out, int64_t n,
                                                       uint64_t *status, unsigned int *ticket)
{
    constexpr int kTile = kT * kIt;
    __shared__ unsigned int s_tile;
    __shared__ uint64_t s_prefix;
    if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1u);
    __syncthreads();
    const int64_t tile = s_tile;
    const int64_t base = tile * kTile + (int64_t)threadIdx.x * kIt;
    uint64_t v[kIt];
    uint64_t acc = 0;
    // a thread's kIt items are contiguous (64 or 128 bytes): 16-byte vector loads when the 8 are in range and
    // the array is 16-byte aligned (every caller's is)
    const bool vec = base + kIt <= n && ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) & 15) == 0;
    if (vec) {
        const ulonglong2 *q = reinterpret_cast<const ulonglong2 *>(in + base);
#pragma unroll
        for (int k = 0; k < kIt / 2; k++) {
            const ulonglong2 w = q[k];
            v[2 * k] = w.x;
            v[2 * k + 1] = w.y;
        }
    } else {
#pragma unroll
        for (int k = 0; k < kIt; k++) {
            const int64_t i = base + k;
            v[k] = i < n ? in[i] : 0;
        }
    }
#pragma unroll
    for (int k = 0; k < kIt; k++) acc += v[k];
    uint64_t tot;
    const uint64_t exc = block_exclusive<SumU64, kT>(acc, &tot);
    if (threadIdx.x < 32) {  // warp 0: publish, then look back 32 predecessors at a time
        const int lane = threadIdx.x;
        uint64_t prefix = 0;
        if (tile == 0) {
            if (lane == 0) *(volatile uint64_t *)(status) = kFlagInc | tot;
        } else {
            if (lane == 0) *(volatile uint64_t *)(status + tile) = kFlagAgg | tot;
            for (int64_t j_end = tile;; j_end -= 32) {
                const int64_t j = j_end - 1 - lane;  // lane 0 = nearest predecessor
                uint64_t v = kFlagInc;               // before tile 0: an inclusive prefix of 0
                if (j >= 0) {
                    do {
                        asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(status + j));
                    } while ((v & ~kValMask) == 0);
                }
                const uint32_t inc = __ballot_sync(0xffffffffu, (v & ~kValMask) == kFlagInc);
                const int first = inc ? __ffs(inc) - 1 : 32;
                uint64_t c = lane <= first ? (v & kValMask) : 0;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
                prefix += c;
                if (inc) break;
            }
            if (lane == 0) *(volatile uint64_t *)(status + tile) = kFlagInc | (prefix + tot);
        }
        if (lane == 0) s_prefix = prefix;
    }
    __syncthreads();
    uint64_t pre = s_prefix + exc;
    if (vec) {
        ulonglong2 *q = reinterpret_cast<ulonglong2 *>(out + base);
#pragma unroll
        for (int k = 0; k < kIt / 2; k++) {
            const uint64_t a0 = pre;
            pre += v[2 * k];
            q[k] = make_ulonglong2(a0, pre);
            pre += v[2 * k + 1];
        }
    } else {
#pragma unroll
        for (int k = 0; k < kIt; k++) {
            const int64_t i = base + k;
            if (i < n) out[i] = pre;
            pre += v[k];
        }
    }
    if (tile == (n - 1) / kTile && threadIdx.x == ((n - 1) % kTile) / kIt) out[n] = pre;  // total
}

#ifndef FM_SCAN_BIG_MIN
#define FM_SCAN_BIG_MIN (1 << 20)
#endif
cudaError_t run_scan_lb(const uint64_t *in, uint64_t *out, int64_t n, void *tmp, size_t tmp_bytes, cudaStream_t st,
                        bool small = false, bool zeroed = false)
{
    // long arrays: 4096-item tiles (16 per thread) -- the look-back chain is per tile, and a block's
    // threads wait at its barrier for it (ncu at n = 1e7 with 2048-item tiles: 50 barrier-stall
    // samples per issued instruction, issue active 11 %)
    const bool big = !small && n >= FM_SCAN_BIG_MIN;
    const int64_t tile = small ? 128 * kItems : big ? kThreads * 16 : kTile;
    const int64_t nb = (n + tile - 1) / tile;
    const size_t need = sizeof(uint64_t) * (size_t)(nb + 1);
    if (tmp_bytes < need) return cudaErrorInvalidValue;
    // (zeroed: the caller cleared tmp -- the pipelined sample groups clear every group's words up
    // front: a memset between the groups' kernels would wait for the resident sampler)
    cudaError_t e = zeroed ? cudaSuccess : cudaMemsetAsync(tmp, 0, need, st);
    if (e != cudaSuccess) return e;
    count_launch();
    uint64_t *status = (uint64_t *)tmp;
    unsigned int *ticket = (unsigned int *)(status + nb);
    if (small)
        k_scan_lb<128, 16, kItems><<<(unsigned)nb, 128, 0, st>>>(in, out, n, status, ticket);
    else if (big)
        k_scan_lb<kThreads, 1, 16><<<(unsigned)nb, kThreads, 0, st>>>(in, out, n, status, ticket);
    else
        k_scan_lb<kThreads, 1, kItems><<<(unsigned)nb, kThreads, 0, st>>>(in, out, n, status, ticket);
    return cudaGetLastError();
}

}  // namespace

// (sized for the small-footprint variant's 1024-item tiles)
size_t scan_tmp_bytes(int64_t n) { return sizeof(int64_t) * (size_t)((n + 1023) / 1024 + 2); }

// non-negative sums only (all callers): one launch + one memset
cudaError_t scan_exclusive_i64(const int64_t *in, int64_t *out, int64_t n, void *tmp, size_t tmp_bytes,
                               cudaStream_t st, bool small, bool zeroed)
{
    if (n == 0) return cudaMemsetAsync(out, 0, sizeof(int64_t), st);
    return run_scan_lb((const uint64_t *)in, (uint64_t *)out, n, tmp, tmp_bytes, st, small, zeroed);
}

cudaError_t scan_exclusive_u64(const uint64_t *in, uint64_t *out, int64_t n, void *tmp, size_t tmp_bytes,
                               cudaStream_t st)
{
    if (n == 0) return cudaMemsetAsync(out, 0, sizeof(uint64_t), st);
    return run_scan_lb(in, out, n, tmp, tmp_bytes, st);
}

cudaError_t suffix_max_f64(const double *in, double *out, int64_t n, void *tmp, size_t tmp_bytes,
                           cudaStream_t st)
{
    count_launch();
    k_set_f64<<<1, 1, 0, st>>>(out + n, 0.0);
    return run_scan<MaxF64, true, true>(in, out, n, tmp, tmp_bytes, st);
}

}  // namespace fm
