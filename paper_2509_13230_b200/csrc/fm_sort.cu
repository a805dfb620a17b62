// fm_sort.cu -- a2: stable LSD radix sort of (uint64 key, int32 id) pairs, "one-sweep" style.
//
// The sort key is ~bits(kappa): kappa >= 0 doubles order like their bit patterns, so sorting
// the complement ascending gives kappa descending, and stability keeps ties in ascending id
// (R9; P:L133 step (i), Alg. 1 line 3).  8-bit digits; a digit that is the same in every
// key (seen in the up-front histograms, on the device) turns its pass into a plain copy.
//
// Launches: one memset of the look-back status, then ONE kernel per digit pass (the digit
// histograms of all positions come with the keys from k_validate_key).  A pass kernel takes tiles in ticket order (atomic counter),
// ranks its 2048 keys stably (warp __match_any_sync ranks + cross-warp prefix in shared
// memory), publishes its per-digit counts and resolves its global offsets by decoupled
// look-back over the preceding tiles (64-bit status words: 2 flag bits + 62-bit count), stages
// the tile in digit order in shared memory and writes each digit run contiguously (coalesced).
// Each pass reads and writes the keys once (24 B per key).
#include "fm_internal.cuh"

namespace fm {
namespace {

constexpr int kThreads = 256;
#ifndef FM_SORT_ITEMS
#define FM_SORT_ITEMS 8
#endif
constexpr int kItems = FM_SORT_ITEMS;
#ifndef FM_SORT_LB
#define FM_SORT_LB 8
#endif
constexpr int kLB = FM_SORT_LB;  // predecessor tiles read per look-back step
constexpr int kTile = kThreads * kItems;  // 2048 keys per tile, 256 per warp
constexpr int kRadix = 256;
constexpr int kPasses = 8;
constexpr uint64_t kFlagAgg = 1ull << 62, kFlagInc = 2ull << 62, kValMask = (1ull << 62) - 1;

__device__ __forceinline__ uint64_t ld_volatile_u64(const uint64_t *p)
{
    uint64_t v;
    asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(p));
    return v;
}

__device__ __noinline__ void copy_tile(const uint64_t *__restrict__ kin, const int32_t *__restrict__ vin,
                                       uint64_t *__restrict__ kout, int32_t *__restrict__ vout, int64_t n)
{
    const int64_t t0 = (int64_t)blockIdx.x * kTile;
    for (int r = 0; r < kItems; r++) {
        const int64_t i = t0 + r * kThreads + threadIdx.x;
        if (i < n) {
            kout[i] = __ldcs(kin + i);
            vout[i] = __ldcs(vin + i);
        }
    }
}

__global__ void __launch_bounds__(kThreads, 4) k_pass(const uint64_t *__restrict__ kin, const int32_t *__restrict__ vin,
                                                   uint64_t *__restrict__ kout, int32_t *__restrict__ vout, int64_t n,
                                                   int shift, const unsigned int *__restrict__ hist,
                                                   uint64_t *status, unsigned int *tile_counter)
{
    __shared__ int wcnt[kThreads / 32][kRadix];
    __shared__ int64_t s_base[kRadix];   // global position of the tile's first key of each digit
    __shared__ int s_lstart[kRadix];     // tile-local position of the tile's first key of each digit
    __shared__ unsigned int s_wsum[kThreads / 32];
    __shared__ int s_wtot[kThreads / 32];
    __shared__ unsigned int s_tile;
    __shared__ uint64_t s_key[kTile];    // the tile in digit order (stable): coalesced global writes
    __shared__ int32_t s_val[kTile];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    // a digit no key varies in (one bin holds all n keys, known from the up-front histograms without
    // a host round trip): the pass is a stable identity -- a plain coalesced copy of the tile, no
    // ranking, no look-back (e.g. the sign / high exponent byte when every kappa < 2)
    if (__syncthreads_or(hist[threadIdx.x] == (unsigned int)n)) {
        copy_tile(kin, vin, kout, vout, n);  // (not inlined: the ranking path keeps its registers)
        return;
    }
    unsigned int hv = hist[threadIdx.x], inc = hv;
    if (threadIdx.x == 0) s_tile = atomicAdd(tile_counter, 1u);
    for (int w = 0; w < kThreads / 32; w++) wcnt[w][threadIdx.x] = 0;
    // exclusive scan of the pass's global digit counts: the base of each digit
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned int t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
    }
    if (lane == 31) s_wsum[wid] = inc;
    __syncthreads();
    uint64_t dbase = inc - hv;
    for (int w = 0; w < wid; w++) dbase += s_wsum[w];
    const int64_t tile = s_tile;
    const uint32_t lt = (1u << lane) - 1u;
    const int64_t wbase = tile * kTile + (int64_t)wid * (kTile / (kThreads / 32));
    const int nvalid = (int)min((int64_t)kTile, n - tile * kTile);
    uint64_t key[kItems];
    int32_t val[kItems];
    int dig[kItems], loc[kItems];
    // all of the thread's loads issued before the first rank (the warp syncs below would
    // otherwise serialise one load latency per item)
#pragma unroll
    for (int r = 0; r < kItems; r++) {
        const int64_t i = wbase + r * 32 + lane;  // warp-contiguous, in input order
        const bool ok = i < n;
        key[r] = ok ? __ldcs(kin + i) : 0;
        val[r] = ok ? __ldcs(vin + i) : 0;
    }
#pragma unroll
    for (int r = 0; r < kItems; r++) {
        const bool ok = wbase + r * 32 + lane < n;
        dig[r] = ok ? (int)((key[r] >> shift) & 0xFF) : kRadix;
        const uint32_t peers = __match_any_sync(0xffffffffu, dig[r]);
        const int rank = __popc(peers & lt);
        const int leader = __ffs(peers) - 1;
        loc[r] = ok ? wcnt[wid][dig[r]] + rank : 0;
        __syncwarp();
        if (ok && lane == leader) wcnt[wid][dig[r]] += __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    // thread d: tile-local prefix over warps, the tile's count of digit d, and its global base
    int acc = 0;
    {
        const int d = threadIdx.x;
        for (int w = 0; w < kThreads / 32; w++) {
            const int c = wcnt[w][d];
            wcnt[w][d] = acc;
            acc += c;
        }
        const uint64_t cnt = (uint64_t)acc;
        uint64_t *my = status + tile * kRadix + d;
        uint64_t prefix = 0;
        if (tile == 0) {
            *(volatile uint64_t *)my = kFlagInc | cnt;
        } else {
            *(volatile uint64_t *)my = kFlagAgg | cnt;
            // look back kLB predecessor tiles at a time (independent loads in flight)
            for (int64_t j = tile - 1; j >= 0; j -= kLB) {
                uint64_t v[kLB];
#pragma unroll
                for (int k = 0; k < kLB; k++) v[k] = j - k >= 0 ? ld_volatile_u64(status + (j - k) * kRadix + d) : kFlagInc;
                bool done = false;
#pragma unroll
                for (int k = 0; k < kLB; k++) {
                    if (done) break;
                    while ((v[k] & ~kValMask) == 0) v[k] = ld_volatile_u64(status + (j - k) * kRadix + d);
                    prefix += v[k] & kValMask;
                    done = (v[k] & ~kValMask) == kFlagInc;
                }
                if (done) break;
            }
            *(volatile uint64_t *)my = kFlagInc | (prefix + cnt);
        }
        s_base[d] = (int64_t)(dbase + prefix);
    }
    // tile-local exclusive scan of the digit counts (block-wide over the 256 digits)
    {
        int inc2 = acc;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, inc2, o);
            if (lane >= o) inc2 += t;
        }
        if (lane == 31) s_wtot[wid] = inc2;
        __syncthreads();
        int off = inc2 - acc;
        for (int w = 0; w < wid; w++) off += s_wtot[w];
        s_lstart[threadIdx.x] = off;
    }
    __syncthreads();
    // stage the tile in digit order, then write it out contiguously per digit run
#pragma unroll
    for (int r = 0; r < kItems; r++) {
        if (dig[r] < kRadix) {
            const int p = s_lstart[dig[r]] + wcnt[wid][dig[r]] + loc[r];
            s_key[p] = key[r];
            s_val[p] = val[r];
        }
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kItems; r++) {
        const int p = r * kThreads + threadIdx.x;
        if (p < nvalid) {
            const uint64_t k = s_key[p];
            const int d = (int)((k >> shift) & 0xFF);
            const int64_t dst = s_base[d] + (p - s_lstart[d]);
            kout[dst] = k;
            vout[dst] = s_val[p];
        }
    }
}

}  // namespace

size_t radix_tmp_bytes(int64_t n)
{
    const int64_t nt = (n + kTile - 1) / kTile;
    return sizeof(uint64_t) * (size_t)(kPasses * nt * kRadix) + sizeof(unsigned int) * kPasses + 512;
}

cudaError_t radix_sort_u64_i32(uint64_t *keys_a, uint64_t *keys_b, int32_t *vals_a, int32_t *vals_b, int64_t n,
                               uint64_t vary_bits, const unsigned int *hist, uint64_t **key_out, int32_t **val_out,
                               void *tmp, size_t tmp_bytes, cudaStream_t st)
{
    const int64_t nt = (n + kTile - 1) / kTile;
    if (tmp_bytes < radix_tmp_bytes(n)) return cudaErrorInvalidValue;
    uint64_t *status = (uint64_t *)tmp;
    unsigned int *tiles = (unsigned int *)(status + kPasses * nt * kRadix);
    cudaError_t e = cudaMemsetAsync(tmp, 0, radix_tmp_bytes(n) - 512, st);
    if (e != cudaSuccess) return e;
    uint64_t *ki = keys_a, *ko = keys_b;
    int32_t *vi = vals_a, *vo = vals_b;
    for (int p = 0; p < kPasses; p++) {
        const int shift = 8 * p;
        if (((vary_bits >> shift) & 0xFFull) == 0) continue;
        count_launch();
        k_pass<<<(unsigned)nt, kThreads, 0, st>>>(ki, vi, ko, vo, n, shift, hist + p * kRadix,
                                                  status + (int64_t)p * nt * kRadix, tiles + p);
        uint64_t *tk = ki; ki = ko; ko = tk;
        int32_t *tv = vi; vi = vo; vo = tv;
    }
    *key_out = ki;
    *val_out = vi;
    return cudaGetLastError();
}

}  // namespace fm
