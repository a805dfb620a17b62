// fm_sort.cu -- a2: stable LSD radix sort of (uint64 key, int32 id) pairs, "one-sweep" style.
//
// The sort key is ~bits(kappa): kappa >= 0 doubles order like their bit patterns, so sorting
// the complement ascending gives kappa descending, and stability keeps ties in ascending id
// (R9; P:L133 step (i), Alg. 1 line 3).  8-bit digits; a digit that is the same in every
// key (seen in the up-front histograms, on the device) turns its pass into a plain copy.
//
// Launches: one memset of the look-back status, then ONE kernel per digit pass (the digit
// histograms of all positions come with the keys from k_validate_key).  A pass kernel takes tiles in
// ticket order (atomic counter), ranks its 2048 (4096 from 2^20 keys) keys stably (warp
// __match_any_sync ranks of all items first, then one counter update per item by the match's
// leader lane + cross-warp prefix in shared memory), publishes its per-digit counts and resolves its global offsets by decoupled
// look-back over the preceding tiles (64-bit status words: 2 flag bits + 62-bit count), stages
// the tile in digit order in shared memory and writes each digit run contiguously (coalesced).
// Each pass reads and writes the keys once (24 B per key).
#include <cstdlib>
#include <mutex>

#include "fm_internal.cuh"

namespace fm {
namespace {

constexpr int kThreads = 256;
#ifndef FM_SORT_ITEMS_BIG
#define FM_SORT_ITEMS_BIG 16
#endif
#ifndef FM_SORT_BIG_MIN
#define FM_SORT_BIG_MIN (1 << 20)
#endif
// keys per thread: 8 (tiles of 2048 keys) below FM_SORT_BIG_MIN keys, else 16 (tiles of 4096: half
// the tiles, look-back chains and status traffic, twice the loads in flight per thread)
constexpr int kItemsSmall = 8, kItemsBig = FM_SORT_ITEMS_BIG;
#ifndef FM_SORT_LB
#define FM_SORT_LB 8
#endif
constexpr int kLB = FM_SORT_LB;  // predecessor tiles read per look-back step
constexpr int kRadix = 256;
constexpr int kPasses = 8;
constexpr uint64_t kFlagAgg = 1ull << 62, kFlagInc = 2ull << 62, kValMask = (1ull << 62) - 1;

__device__ __forceinline__ uint64_t ld_volatile_u64(const uint64_t *p)
{
    uint64_t v;
    asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(p));
    return v;
}

template <int kI>
__device__ __noinline__ void copy_tile(const uint64_t *__restrict__ kin, const int32_t *__restrict__ vin,
                                       uint64_t *__restrict__ kout, int32_t *__restrict__ vout, int64_t n)
{
    const int64_t t0 = (int64_t)blockIdx.x * (kThreads * kI);
    for (int r = 0; r < kI; r++) {
        const int64_t i = t0 + r * kThreads + threadIdx.x;
        if (i < n) {
            kout[i] = __ldcs(kin + i);
            vout[i] = __ldcs(vin + i);
        }
    }
}

// dynamic shared memory of a pass block: the tile in digit order (keys, ids), the per-warp digit
// counters, the per-digit global base and tile-local start
template <int kI>
constexpr size_t pass_smem_bytes()
{
    return (size_t)kThreads * kI * (sizeof(uint64_t) + sizeof(int32_t)) + sizeof(int) * (kThreads / 32) * kRadix +
           sizeof(int64_t) * kRadix + sizeof(int) * kRadix;
}

#ifndef FM_SORT_BIG_BLOCKS
#define FM_SORT_BIG_BLOCKS 2
#endif
template <int kI>
__global__ void __launch_bounds__(kThreads, kI > 8 ? FM_SORT_BIG_BLOCKS : 4)
    k_pass(const uint64_t *__restrict__ kin, const int32_t *__restrict__ vin, uint64_t *__restrict__ kout,
           int32_t *__restrict__ vout, int64_t n, int shift, const unsigned int *__restrict__ hist, uint64_t *status,
           unsigned int *tile_counter)
{
    constexpr int kTile = kThreads * kI;
    extern __shared__ __align__(16) unsigned char s_raw[];
    uint64_t *s_key = reinterpret_cast<uint64_t *>(s_raw);             // the tile in digit order (stable): coalesced global writes
    int64_t *s_base = reinterpret_cast<int64_t *>(s_key + kTile);      // global position of the tile's first key of each digit
    int32_t *s_val = reinterpret_cast<int32_t *>(s_base + kRadix);
    int(*wcnt)[kRadix] = reinterpret_cast<int(*)[kRadix]>(s_val + kTile);
    int *s_lstart = reinterpret_cast<int *>(wcnt + kThreads / 32);      // tile-local position of the tile's first key of each digit
    __shared__ unsigned int s_wsum[kThreads / 32];
    __shared__ int s_wtot[kThreads / 32];
    __shared__ unsigned int s_tile;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    // a digit no key varies in (one bin holds all n keys, known from the up-front histograms without
    // a host round trip): the pass is a stable identity -- a plain coalesced copy of the tile, no
    // ranking, no look-back (e.g. the sign / high exponent byte when every kappa < 2)
    if (__syncthreads_or(hist[threadIdx.x] == (unsigned int)n)) {
        copy_tile<kI>(kin, vin, kout, vout, n);  // (not inlined: the ranking path keeps its registers)
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
    uint64_t key[kI];
    int32_t val[kI];
    int loc[kI];
    // all of the thread's loads issued before the first rank (the warp syncs below would
    // otherwise serialise one load latency per item)
#pragma unroll
    for (int r = 0; r < kI; r++) {
        const int64_t i = wbase + r * 32 + lane;  // warp-contiguous, in input order
        const bool ok = i < n;
        key[r] = ok ? __ldcs(kin + i) : 0;
        val[r] = ok ? __ldcs(vin + i) : 0;
    }
    // stable rank of each key among the warp's keys of the same digit.  Phase A: the peer masks of
    // all items (independent warp matches, no shared memory); loc packs rank among the peers of the
    // same item | leader lane << 8 | peer count << 16.  Phase B: per item, the leader bumps the
    // warp's digit counter and broadcasts its old value (one LDS + STS by one lane, one shuffle).
#pragma unroll
    for (int r = 0; r < kI; r++) {
        const bool ok = wbase + r * 32 + lane < n;
        const int d = ok ? (int)((key[r] >> shift) & 0xFF) : kRadix;
        // the lanes holding the same digit: nine ballots (one per digit bit and one for validity)
        // instead of __match_any_sync -- MATCH.ANY measured as the pass's bottleneck on the B200
        // (45 % of its stall samples sat on the 16 matches' results)
        uint32_t peers = 0xffffffffu;
#ifdef FM_SORT_MATCH
        peers = __match_any_sync(0xffffffffu, d);
#else
#pragma unroll
        for (int b = 0; b < 9; b++) {
            const bool bit = (d >> b) & 1;
            const uint32_t bal = __ballot_sync(0xffffffffu, bit);
            peers &= bit ? bal : ~bal;
        }
#endif
        loc[r] = __popc(peers & lt) | ((__ffs(peers) - 1) << 8) | (__popc(peers) << 16);
    }
#pragma unroll
    for (int r = 0; r < kI; r++) {
        const bool ok = wbase + r * 32 + lane < n;
        const int d = (int)((key[r] >> shift) & 0xFF);
        const int leader = (loc[r] >> 8) & 0xFF;
        int base = 0;
        if (ok && lane == leader) {
            base = wcnt[wid][d];
            wcnt[wid][d] = base + (loc[r] >> 16);
        }
        base = __shfl_sync(0xffffffffu, base, leader);
        loc[r] = ok ? base + (loc[r] & 0xFF) : -1;
        __syncwarp();
    }
    __syncthreads();
    // thread d: tile-local prefix over warps and the tile's count of digit d; the count is published
    // and the first look-back loads are issued BEFORE the tile is staged in shared memory, so the
    // predecessors' status words travel while the block scans and stages (their latency was exposed)
    int acc = 0;
    const int d_own = threadIdx.x;
    uint64_t *const my = status + tile * kRadix + d_own;
    uint64_t v[kLB];
    {
        for (int w = 0; w < kThreads / 32; w++) {
            const int c = wcnt[w][d_own];
            wcnt[w][d_own] = acc;
            acc += c;
        }
        if (tile == 0) {
            *(volatile uint64_t *)my = kFlagInc | (uint64_t)acc;
        } else {
            *(volatile uint64_t *)my = kFlagAgg | (uint64_t)acc;
#pragma unroll
            for (int k = 0; k < kLB; k++)
                v[k] = tile - 1 - k >= 0 ? ld_volatile_u64(status + (tile - 1 - k) * kRadix + d_own) : kFlagInc;
        }
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
    for (int r = 0; r < kI; r++) {
        if (loc[r] >= 0) {
            const int d = (int)((key[r] >> shift) & 0xFF);
            const int p = s_lstart[d] + wcnt[wid][d] + loc[r];
            s_key[p] = key[r];
            s_val[p] = val[r];
        }
    }
    // finish the look-back: kLB predecessor tiles at a time (independent loads in flight)
    {
        uint64_t prefix = 0;
        if (tile > 0) {
            for (int64_t j = tile - 1;; j -= kLB) {
                bool done = false;
#pragma unroll
                for (int k = 0; k < kLB; k++) {
                    if (done) break;
                    while ((v[k] & ~kValMask) == 0) v[k] = ld_volatile_u64(status + (j - k) * kRadix + d_own);
                    prefix += v[k] & kValMask;
                    done = (v[k] & ~kValMask) == kFlagInc;
                }
                if (done) break;
#pragma unroll
                for (int k = 0; k < kLB; k++)
                    v[k] = j - kLB - k >= 0 ? ld_volatile_u64(status + (j - kLB - k) * kRadix + d_own) : kFlagInc;
            }
            *(volatile uint64_t *)my = kFlagInc | (prefix + (uint64_t)acc);
        }
        s_base[d_own] = (int64_t)(dbase + prefix);
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kI; r++) {
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

template <int kI>
cudaError_t launch_pass(const uint64_t *ki, const int32_t *vi, uint64_t *ko, int32_t *vo, int64_t n, int shift,
                        const unsigned int *hist, uint64_t *status, unsigned int *tiles, cudaStream_t st)
{
    static std::once_flag once[kMaxDevices];
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 0 || dev >= kMaxDevices) return cudaErrorInvalidDevice;
    std::call_once(once[dev], [] {
        cudaFuncSetAttribute(k_pass<kI>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pass_smem_bytes<kI>());
    });
    const int64_t nt = (n + kThreads * kI - 1) / (kThreads * kI);
    k_pass<kI><<<(unsigned)nt, kThreads, pass_smem_bytes<kI>(), st>>>(ki, vi, ko, vo, n, shift, hist, status, tiles);
    return cudaGetLastError();
}

}  // namespace

size_t radix_tmp_bytes(int64_t n)
{
    const int64_t nt = (n + kThreads * kItemsSmall - 1) / (kThreads * kItemsSmall);  // (the smaller tile: an upper bound)
    return sizeof(uint64_t) * (size_t)(kPasses * nt * kRadix) + sizeof(unsigned int) * kPasses + 512;
}

cudaError_t radix_sort_u64_i32(uint64_t *keys_a, uint64_t *keys_b, int32_t *vals_a, int32_t *vals_b, int64_t n,
                               uint64_t vary_bits, const unsigned int *hist, uint64_t **key_out, int32_t **val_out,
                               void *tmp, size_t tmp_bytes, cudaStream_t st)
{
    // (FM_SORT_BIG_MIN in the environment: the key count from which the 4096-key tiles are used; tests)
    const char *bm = getenv("FM_SORT_BIG_MIN");
    const bool big = n >= (bm && *bm ? strtoll(bm, nullptr, 10) : (long long)FM_SORT_BIG_MIN);
    const int64_t tile = kThreads * (big ? kItemsBig : kItemsSmall);
    const int64_t nt = (n + tile - 1) / tile;
    if (tmp_bytes < radix_tmp_bytes(n)) return cudaErrorInvalidValue;
    uint64_t *status = (uint64_t *)tmp;
    const int64_t nt_max = (n + kThreads * kItemsSmall - 1) / (kThreads * kItemsSmall);
    unsigned int *tiles = (unsigned int *)(status + kPasses * nt_max * kRadix);
    cudaError_t e = cudaMemsetAsync(tmp, 0, radix_tmp_bytes(n) - 512, st);
    if (e != cudaSuccess) return e;
    uint64_t *ki = keys_a, *ko = keys_b;
    int32_t *vi = vals_a, *vo = vals_b;
    for (int p = 0; p < kPasses; p++) {
        const int shift = 8 * p;
        if (((vary_bits >> shift) & 0xFFull) == 0) continue;
        count_launch();
        uint64_t *stp = status + (int64_t)p * nt * kRadix;
        e = big ? launch_pass<kItemsBig>(ki, vi, ko, vo, n, shift, hist + p * kRadix, stp, tiles + p, st)
                : launch_pass<kItemsSmall>(ki, vi, ko, vo, n, shift, hist + p * kRadix, stp, tiles + p, st);
        if (e != cudaSuccess) return e;
        uint64_t *tk = ki; ki = ko; ko = tk;
        int32_t *tv = vi; vi = vo; vo = tv;
    }
    *key_out = ki;
    *val_out = vi;
    return cudaGetLastError();
}

}  // namespace fm
