// fm_sort.cu -- a2: stable LSD radix sort of (uint64 key, int32 id) pairs.
//
// The sort key is ~bits(kappa): kappa >= 0 doubles order like their bit patterns, so sorting
// the complement ascending gives kappa descending, and stability keeps ties in ascending id
// (R9; P:L133 step (i), Alg. 1 line 3).  8-bit digits; a digit none of whose bits
// varies across the keys is skipped.  Per digit: tile histogram -> exclusive scan (digit-major,
// so the scan yields each tile's global base per digit) -> stable scatter (warp-level
// __match_any_sync ranks, cross-warp prefix in shared memory).
#include "fm_internal.cuh"

namespace fm {
namespace {

constexpr int kThreads = 256;
constexpr int kItems = 8;
constexpr int kTile = kThreads * kItems;  // 2048 keys per tile, 256 per warp
constexpr int kRadix = 256;

__global__ void __launch_bounds__(kThreads) k_hist(const uint64_t *keys, int64_t n, int shift, int64_t nt,
                                                   int64_t *counts)
{
    __shared__ int h[kRadix];
    h[threadIdx.x] = 0;
    __syncthreads();
    const int64_t base = (int64_t)blockIdx.x * kTile;
#pragma unroll
    for (int k = 0; k < kItems; k++) {
        const int64_t i = base + (int64_t)k * kThreads + threadIdx.x;
        if (i < n) atomicAdd(&h[(keys[i] >> shift) & 0xFF], 1);
    }
    __syncthreads();
    counts[(int64_t)threadIdx.x * nt + blockIdx.x] = h[threadIdx.x];
}

__global__ void __launch_bounds__(kThreads) k_scatter(const uint64_t *__restrict__ kin, const int32_t *__restrict__ vin,
                                                      uint64_t *__restrict__ kout, int32_t *__restrict__ vout,
                                                      int64_t n, int shift, int64_t nt,
                                                      const int64_t *__restrict__ offsets)
{
    __shared__ int wcnt[kThreads / 32][kRadix];
    __shared__ int64_t tbase[kRadix];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int w = 0; w < kThreads / 32; w++) wcnt[w][threadIdx.x] = 0;
    tbase[threadIdx.x] = offsets[(int64_t)threadIdx.x * nt + blockIdx.x];
    __syncthreads();
    const uint32_t lt = (1u << lane) - 1u;
    const int64_t wbase = (int64_t)blockIdx.x * kTile + (int64_t)wid * (kTile / (kThreads / 32));
    uint64_t key[kItems];
    int32_t val[kItems];
    int dig[kItems], loc[kItems];
#pragma unroll
    for (int r = 0; r < kItems; r++) {
        const int64_t i = wbase + r * 32 + lane;  // warp-contiguous, in input order
        const bool ok = i < n;
        key[r] = ok ? kin[i] : 0;
        val[r] = ok ? vin[i] : 0;
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
    {  // per digit: exclusive prefix over warps (tile-local stable order: warp 0 items first)
        int acc = 0;
        for (int w = 0; w < kThreads / 32; w++) {
            const int c = wcnt[w][threadIdx.x];
            wcnt[w][threadIdx.x] = acc;
            acc += c;
        }
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kItems; r++) {
        if (dig[r] < kRadix) {
            const int64_t dst = tbase[dig[r]] + wcnt[wid][dig[r]] + loc[r];
            kout[dst] = key[r];
            vout[dst] = val[r];
        }
    }
}

}  // namespace

size_t radix_tmp_bytes(int64_t n)
{
    const int64_t nt = (n + kTile - 1) / kTile;
    const int64_t m = nt * kRadix;
    return sizeof(int64_t) * (size_t)(m + 1) + scan_tmp_bytes(m) + 256;
}

cudaError_t radix_sort_u64_i32(uint64_t *keys_a, uint64_t *keys_b, int32_t *vals_a, int32_t *vals_b, int64_t n,
                               uint64_t vary_bits, uint64_t **key_out, int32_t **val_out, void *tmp,
                               size_t tmp_bytes, cudaStream_t st)
{
    const int64_t nt = (n + kTile - 1) / kTile;
    const int64_t m = nt * kRadix;
    if (tmp_bytes < radix_tmp_bytes(n)) return cudaErrorInvalidValue;
    int64_t *counts = (int64_t *)tmp;
    void *scan_tmp = (void *)(((uintptr_t)(counts + m + 1) + 255) & ~(uintptr_t)255);
    uint64_t *ki = keys_a, *ko = keys_b;
    int32_t *vi = vals_a, *vo = vals_b;
    for (int shift = 0; shift < 64; shift += 8) {
        if (((vary_bits >> shift) & 0xFFull) == 0) continue;
        count_launch();
        k_hist<<<(unsigned)nt, kThreads, 0, st>>>(ki, n, shift, nt, counts);
        cudaError_t e = scan_exclusive_i64(counts, counts, m, scan_tmp, scan_tmp_bytes(m), st);
        if (e != cudaSuccess) return e;
        count_launch();
        k_scatter<<<(unsigned)nt, kThreads, 0, st>>>(ki, vi, ko, vo, n, shift, nt, counts);
        uint64_t *tk = ki; ki = ko; ko = tk;
        int32_t *tv = vi; vi = vo; vo = tv;
    }
    *key_out = ki;
    *val_out = vi;
    return cudaGetLastError();
}

}  // namespace fm
