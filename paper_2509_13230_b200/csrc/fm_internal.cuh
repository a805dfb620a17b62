// fm_internal.cuh -- internal definitions shared by the CUDA translation units of the product
// library (NOT shared with oracle/).  sm_100a only.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "fastmaxent.h"

namespace fm {

constexpr int kG = 16;                         // work unit: one expected draw = 2^G (DESIGN 3.4)
constexpr int64_t kUnit = int64_t(1) << kG;
constexpr uint32_t kPlanMagic = 0x4C504D46u;   // "FMPL"
constexpr uint32_t kOwnerMagic = 0x57504D46u;  // "FMPW"
constexpr int kMaxDevices = 64;

// device-side error flags (atomicOr)
enum : uint32_t {
    kErrInvalid = 1u,     // a1 validation failed
    kErrState = 2u,       // planner invariant violated (cuts not strictly increasing)
    kErrBound = 4u,       // p > q (1 + 2^-50)
    kFlagWeightSat = 8u,  // ECM weight clamped
};

// one plan segment as the sampler reads it (96 B in 16-byte parts).  The plan stores UBCM records
// with a 64-byte stride (the first four parts; the ECM fields are not stored)
__host__ __device__ constexpr int kRecStride(int model) { return model == 0 ? 64 : 96; }
struct __align__(16) SegRec {
    int32_t u, a, b, sigma;  // focal rank, candidates [a, b), segment index in the row
    double h0, x0;           // initial bound at a-1: q0 = x0 / d0, h0 = -log(1 - q0)
    double d0, ku;           // ..., kappa_s[u]
    int32_t id_u, excl;      // perm[u]; directed: candidate rank of u's own node, else -1
    double rh0;              // RN(1 / h0): the sampler divides E / h by Markstein's correction
    double yu, ly_u;         // ECM: y_s[u], log y_s[u]
    double omT, iomT;        // ECM: 1 - T, RN(1 / (1 - T))
};

// double2 words per candidate in Plan::cand (one 16- or 32-byte record: one L2 sector per gather)
__host__ __device__ constexpr int kCandWords(int model) { return model == 0 ? 1 : 2; }

struct Plan {
    uint32_t magic;
    int model;
    int kind;           // FM_UNDIRECTED, FM_BIPARTITE, FM_DIRECTED (R16)
    int64_t n, nc, S;   // rows (+ set), candidates (- set; == n undirected)
    int F;
    int device;
    // a2/a3 (rank space)
    int32_t *perm;      // [n] rank -> id
    double *kappa_s;    // [n]
    double *y_s;        // [n] ECM
    double *ymax;       // [nc+1] ECM, over the candidates
    // candidates (the - set); aliases of the row arrays when undirected
    int32_t *cperm;
    double *ckappa, *cy, *cly;
    int32_t *excl;      // [n] directed: candidate rank of each row's own node
    double2 *cand;      // ECM: [2 nc] the sampler's 32-byte gather record per candidate rank:
                        //   (kappa, y), (log y, id); id in the low word.  NULL for UBCM
    // a4 segments
    int64_t n_seg;
    double *ly_s;       // [n] ECM: log y_s
    unsigned char *rec; // [n_seg] packed records for the sampler, stride kRecStride(model) bytes
    int64_t est_draws;  // sum of segment work estimates / 2^G
    // chunking (does not change results)
    // three chunkings: [0] coarse, [1] fine (the last samples of a call: short tail), [2] big (the
    // bulk of a call with many waves of work: fewer task switches; n_chunks[2] = 0: not built)
    int64_t n_chunks[3];
    int64_t *chunk_seg[3];   // [n_chunks+1] first segment of each lane-chunk
    int64_t *chunk_cap[3];   // [n_chunks+1] exclusive prefix of the lane-chunk scratch slots (edges)
    int64_t chunk_target[3]; // work per lane-chunk (units 2^G)
    int64_t wmax;         // bound of one segment's work (units 2^G)
    int64_t cap_per_sample;  // scratch edges per sample (upper bound of chunk_cap[n_chunks])
    bool slots_aligned;      // every scratch slot starts at a multiple of 4 edges (32 bytes)
    unsigned int *dev_flags; // planner invariant flags (checked by fm_sample_*)
    // capacity hint for the final edge list of a call (a performance hint, never a result):
    // edges per sample <= out_ratio * (est_draws - n_seg) + margin; raised when a call overflows,
    // lowered to the observed ratio (+1 %) otherwise.  Guarded by the library's object mutex.
    double out_ratio;
};

struct Owner {
    uint32_t magic;
    void *edges;    // device
    void *weights;  // device
    int64_t *offsets_host;
    cudaStream_t stream;
};

// ------------------------------------------------------------------------------------------
// Philox4x32-10 (Salmon et al., SC'11) -- DESIGN.md R1.
// ------------------------------------------------------------------------------------------
// round keys k + r * (0x9E3779B9, 0xBB67AE85), r = 0..9 (precomputed on the host: the kernel
// reads them from the constant bank as LOP3 operands)
struct PhiloxKey {
    uint32_t k0[10], k1[10];
};
inline PhiloxKey philox_key(uint64_t seed)
{
    PhiloxKey K;
    uint32_t a = (uint32_t)(seed & 0xffffffffu), b = (uint32_t)(seed >> 32);
    for (int r = 0; r < 10; r++) {
        K.k0[r] = a;
        K.k1[r] = b;
        a += 0x9E3779B9u;
        b += 0xBB67AE85u;
    }
    return K;
}
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, const PhiloxKey &K)
{
#pragma unroll
    for (int r = 0; r < 10; r++) {
        const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
        c = make_uint4(hi1 ^ c.y ^ K.k0[r], lo1, hi0 ^ c.w ^ K.k1[r], lo0);
    }
    return c;
}

__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint32_t k0, uint32_t k1)
{
#pragma unroll
    for (int r = 0; r < 10; r++) {
        const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
        c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return c;
}

// u01(k) = (k + 0.5) 2^-32 (R2); every operation exact.  The word is placed in the
// mantissa of 2^52 (v = 2^52 + k, no conversion instruction: the I2F conversions are
// variable-latency and compete for the six dependency scoreboards with the gathers), then
// v - (2^52 - 1/2) = k + 1/2 exactly (Sterbenz) and the scale is a power of two.
__device__ __forceinline__ double u01(uint32_t k)
{
    return __dmul_rn(__dsub_rn(__hiloint2double(0x43300000, (int)k), 0x1p52 - 0.5), 0x1p-32);
}
// the same value through a conversion instruction (the ECM sampler: measured faster there, the
// form above costs it a register spill)
__device__ __forceinline__ double u01_cvt(uint32_t k)
{
    return __dmul_rn(__dadd_rn((double)k, 0.5), 0x1p-32);
}

// every kernel launch of the library is counted (fm_timing.launches)
void count_launch(int n = 1);

// ------------------------------------------------------------------------------------------
// launch helpers (fm_scan.cu)
// ------------------------------------------------------------------------------------------
// exclusive prefix sum of int64 in[0..n) -> out[0..n], out[n] = total.  in == out allowed.
cudaError_t scan_exclusive_i64(const int64_t *in, int64_t *out, int64_t n, void *tmp, size_t tmp_bytes,
                               cudaStream_t st, bool small = false, bool zeroed = false);
size_t scan_tmp_bytes(int64_t n);
// same for uint64
cudaError_t scan_exclusive_u64(const uint64_t *in, uint64_t *out, int64_t n, void *tmp, size_t tmp_bytes,
                               cudaStream_t st);
// reverse inclusive max: out[t] = max(in[t], out[t+1]), out[n] = 0.0 (out has n+1 entries)
cudaError_t suffix_max_f64(const double *in, double *out, int64_t n, void *tmp, size_t tmp_bytes,
                           cudaStream_t st);

// closed-form expectations k, kvar (and ECM s, svar) of the listed nodes (fm_expect.cu, T1)
cudaError_t launch_expected(int model, int64_t n, const double *x, const double *y, const int32_t *nodes,
                            int64_t n_nodes, double *k, double *kvar, double *s, double *svar, cudaStream_t st);

// radix sort (fm_sort.cu): sort (key, val) pairs ascending by key, stable.  Buffers are
// ping-ponged; on return *key_out/*val_out point to the sorted arrays (one of the two buffers).
// vary_bits: OR of (key ^ key0) over all keys -- digits with no varying bit are skipped.
// hist: [8][256] digit counts of every byte position (computed by the caller's key kernel)
cudaError_t radix_sort_u64_i32(uint64_t *keys_a, uint64_t *keys_b, int32_t *vals_a, int32_t *vals_b, int64_t n,
                               uint64_t vary_bits, const unsigned int *hist, uint64_t **key_out, int32_t **val_out,
                               void *tmp, size_t tmp_bytes, cudaStream_t st);
size_t radix_tmp_bytes(int64_t n);

}  // namespace fm
