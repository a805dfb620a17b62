// microbench_ops.cu -- per-op costs and pipe peaks on the B200 for the sampler's compute roofline
// (DESIGN.md section 7).  Standalone benchmark, not part of the product library.
//
// Each kernel runs M iterations per thread over a full grid of one op on data that varies per
// iteration (a cheap integer hash), plus a baseline kernel with the hash only.  Under
//   ncu --metrics smsp__inst_executed.sum,smsp__inst_executed_pipe_fp64.sum,... ./microbench_ops
// (inst(op kernel) - inst(base kernel)) / (M * warps) = warp instructions per op call;
// the plain run prints the time per op and the DFMA / integer issue peaks.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -lineinfo -o microbench_ops microbench_ops.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int M = 2048;

__device__ __forceinline__ uint32_t hsh(uint32_t i, uint32_t t) { return (i * 0x9E3779B9u) ^ (t * 0x85EBCA6Bu); }
__device__ __forceinline__ double u01(uint32_t k) { return __dmul_rn(__dadd_rn((double)k, 0.5), 0x1p-32); }

__device__ __forceinline__ uint4 philox(uint4 c, uint32_t k0, uint32_t k1)
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

__global__ void k_base(double *out, uint32_t seed)
{
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t acc = 0;
    for (int i = 0; i < M; i++) acc += hsh(i + seed, t);
    out[t] = acc;
}
__global__ void k_base_u01(double *out, uint32_t seed)
{
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    double acc = 0;
    for (int i = 0; i < M; i++) acc = __dadd_rn(acc, u01(hsh(i + seed, t)));
    out[t] = acc;
}
__global__ void k_philox(double *out, uint32_t seed, uint32_t k0, uint32_t k1)
{
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t acc = 0;
    for (int i = 0; i < M; i++) {
        const uint4 w = philox(make_uint4(i + seed, 3u, t, 7u), k0, k1);
        acc += w.x ^ w.y;
    }
    out[t] = acc;
}
__global__ void k_log(double *out, uint32_t seed)
{
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    double acc = 0;
    for (int i = 0; i < M; i++) acc = __dadd_rn(acc, log(u01(hsh(i + seed, t))));
    out[t] = acc;
}
// log1p over the sampler's range of X = kappa_u kappa_v (1e-9 .. 1e3): X = u01 * 2^e with the
// exponent e in [-30, 10] WARP-UNIFORM (a function of the warp index and the iteration only), so
// every warp call takes one range path of log1p: the divergent cost of a warp whose lanes take
// both paths is not counted as algorithmic work (round-2 fix: the round-1 kernels drew e per lane
// from (h >> 26) - 30, i.e. e in [-30, 33], and executed both paths in most warps).
// emin/erange select a sub-range: [-30, 10] (all), [-30, -2] (the small-X path), [0, 10] (large X).
template <int emin, int erange>
__device__ __forceinline__ int warp_exp(uint32_t i)
{
    const uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    return emin + (int)((hsh(i * 7u + 3u, w) >> 8) % (uint32_t)erange);
}
template <int emin, int erange>
__global__ void k_base_log1p(double *out, uint32_t seed)
{
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    double acc = 0;
    for (int i = 0; i < M; i++) {
        const uint32_t h = hsh(i + seed, t);
        acc = __dadd_rn(acc, ldexp(u01(h), warp_exp<emin, erange>(i + seed)));
    }
    out[t] = acc;
}
template <int emin, int erange>
__global__ void k_log1p(double *out, uint32_t seed)
{
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    double acc = 0;
    for (int i = 0; i < M; i++) {
        const uint32_t h = hsh(i + seed, t);
        acc = __dadd_rn(acc, log1p(ldexp(u01(h), warp_exp<emin, erange>(i + seed))));
    }
    out[t] = acc;
}
__global__ void k_ddiv(double *out, uint32_t seed)
{
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    double acc = 0;
    for (int i = 0; i < M; i++) acc = __dadd_rn(acc, __ddiv_rn(u01(hsh(i + seed, t)), acc + 1.5));
    out[t] = acc;
}
__global__ void k_base_ddiv(double *out, uint32_t seed)
{
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    double acc = 0;
    for (int i = 0; i < M; i++) acc = __dadd_rn(acc, __dmul_rn(u01(hsh(i + seed, t)), acc + 1.5));
    out[t] = acc;
}
// DFMA peak: 8 independent chains
__global__ void k_dfma(double *out, uint32_t seed)
{
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    double a[8];
#pragma unroll
    for (int j = 0; j < 8; j++) a[j] = 1.0 + 1e-9 * (t + j + seed);
    const double b = 0.999999, c = 1e-7;
    for (int i = 0; i < M; i++) {
#pragma unroll
        for (int j = 0; j < 8; j++) a[j] = __fma_rn(a[j], b, c);
    }
    double s = 0;
#pragma unroll
    for (int j = 0; j < 8; j++) s += a[j];
    out[t] = s;
}
// integer issue peak: 8 independent chains of IADD3/LOP3
__global__ void k_int(double *out, uint32_t seed)
{
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t a[8];
#pragma unroll
    for (int j = 0; j < 8; j++) a[j] = t + j + seed;
    for (int i = 0; i < M; i++) {
#pragma unroll
        for (int j = 0; j < 8; j++) a[j] = (a[j] ^ 0x5bd1e995u) + (uint32_t)i;
    }
    uint32_t s = 0;
#pragma unroll
    for (int j = 0; j < 8; j++) s ^= a[j];
    out[t] = s;
}

int main()
{
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const int threads = 256, blocks = sms * 8;  // 64 warps per SM resident (occupancy permitting)
    const long long nthreads = (long long)threads * blocks;
    double *out;
    cudaMalloc(&out, sizeof(double) * nthreads);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    printf("{\"sms\": %d, \"clock_khz_attr\": %d, \"threads\": %lld, \"iters\": %d, \"kernels\": {", sms, clk, nthreads,
           M);
    const char *names[] = {"base", "base_u01", "philox", "log", "base_log1p", "log1p", "base_ddiv", "ddiv", "dfma8",
                           "int8", "base_log1p_small", "log1p_small", "base_log1p_large", "log1p_large"};
    for (int k = 0; k < 14; k++) {
        float best = 1e30f;
        for (int rep = 0; rep < 5; rep++) {
            cudaEventRecord(a);
            switch (k) {
            case 0: k_base<<<blocks, threads>>>(out, rep); break;
            case 1: k_base_u01<<<blocks, threads>>>(out, rep); break;
            case 2: k_philox<<<blocks, threads>>>(out, rep, 0x12345678u, 0x9abcdef0u); break;
            case 3: k_log<<<blocks, threads>>>(out, rep); break;
            case 4: k_base_log1p<-30, 41><<<blocks, threads>>>(out, rep); break;
            case 5: k_log1p<-30, 41><<<blocks, threads>>>(out, rep); break;
            case 6: k_base_ddiv<<<blocks, threads>>>(out, rep); break;
            case 7: k_ddiv<<<blocks, threads>>>(out, rep); break;
            case 8: k_dfma<<<blocks, threads>>>(out, rep); break;
            case 9: k_int<<<blocks, threads>>>(out, rep); break;
            case 10: k_base_log1p<-30, 29><<<blocks, threads>>>(out, rep); break;
            case 11: k_log1p<-30, 29><<<blocks, threads>>>(out, rep); break;
            case 12: k_base_log1p<0, 11><<<blocks, threads>>>(out, rep); break;
            case 13: k_log1p<0, 11><<<blocks, threads>>>(out, rep); break;
            }
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (ms < best) best = ms;
        }
        const double calls = (double)nthreads * M;  // thread-level op calls
        printf("%s\"%s\": {\"ms\": %.6f, \"ns_per_warp_call\": %.6g}", k ? ", " : "", names[k], best,
               best * 1e6 / (calls / 32.0));
    }
    printf("}, \"err\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
