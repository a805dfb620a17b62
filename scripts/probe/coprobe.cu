// Co-residency probe (round 2): can a small-footprint streaming copy kernel (128 threads, <= 32
// registers: the 4096 registers per SM that three 256-thread sampler blocks at 80 registers leave
// free) run NEXT TO the persistent sampler, and what bandwidth does one such block per SM reach?
// Built as its own shared library; scripts/probe/coprobe.py drives it together with libfastmaxent.
#include <cuda_runtime.h>
#include <stdint.h>

__global__ void __launch_bounds__(128, 16) k_copy_small(int4 *__restrict__ dst, const int4 *__restrict__ src, long n)
{
    const long stride = (long)gridDim.x * 512;
    for (long i = (long)blockIdx.x * 512 + threadIdx.x; i < n; i += stride) {
        int4 v0, v1, v2, v3;
        v0 = __ldcs(src + i);
        if (i + 128 < n) v1 = __ldcs(src + i + 128);
        if (i + 256 < n) v2 = __ldcs(src + i + 256);
        if (i + 384 < n) v3 = __ldcs(src + i + 384);
        __stcs(dst + i, v0);
        if (i + 128 < n) __stcs(dst + i + 128, v1);
        if (i + 256 < n) __stcs(dst + i + 256, v2);
        if (i + 384 < n) __stcs(dst + i + 384, v3);
    }
}

// many short blocks: block b copies int4 [b * per, (b + 1) * per) and exits (like the compaction's blocks)
__global__ void __launch_bounds__(128, 16) k_copy_short(int4 *__restrict__ dst, const int4 *__restrict__ src, long n, long per)
{
    const long a = (long)blockIdx.x * per, z = a + per < n ? a + per : n;
    for (long i = a + threadIdx.x; i < z; i += 512) {
        int4 v0, v1, v2, v3;
        v0 = __ldcs(src + i);
        if (i + 128 < z) v1 = __ldcs(src + i + 128);
        if (i + 256 < z) v2 = __ldcs(src + i + 256);
        if (i + 384 < z) v3 = __ldcs(src + i + 384);
        __stcs(dst + i, v0);
        if (i + 128 < z) __stcs(dst + i + 128, v1);
        if (i + 256 < z) __stcs(dst + i + 256, v2);
        if (i + 384 < z) __stcs(dst + i + 384, v3);
    }
}

extern "C" int probe_copy_short(void *dst, const void *src, long n_int4, long per, void *stream)
{
    const long blocks = (n_int4 + per - 1) / per;
    k_copy_short<<<(unsigned)blocks, 128, 0, (cudaStream_t)stream>>>((int4 *)dst, (const int4 *)src, n_int4, per);
    return (int)cudaGetLastError();
}

extern "C" int probe_copy(void *dst, const void *src, long n_int4, int blocks, int carve_pct, void *stream)
{
    if (carve_pct >= 0) {
        cudaError_t e = cudaFuncSetAttribute(k_copy_small, cudaFuncAttributePreferredSharedMemoryCarveout, carve_pct);
        if (e != cudaSuccess) return (int)e;
    }
    k_copy_small<<<blocks, 128, 0, (cudaStream_t)stream>>>((int4 *)dst, (const int4 *)src, n_int4);
    return (int)cudaGetLastError();
}

extern "C" int probe_regs(void)
{
    cudaFuncAttributes fa;
    if (cudaFuncGetAttributes(&fa, k_copy_small) != cudaSuccess) return -1;
    return fa.numRegs;
}
