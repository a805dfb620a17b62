// Does the B200 box run two kernels from two streams concurrently?  Kernel A spins until kernel B
// (launched second, other stream) sets a flag; a watchdog bounds the spin.  Variants: the first
// stream is the legacy default stream or a non-blocking stream; kernel A is 1 block or a
// persistent grid with heavy per-SM resources (like the sampler).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_wait(volatile int *flag, long long limit, int *timed_out)
{
    if (threadIdx.x == 0) {
        long long t0 = clock64();
        while (*flag == 0) {
            if (clock64() - t0 > limit) { atomicExch(timed_out, 1); break; }
        }
    }
    __syncthreads();
}
__global__ void k_set(volatile int *flag) { if (threadIdx.x == 0 && blockIdx.x == 0) *flag = 1; }

static void run(const char *name, cudaStream_t sa, cudaStream_t sb, int blocks_a, int threads_a, size_t smem_a)
{
    int *flag, *to;
    cudaMalloc(&flag, 4); cudaMalloc(&to, 4);
    cudaMemset(flag, 0, 4); cudaMemset(to, 0, 4);
    cudaDeviceSynchronize();
    k_wait<<<blocks_a, threads_a, smem_a, sa>>>(flag, 2000000000LL, to);  // ~1 s at 2 GHz
    k_set<<<1, 32, 0, sb>>>(flag);
    cudaError_t e = cudaDeviceSynchronize();
    int h = -1;
    cudaMemcpy(&h, to, 4, cudaMemcpyDeviceToHost);
    printf("%-60s %s (%s)\n", name, h == 0 ? "CONCURRENT" : "SERIALISED (A timed out)", cudaGetErrorString(e));
    cudaFree(flag); cudaFree(to);
}

int main()
{
    cudaStream_t nb1, nb2;
    cudaStreamCreateWithFlags(&nb1, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&nb2, cudaStreamNonBlocking);
    const char *mc = getenv("CUDA_DEVICE_MAX_CONNECTIONS");
    printf("CUDA_DEVICE_MAX_CONNECTIONS=%s\n", mc ? mc : "(unset)");
    run("A legacy default stream (1 block), B non-blocking", 0, nb1, 1, 32, 0);
    run("A non-blocking (1 block), B non-blocking", nb1, nb2, 1, 32, 0);
    run("A non-blocking (444 x 256, 27 KB smem), B non-blocking", nb1, nb2, 444, 256, 27 * 1024);
    run("A non-blocking (148 x 32, 64 KB smem), B non-blocking", nb1, nb2, 148, 32, 64 * 1024);
    return 0;
}
