// Does compute-sanitizer racecheck model the fused legs' synchronisation?
// Warp 0 writes a shared array; warp 1 waits on an mbarrier (try_wait.parity spin with
// the fused kernels' suspend-time hint) and reads.  Race-free by construction in both
// modes:
//   mode 0: every producer lane arrives (mbarrier count 32);
//   mode 1: the fused kernels' pattern -- the lanes __syncwarp, then lane 0 alone
//           arrives (count 1), as Rings::done() in kernels_fused.cu.
// A hazard reported in mode 1 but not in mode 0 means racecheck does not carry the
// other lanes' writes through __syncwarp + a single-lane arrive (the fused legs'
// reports in profiles/r02_sanitizer.txt are of that kind).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -o tools/mb_racecheck_bin tools/mb_racecheck.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned su(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }

__global__ void k(int *out, int mode)
{
    __shared__ __align__(8) unsigned long long bar;
    __shared__ int buf[32];
    if (threadIdx.x == 0)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(&bar)), "r"(mode ? 1 : 32) : "memory");
    __syncthreads();
    if (threadIdx.x < 32) {
        buf[threadIdx.x] = threadIdx.x * 3;
        if (mode)
            __syncwarp();
        if (!mode || threadIdx.x == 0)
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(&bar)) : "memory");
    } else {
        asm volatile(
            "{\n .reg .pred P1;\n WAIT:\n"
            " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
            " @!P1 bra WAIT;\n}\n" ::"r"(su(&bar)),
            "r"(0), "r"(0x989680)
            : "memory");
        out[threadIdx.x - 32] = buf[(threadIdx.x - 32 + 1) & 31];
    }
}

int main(int argc, char **argv)
{
    const int mode = argc > 1 ? atoi(argv[1]) : 0;
    int *d;
    cudaMalloc(&d, 32 * sizeof(int));
    k<<<1, 64>>>(d, mode);
    int h[32];
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    int ok = 1;
    for (int i = 0; i < 32; i++)
        ok &= h[i] == 3 * ((i + 1) & 31);
    printf("mb_racecheck mode %d: result %s\n", mode, ok ? "correct" : "WRONG");
    return 0;
}
