// Probe: does a tiled fp64 tensor map with elementStrides[0] = 2 de-interleave a row
// (box of 2*n columns -> n every-other elements, packed in shared memory)?
// nvcc -gencode arch=compute_100a,code=sm_100a tools/tma_estride_probe.cu -o /tmp/p
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cuda_runtime.h>

struct M1 { CUtensorMap m; };
__device__ __forceinline__ unsigned s32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }

__global__ void k(const __grid_constant__ M1 M, int rank, int x, int y, unsigned tx, double *out, int *ok)
{
    extern __shared__ __align__(1024) double sm[];
    unsigned long long *bar = reinterpret_cast<unsigned long long *>(sm + 4096);
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm[i] = -1.0;
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(bar)) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(bar)), "r"(tx) : "memory");
        if (rank == 2)
            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                         ::"r"(s32(sm)), "l"(reinterpret_cast<unsigned long long>(&M.m)), "r"(x), "r"(y), "r"(s32(bar)) : "memory");
        else
            asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                         ::"r"(s32(sm)), "l"(reinterpret_cast<unsigned long long>(&M.m)), "r"(x), "r"(y), "r"(0), "r"(s32(bar)) : "memory");
        unsigned done = 0;
        long long t0 = clock64();
        while (!done && clock64() - t0 < 200000000LL)
            asm volatile("{\n .reg .pred P1;\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], 0;\n selp.u32 %0, 1, 0, P1;\n}\n"
                         : "=r"(done) : "r"(s32(bar)) : "memory");
        *ok = done;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) out[i] = sm[i];
}

int main()
{
    void *p = nullptr; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    auto fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
    const int W = 416, R = 8, NP = 5;
    double *h = new double[(size_t)W * R * NP];
    for (int z = 0; z < NP; z++) for (int r = 0; r < R; r++) for (int x = 0; x < W; x++) h[((size_t)z * R + r) * W + x] = z * 100000 + r * 1000 + x;
    double *g; cudaMalloc(&g, sizeof(double) * W * R * NP); cudaMemcpy(g, h, sizeof(double) * W * R * NP, cudaMemcpyHostToDevice);
    double *o; cudaMalloc(&o, 1024 * 8); int *okd; cudaMalloc(&okd, 4);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 4096 * 8 + 64);
    struct Case { int rank, box0, es0, x; unsigned tx; } cases[] = {
        {2, 192, 2, 6, 96 * 8}, {2, 192, 2, 7, 96 * 8}, {2, 192, 2, -3, 96 * 8}, {2, 192, 2, 406, 96 * 8},
        {3, 192, 2, 6, 5 * 96 * 8}, {3, 192, 2, 7, 5 * 96 * 8}, {2, 192, 1, 6, 192 * 8}};
    for (auto &c : cases) {
        M1 M;
        cuuint64_t dims[3] = {(cuuint64_t)W, (cuuint64_t)R, (cuuint64_t)NP};
        cuuint64_t st[2] = {(cuuint64_t)W * 8, (cuuint64_t)W * R * 8};
        cuuint32_t box[3] = {(cuuint32_t)c.box0, 1, (cuuint32_t)NP}, es[3] = {(cuuint32_t)c.es0, 1, 1};
        CUresult r = fn(&M.m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, c.rank, g, dims, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        printf("rank %d box0 %d es0 %d x %d: encode %d", c.rank, c.box0, c.es0, c.x, (int)r);
        if (r != CUDA_SUCCESS) { printf("\n"); continue; }
        k<<<1, 128, 4096 * 8 + 64>>>(M, c.rank, c.x, 2, c.tx, o, okd);
        cudaError_t e = cudaDeviceSynchronize();
        double hs[1024]; int ok = 0;
        cudaMemcpy(hs, o, sizeof(hs), cudaMemcpyDeviceToHost); cudaMemcpy(&ok, okd, 4, cudaMemcpyDeviceToHost);
        printf(" kernel %s, mbar complete %d\n  sm[0..5] = %.0f %.0f %.0f %.0f %.0f %.0f ; sm[94..97] = %.0f %.0f %.0f %.0f ; sm[190..193] = %.0f %.0f %.0f %.0f ; sm[96*4+0..1] %.0f %.0f sm[480] %.0f\n",
               cudaGetErrorString(e), ok, hs[0], hs[1], hs[2], hs[3], hs[4], hs[5], hs[94], hs[95], hs[96], hs[97], hs[190], hs[191], hs[192], hs[193], hs[384], hs[385], hs[480]);
        if (e != cudaSuccess) return 1;
    }
    return 0;
}
