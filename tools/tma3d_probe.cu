// Probe: rank-3 fp64 TMA tile boxes like k3_rb7t's (tools/r2_* debugging).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

struct M1 { CUtensorMap m; };
__device__ __forceinline__ unsigned s32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }

__global__ void k(const __grid_constant__ M1 M, int bx, int by, int x, int y, int z, double *out)
{
    extern __shared__ __align__(1024) double sm[];
    unsigned long long *bar = reinterpret_cast<unsigned long long *>(sm + 8192);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(bar)) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(bar)), "r"(bx * by * 8) : "memory");
        asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                     ::"r"(s32(sm)), "l"(reinterpret_cast<unsigned long long>(&M.m)), "r"(x), "r"(y), "r"(z), "r"(s32(bar)) : "memory");
        asm volatile("{\n .reg .pred P1;\n W:\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n @!P1 bra W;\n}\n" ::"r"(s32(bar)) : "memory");
        out[0] = sm[0]; out[1] = sm[bx * by - 1];
    }
}

int main(int argc, char **argv)
{
    const int sel = argc > 1 ? atoi(argv[1]) : -1;
    void *p = nullptr; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    auto fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
    const int px = 288, ny2 = 257, nz2 = 257;
    double *g; cudaMalloc(&g, sizeof(double) * px * ny2 * nz2); cudaMemset(g, 0, sizeof(double) * px * ny2 * nz2);
    double *o; cudaMalloc(&o, 16);
    int cases[][5] = {{64, 1, 5, 5, 5}, {256, 1, 5, 5, 5}, {64, 2, 5, 5, 5}, {16, 12, 5, 5, 5}, {64, 12, 0, 0, 0}};
    (void)0;
    for (int ci = 0; ci < 5; ci++) {
        auto &c = cases[ci];
        if (sel >= 0 && ci != sel)
            continue;
        M1 M;
        cuuint64_t dims[3] = {(cuuint64_t)px, (cuuint64_t)ny2, (cuuint64_t)nz2};
        cuuint64_t st[2] = {(cuuint64_t)px * 8, (cuuint64_t)px * ny2 * 8};
        cuuint32_t box[3] = {(cuuint32_t)c[0], (cuuint32_t)c[1], 1}, es[3] = {1, 1, 1};
        CUresult r = fn(&M.m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, g, dims, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192 * 8 + 16);
        k<<<1, 32, 8192 * 8 + 16>>>(M, c[0], c[1], c[2], c[3], c[4], o);
        cudaError_t e = cudaDeviceSynchronize();
        printf("box %dx%d at (%d,%d,%d): encode %d, kernel %s\n", c[0], c[1], c[2], c[3], c[4], (int)r, cudaGetErrorString(e));
        if (e != cudaSuccess) return 1;
    }
    return 0;
}
