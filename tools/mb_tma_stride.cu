// Probe: semantics of cuTensorMapEncodeTiled elementStrides = 2 on fp64 rows
// (does a box of 256 traversed with stride 2 land 128 packed elements?).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
__device__ __forceinline__ unsigned su(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__global__ void k(const __grid_constant__ CUtensorMap m, double *out, int x, int y, int txb, int *ok)
{
    __shared__ __align__(128) double s[512];
    __shared__ __align__(8) unsigned long long bar;
    for (int i = threadIdx.x; i < 512; i += blockDim.x) s[i] = -1.0;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar)), "r"(txb));
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(su(s)), "l"((unsigned long long)&m), "r"(x), "r"(y), "r"(su(&bar)) : "memory");
        unsigned done = 0;
        for (long it = 0; it < 2000000 && !done; it++)
            asm volatile("{\n.reg .pred P;\nmbarrier.test_wait.parity.shared::cta.b64 P, [%1], 0;\nselp.u32 %0, 1, 0, P;\n}" : "=r"(done) : "r"(su(&bar)));
        *ok = done;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 512; i += blockDim.x) out[i] = s[i];
}
int main()
{
    const int W = 1000, R = 4;
    double *g, *o;
    cudaMalloc(&g, W * R * 8);
    cudaMallocManaged(&o, 512 * 8);
    double h[W * R];
    for (int i = 0; i < W * R; i++) h[i] = i;
    cudaMemcpy(g, h, sizeof h, cudaMemcpyHostToDevice);
    void *p; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    auto fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
    CUtensorMap m;
    cuuint64_t dims[2] = {W, R}; cuuint64_t str[1] = {W * 8};
    cuuint32_t box[2] = {256, 1}; cuuint32_t es[2] = {2, 1};
    CUresult r = fn(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, g, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode %d\n", (int)r);
    int *ok; cudaMallocManaged(&ok, 4);
    setvbuf(stdout, NULL, _IONBF, 0);
    for (int txb : {128 * 8, 256 * 8})
    for (int x : {10, 11, -6, -5, 900, 901}) {
        k<<<1, 128>>>(m, o, x, 1, txb, ok);
        cudaError_t e = cudaDeviceSynchronize();
        printf("tx=%d x=%d err=%d done=%d: s[0..3]=%g %g %g %g  s[127]=%g s[128]=%g\n", txb, x, (int)e, *ok, o[0], o[1], o[2], o[3], o[127], o[128]);
        if (x == 900 || x == 901) printf("   s[45..52]= %g %g %g %g %g %g %g %g\n", o[45], o[46], o[47], o[48], o[49], o[50], o[51], o[52]);
    }
    return 0;
}
