// Probe: cudaMalloc cost for one large block vs many smaller ones (bmg_setup allocation).
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>
#include <vector>
static double ms_since(std::chrono::steady_clock::time_point t)
{
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t).count();
}
int main()
{
    cudaFree(0);
    const size_t GB = 1ull << 30;
    for (int rep = 0; rep < 2; rep++) {
        auto t = std::chrono::steady_clock::now();
        void *p;
        cudaMalloc(&p, 5 * GB + GB / 2);
        double a = ms_since(t);
        t = std::chrono::steady_clock::now();
        cudaMemset(p, 0, 5 * GB + GB / 2);
        cudaDeviceSynchronize();
        double m = ms_since(t);
        t = std::chrono::steady_clock::now();
        cudaFree(p);
        double f = ms_since(t);
        printf("one 5.5 GB block: malloc %.2f ms, memset %.2f ms, free %.2f ms\n", a, m, f);
        std::vector<void *> ps;
        t = std::chrono::steady_clock::now();
        size_t sz[] = {1610612736, 536870912, 536870912, 671088640, 134217728, 134217728, 134217728, 1073741824,
                       167772160, 33554432, 33554432, 33554432, 268435456};
        for (size_t s : sz) {
            cudaMalloc(&p, s);
            ps.push_back(p);
        }
        double b = ms_since(t);
        for (void *q : ps)
            cudaFree(q);
        printf("13 blocks (same total): malloc %.2f ms\n", b);
    }
    cudaMemPool_t pool;
    cudaDeviceGetDefaultMemPool(&pool, 0);
    auto t = std::chrono::steady_clock::now();
    void *p;
    cudaMallocAsync(&p, 5 * GB + GB / 2, 0);
    cudaStreamSynchronize(0);
    printf("mallocAsync 5.5 GB: %.2f ms\n", ms_since(t));
    return 0;
}
