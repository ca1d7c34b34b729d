// line.cuh -- per-line helpers of the zebra line relaxation (DESIGN §3 c11,
// §5.5): the tridiagonal row of a line point and parallel cyclic reduction
// over warp shuffles.
#pragma once
#include "bmg_internal.cuh"

namespace bmg {

// Chunk-local coefficients and right-hand side at position k of line `lc`.
template <int Y>
__device__ __forceinline__ void line_row(const Op &A, const double *__restrict__ f, const double *__restrict__ u,
                                         int lc, int k, double &lo, double &di, double &up, double &d)
{
    const long long P = A.pitch;
    const int i = Y ? lc : k + 1, j = Y ? k + 1 : lc;
    const long long p = (long long)j * P + i;
    di = A.O[p];
    double off;
    if (Y) {
        lo = A.S[p];
        up = A.S[p + P];
        off = A.W[p] * u[p - 1];
        off = fma(A.W[p + 1], u[p + 1], off);
        if (A.kind == 9) {
            off = fma(A.SW[p], u[p - P - 1], off);
            off = fma(A.NW[p + 1 - P], u[p - P + 1], off);  // SE(i,j) = NW(i+1,j-1)
            off = fma(A.NW[p], u[p + P - 1], off);
            off = fma(A.SW[p + P + 1], u[p + P + 1], off);  // NE(i,j) = SW(i+1,j+1)
        }
    } else {
        lo = A.W[p];
        up = A.W[p + 1];
        off = A.S[p] * u[p - P];
        off = fma(A.S[p + P], u[p + P], off);
        if (A.kind == 9) {
            off = fma(A.SW[p], u[p - P - 1], off);
            off = fma(A.NW[p + 1 - P], u[p - P + 1], off);
            off = fma(A.NW[p], u[p + P - 1], off);
            off = fma(A.SW[p + P + 1], u[p + P + 1], off);
        }
    }
    d = f[p] - off;
}

template <int Y>
__device__ __forceinline__ long long grid_index(const Op &A, int lc, int k)
{
    return Y ? (long long)(k + 1) * A.pitch + lc : (long long)lc * A.pitch + (k + 1);
}


// Parallel cyclic reduction over warp shuffles.
struct Eq {
    double lo, d, up, r;
};

__device__ __forceinline__ Eq shfl_eq(const Eq &e, int src)
{
    Eq o;
    o.lo = __shfl_sync(0xffffffffu, e.lo, src);
    o.d = __shfl_sync(0xffffffffu, e.d, src);
    o.up = __shfl_sync(0xffffffffu, e.up, src);
    o.r = __shfl_sync(0xffffffffu, e.r, src);
    return o;
}

// one PCR step on equation e (index i) with its neighbours em (i-s) and ep (i+s)
__device__ __forceinline__ Eq pcr_step(const Eq &e, const Eq &em, const Eq &ep, bool has_m, bool has_p)
{
    const double k1 = has_m ? e.lo * __drcp_rn(em.d) : 0.0;
    const double k2 = has_p ? e.up * __drcp_rn(ep.d) : 0.0;
    Eq o;
    o.lo = has_m ? -em.lo * k1 : 0.0;
    o.up = has_p ? -ep.up * k2 : 0.0;
    o.d = e.d - (has_m ? em.up * k1 : 0.0) - (has_p ? ep.lo * k2 : 0.0);
    o.r = e.r - (has_m ? em.r * k1 : 0.0) - (has_p ? ep.r * k2 : 0.0);
    return o;
}


// The 64 equations (2 per lane: e0 = index 2*lane, e1 = 2*lane+1) of a
// tridiagonal system, reduced by PCR in 6 steps; afterwards equation i reads
// e.d x_i = e.r.
__device__ __forceinline__ void pcr64(Eq &e0, Eq &e1, int lane)
{
    // PCR, stride 1: neighbours of 2t are (2t-1: lane t-1 slot 1) and (2t+1: own slot 1);
    // of 2t+1: (own slot 0) and (2t+2: lane t+1 slot 0)
    {
        const Eq m1 = shfl_eq(e1, lane > 0 ? lane - 1 : 0);
        const Eq p0 = shfl_eq(e0, lane < 31 ? lane + 1 : 31);
        const Eq n0 = pcr_step(e0, m1, e1, lane > 0, true);
        const Eq n1 = pcr_step(e1, e0, p0, true, lane < 31);
        e0 = n0;
        e1 = n1;
    }
    // strides 2, 4, .., 32 (in equations) = 1, 2, .., 16 lanes, same slot
#pragma unroll
    for (int sl = 1; sl < 32; sl <<= 1) {
        const bool hm = lane >= sl, hp = lane + sl < 32;
        const Eq a0 = shfl_eq(e0, hm ? lane - sl : lane), b0 = shfl_eq(e0, hp ? lane + sl : lane);
        const Eq a1 = shfl_eq(e1, hm ? lane - sl : lane), b1 = shfl_eq(e1, hp ? lane + sl : lane);
        e0 = pcr_step(e0, a0, b0, hm, hp);
        e1 = pcr_step(e1, a1, b1, hm, hp);
    }
}

}  // namespace bmg
