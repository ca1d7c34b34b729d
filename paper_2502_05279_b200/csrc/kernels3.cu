// kernels3.cu -- the 3-D BoxMG kernels (DESIGN.md §3
// c16-c24, §5.8): stencil ingest, operator-induced interpolation, Galerkin
// RAP, coarsest dense factor/solve, multicolour point Gauss-Seidel, residual,
// restriction, interpolation-correction and the residual norm.  One thread per
// point (x fastest, so every warp reads consecutive doubles of a row).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <climits>
#include <mutex>
#include <cstdlib>
#include <utility>

#include "bmg3.cuh"
#include "bmg_internal.cuh"

namespace bmg3 {

using bmg::rcp_pos;

__device__ __forceinline__ bool inside3(const Grid3 &g, int i, int j, int k)
{
    return i >= 1 && i <= g.nx && j >= 1 && j <= g.ny && k >= 1 && k <= g.nz;
}

// ---------------------------------------------------------------- full row access
// A[p, p+off_e] for e = 0..26 from the symmetric half (e > 13: the lower entry
// 26-e stored at the neighbour).  Ring couplings are 0 by construction.
__device__ __forceinline__ double row_entry(const Op3 &A, long long p, int e)
{
    if (e == 13)
        return A.O[p];
    if (e < 13)
        return A.a[e] ? A.a[e][p] : 0.0;
    const int l = 26 - e;
    return A.a[l] ? A.a[l][p + eoff(A.g, e)] : 0.0;
}

// sum_{q != p} a_pq u_q
template <int KIND>
__device__ __forceinline__ double offdiag(const Op3 &A, const double *__restrict__ u, long long p)
{
    const long long X = 1, Y = A.g.px, Z = A.g.ps;
    if (KIND == 7) {
        const double *W = A.a[12], *S = A.a[10], *B = A.a[4];
        return W[p] * u[p - X] + W[p + X] * u[p + X] + S[p] * u[p - Y] + S[p + Y] * u[p + Y] + B[p] * u[p - Z] +
               B[p + Z] * u[p + Z];
    } else {
        double s = 0.0;
#pragma unroll
        for (int e = 0; e < 13; e++) {
            const long long o = (long long)(e / 9 - 1) * Z + (long long)((e / 3) % 3 - 1) * Y + (e % 3 - 1);
            s += A.a[e][p] * u[p + o] + A.a[e][p - o] * u[p - o];
        }
        return s;
    }
}

// ---------------------------------------------------------------- S0 ingest (c16, c18)
struct PtrArr {
    const double *p[14];
};
struct WPtrArr {
    double *p[14];
};

__global__ void k3_ingest_v(int kind, Grid3 g, PtrArr src, WPtrArr dst, int *err)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y, k = blockIdx.z;
    if (i > g.nx + 1)
        return;
    const long long p = at3(g, i, j, k);
    const bool in = inside3(g, i, j, k);
#pragma unroll
    for (int q = 0; q < 14; q++) {
        if (!dst.p[q])
            continue;
        double v = 0.0;
        if (in) {
            v = src.p[q][p];
            if (q > 0) {
                const int e = q - 1;
                if (!inside3(g, i + e % 3 - 1, j + (e / 3) % 3 - 1, k + e / 9 - 1))
                    v = 0.0;
            } else if (!(v > 0.0)) {
                atomicOr(err, bmg::ERR_DIAG);
            }
        }
        dst.p[q][p] = v;
    }
}

void launch3_ingest(int kind, const Grid3 &g, const double *const src[14], double *const dst[14], int *err,
                    cudaStream_t s)
{
    PtrArr a;
    WPtrArr b;
    for (int q = 0; q < 14; q++) {
        a.p[q] = src[q];
        b.p[q] = dst[q];
    }
    dim3 grid((g.nx + 2 + 127) / 128, g.ny + 2, g.nz + 2);
    k3_ingest_v<<<grid, 128, 0, s>>>(kind, g, a, b, err);
}

// ---------------------------------------------------------------- S1 interpolation (c19)
// P(q, C): 1 if q = 2C, the stored corner weight if C is a corner of q, else 0
__device__ double pw3(const CI3 &ci, int qi, int qj, int qk, int Ci, int Cj, int Ck)
{
    const int q[3] = {qi, qj, qk}, C[3] = {Ci, Cj, Ck};
    int Q[3], corner = 0, nb = 0;
    const int m = (qi & 1) | (qj & 1) << 1 | (qk & 1) << 2;
#pragma unroll
    for (int d = 0; d < 3; d++) {
        if (q[d] & 1) {
            Q[d] = (q[d] + 1) >> 1;
            if (C[d] == Q[d])
                corner |= 1 << nb;
            else if (C[d] != Q[d] - 1)
                return 0.0;
            nb++;
        } else {
            Q[d] = q[d] >> 1;
            if (C[d] != Q[d])
                return 0.0;
        }
    }
    if (m == 0)
        return 1.0;
    return ci.w[slot_base(m) + corner][at3(ci.c, Q[0], Q[1], Q[2])];
}

// The oracle's arithmetic in its order (no contraction), so level-0 weights are
// bitwise equal to it: collapse onto the odd axes, sig, R, sides, den, weights.
__device__ void interp_point(const Op3 &A, const CI3 &ci, double *const *wout, int i, int j, int k, int *err)
{
    const int odd[3] = {i & 1, j & 1, k & 1};
    const int m = odd[0] | odd[1] << 1 | odd[2] << 2;
    const int nodd = odd[0] + odd[1] + odd[2];
    const long long p = at3(A.g, i, j, k);
    double a[27], b[27];
#pragma unroll
    for (int e = 0; e < 27; e++) {
        a[e] = row_entry(A, p, e);
        b[e] = 0.0;
    }
    double sig = 0.0;
    for (int e = 0; e < 27; e++) {
        int o0 = e % 3 - 1, o1 = (e / 3) % 3 - 1, o2 = e / 9 - 1;
        if (!odd[0])
            o0 = 0;
        if (!odd[1])
            o1 = 0;
        if (!odd[2])
            o2 = 0;
        const int t = (o2 + 1) * 9 + (o1 + 1) * 3 + (o0 + 1);
        b[t] = __dadd_rn(b[t], a[e]);
        if (e != 13)
            sig = __dsub_rn(sig, a[e]);
    }
    const double R = __dsub_rn(a[13], sig);
    double eps = __longlong_as_double(0x7FF0000000000000LL);  // +inf
    for (int d = 0; d < 3; d++) {
        if (!odd[d])
            continue;
        for (int s = -1; s <= 1; s += 2) {
            double c = 0.0;
            for (int e = 0; e < 27; e++) {
                const int od = d == 0 ? e % 3 - 1 : d == 1 ? (e / 3) % 3 - 1 : e / 9 - 1;
                if (od == s)
                    c = __dsub_rn(c, b[e]);
            }
            eps = fmin(eps, fabs(c));
        }
    }
    eps = __ddiv_rn(eps, a[13]);
    double sigb = 0.0;
    for (int e = 0; e < 27; e++)
        if (e != 13)
            sigb = __dsub_rn(sigb, b[e]);
    const double den = __dadd_rn(sigb, R > __dmul_rn(eps, sig) ? R : 0.0);
    if (!(den > 0.0)) {
        atomicOr(err, bmg::ERR_DEN);
        return;
    }
    const int I = odd[0] ? (i + 1) >> 1 : i >> 1, J = odd[1] ? (j + 1) >> 1 : j >> 1,
              K = odd[2] ? (k + 1) >> 1 : k >> 1;
    const long long c0 = at3(ci.c, I, J, K);
    const int ncorner = 1 << nodd;
    for (int c = 0; c < ncorner; c++) {
        int C[3] = {I, J, K}, nb = 0;
        for (int d = 0; d < 3; d++)
            if (odd[d]) {
                if (!((c >> nb) & 1))
                    C[d] -= 1;
                nb++;
            }
        double s = 0.0;
        for (int e = 0; e < 27; e++) {
            if (e == 13)
                continue;
            const double pv = pw3(ci, i + e % 3 - 1, j + (e / 3) % 3 - 1, k + e / 9 - 1, C[0], C[1], C[2]);
            s = __dsub_rn(s, __dmul_rn(b[e], pv));
        }
        wout[slot_base(m) + c][c0] = __ddiv_rn(s, den);
    }
}

struct CIW {
    double *w[26];
};

__global__ void k3_interp(Op3 A, CI3 ci, CIW out, int phase, int *err)
{
    const int I = blockIdx.x * blockDim.x + threadIdx.x + 1, J = blockIdx.y + 1, K = blockIdx.z + 1;
    for (int m = 1; m < 8; m++) {
        if (__popc(m) != phase)
            continue;
        const int i = (m & 1) ? 2 * I - 1 : 2 * I, j = (m & 2) ? 2 * J - 1 : 2 * J, k = (m & 4) ? 2 * K - 1 : 2 * K;
        if (i > A.g.nx || j > A.g.ny || k > A.g.nz)
            continue;
        interp_point(A, ci, out.w, i, j, k, err);
    }
}

void launch3_interp(const Op3 &A, double *const ci[26], const Grid3 &cg, int *err, cudaStream_t s)
{
    CI3 v;
    CIW o;
    v.c = cg;
    for (int q = 0; q < 26; q++) {
        v.w[q] = ci[q];
        o.w[q] = ci[q];
    }
    const int hx = (A.g.nx + 1) / 2, hy = (A.g.ny + 1) / 2, hz = (A.g.nz + 1) / 2;
    dim3 grid((hx + 63) / 64, hy, hz);
    for (int phase = 1; phase <= 3; phase++)
        k3_interp<<<grid, 64, 0, s>>>(A, v, o, phase, err);
}

// ---------------------------------------------------------------- S2 Galerkin RAP (c20)
// Gather at coarse C: A_c(C, D) = sum_f sum_g P(f,C) A(f,g) P(g,D) over the fine
// f of C's 3x3x3 box, their stencil neighbours g and g's coarse corners D, kept
// for the 14 stored offsets D - C (lower half and centre).
template <int KIND>
__global__ void k3_rap(Op3 A, CI3 ci, WPtrArr dst)
{
    const int Ci = blockIdx.x * blockDim.x + threadIdx.x + 1, Cj = blockIdx.y + 1, Ck = blockIdx.z + 1;
    if (Ci > ci.c.nx)
        return;
    double acc[14];
#pragma unroll
    for (int q = 0; q < 14; q++)
        acc[q] = 0.0;
    for (int o1 = 0; o1 < 27; o1++) {
        const int fi = 2 * Ci + o1 % 3 - 1, fj = 2 * Cj + (o1 / 3) % 3 - 1, fk = 2 * Ck + o1 / 9 - 1;
        if (!inside3(A.g, fi, fj, fk))
            continue;
        const double w1 = pw3(ci, fi, fj, fk, Ci, Cj, Ck);
        if (w1 == 0.0)
            continue;
        const long long pf = at3(A.g, fi, fj, fk);
        for (int e = 0; e < 27; e++) {
            if (KIND == 7 && e != 4 && e != 10 && e != 12 && e != 13 && e != 14 && e != 16 && e != 22)
                continue;
            const int gi = fi + e % 3 - 1, gj = fj + (e / 3) % 3 - 1, gk = fk + e / 9 - 1;
            if (!inside3(A.g, gi, gj, gk))
                continue;
            const double a = row_entry(A, pf, e);
            if (a == 0.0)
                continue;
            const double wa = w1 * a;
            const int lo0 = (gi & 1) ? (gi + 1) / 2 - 1 : gi / 2, hi0 = (gi & 1) ? (gi + 1) / 2 : gi / 2;
            const int lo1 = (gj & 1) ? (gj + 1) / 2 - 1 : gj / 2, hi1 = (gj & 1) ? (gj + 1) / 2 : gj / 2;
            const int lo2 = (gk & 1) ? (gk + 1) / 2 - 1 : gk / 2, hi2 = (gk & 1) ? (gk + 1) / 2 : gk / 2;
            for (int Dk = lo2; Dk <= hi2; Dk++)
                for (int Dj = lo1; Dj <= hi1; Dj++)
                    for (int Di = lo0; Di <= hi0; Di++) {
                        const int dx = Di - Ci, dy = Dj - Cj, dz = Dk - Ck;
                        if (dx < -1 || dx > 1 || dy < -1 || dy > 1 || dz < -1 || dz > 1)
                            continue;
                        const int ed = (dz + 1) * 9 + (dy + 1) * 3 + (dx + 1);
                        if (ed > 13 || !inside3(ci.c, Di, Dj, Dk))
                            continue;
                        const double w2 = pw3(ci, gi, gj, gk, Di, Dj, Dk);
#pragma unroll
                        for (int q = 0; q < 14; q++)
                            if (q == ed)
                                acc[q] += wa * w2;
                    }
        }
    }
    const long long pc = at3(ci.c, Ci, Cj, Ck);
    dst.p[0][pc] = acc[13];
#pragma unroll
    for (int e = 0; e < 13; e++)
        dst.p[1 + e][pc] = acc[e];
}

void launch3_rap(const Op3 &A, const CI3 &ci, double *const dst[14], int *err, cudaStream_t s)
{
    (void)err;
    WPtrArr d;
    for (int q = 0; q < 14; q++)
        d.p[q] = dst[q];
    dim3 grid((ci.c.nx + 63) / 64, ci.c.ny, ci.c.nz);
    if (A.kind == 7)
        k3_rap<7><<<grid, 64, 0, s>>>(A, ci, d);
    else
        k3_rap<27><<<grid, 64, 0, s>>>(A, ci, d);
}

// ---------------------------------------------------------------- S3 / C5 coarsest (c24)
__global__ void k3_assemble_dense(Op3 A, double *M)
{
    const int n = A.g.nx * A.g.ny * A.g.nz;
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n)
        return;
    const int i = p % A.g.nx + 1, j = (p / A.g.nx) % A.g.ny + 1, k = p / (A.g.nx * A.g.ny) + 1;
    const long long q = at3(A.g, i, j, k);
    for (int e = 0; e < 27; e++) {
        const int qi = i + e % 3 - 1, qj = j + (e / 3) % 3 - 1, qk = k + e / 9 - 1;
        if (!inside3(A.g, qi, qj, qk))
            continue;
        M[(long long)p * n + ((long long)(qk - 1) * A.g.ny + (qj - 1)) * A.g.nx + (qi - 1)] = row_entry(A, q, e);
    }
}

void launch3_assemble_dense(const Op3 &A, double *M, cudaStream_t s)
{
    const int n = A.g.nx * A.g.ny * A.g.nz;
    cudaMemsetAsync(M, 0, sizeof(double) * (size_t)n * n, s);
    k3_assemble_dense<<<(n + 127) / 128, 128, 0, s>>>(A, M);
}

// forward + backward substitution with L (lower triangle) in one CTA
__global__ void k3_coarse_solve(Op3 A, const double *__restrict__ L, const double *__restrict__ f,
                                double *__restrict__ u)
{
    extern __shared__ double b[];
    const int nx = A.g.nx, ny = A.g.ny, n = nx * ny * A.g.nz;
    if (n <= 32) {  // one warp: no barriers (the CTA loop pays two per unknown)
        if (threadIdx.x < 32) {
            const int i = threadIdx.x;
            const long long q = at3(A.g, i % nx + 1, (i / nx) % ny + 1, i / (nx * ny) + 1);
            double x = i < n ? f[q] : 0.0;
            for (int r = 0; r < n; r++) {
                const double br = __shfl_sync(0xffffffffu, x, r) / L[(long long)r * n + r];
                if (i == r)
                    x = br;
                else if (i > r && i < n)
                    x -= L[(long long)i * n + r] * br;
            }
            for (int r = n - 1; r >= 0; r--) {
                const double br = __shfl_sync(0xffffffffu, x, r) / L[(long long)r * n + r];
                if (i == r)
                    x = br;
                else if (i < r)
                    x -= L[(long long)r * n + i] * br;
            }
            if (i < n)
                u[q] = x;
        }
        return;
    }
    for (int t = threadIdx.x; t < n; t += blockDim.x)
        b[t] = f[at3(A.g, t % nx + 1, (t / nx) % ny + 1, t / (nx * ny) + 1)];
    __syncthreads();
    for (int r = 0; r < n; r++) {
        if (threadIdx.x == 0)
            b[r] /= L[(long long)r * n + r];
        __syncthreads();
        const double br = b[r];
        for (int t = r + 1 + threadIdx.x; t < n; t += blockDim.x)
            b[t] -= L[(long long)t * n + r] * br;
        __syncthreads();
    }
    for (int r = n - 1; r >= 0; r--) {
        if (threadIdx.x == 0)
            b[r] /= L[(long long)r * n + r];
        __syncthreads();
        const double br = b[r];
        for (int t = threadIdx.x; t < r; t += blockDim.x)
            b[t] -= L[(long long)r * n + t] * br;
        __syncthreads();
    }
    for (int t = threadIdx.x; t < n; t += blockDim.x)
        u[at3(A.g, t % nx + 1, (t / nx) % ny + 1, t / (nx * ny) + 1)] = b[t];
}

void launch3_coarse_solve(const Op3 &A, const double *Lf, const double *f, double *u, cudaStream_t s)
{
    const int n = A.g.nx * A.g.ny * A.g.nz;
    const int threads = n < 1024 ? ((n + 31) / 32) * 32 : 1024;
    k3_coarse_solve<<<1, threads, sizeof(double) * n, s>>>(A, Lf, f, u);
}

// ---------------------------------------------------------------- C1 point GS (c22)
// 7-point: red-black, colour (i+j+k) mod 2; a thread per point of the colour.
__global__ void k3_relax7(Op3 A, const double *__restrict__ f, double *__restrict__ u, int colour)
{
    const int j = blockIdx.y + 1, k = blockIdx.z + 1;
    const int i = (((colour + j + k) & 1) ? 1 : 2) + 2 * (blockIdx.x * blockDim.x + threadIdx.x);
    if (i > A.g.nx)
        return;
    const long long p = at3(A.g, i, j, k);
    u[p] = (f[p] - offdiag<7>(A, u, p)) * rcp_pos(A.O[p]);
}

// 27-point: eight colours (i mod 2) + 2 (j mod 2) + 4 (k mod 2)
__global__ void k3_relax27(Op3 A, const double *__restrict__ f, double *__restrict__ u, int colour)
{
    const int i = ((colour & 1) ? 1 : 2) + 2 * (blockIdx.x * blockDim.x + threadIdx.x);
    const int j = ((colour & 2) ? 1 : 2) + 2 * blockIdx.y, k = ((colour & 4) ? 1 : 2) + 2 * blockIdx.z;
    if (i > A.g.nx || j > A.g.ny || k > A.g.nz)
        return;
    const long long p = at3(A.g, i, j, k);
    u[p] = (f[p] - offdiag<27>(A, u, p)) * rcp_pos(A.O[p]);
}

void launch3_relax_point(const Op3 &A, const double *f, double *u, int nsweeps, cudaStream_t s, int *nlaunch)
{
    const int hx = (A.g.nx + 1) / 2;
    for (int sw = 0; sw < nsweeps; sw++) {
        if (A.kind == 7) {
            dim3 grid((hx + 127) / 128, A.g.ny, A.g.nz);
            for (int c = 0; c < 2; c++)
                k3_relax7<<<grid, 128, 0, s>>>(A, f, u, c);
            if (nlaunch)
                *nlaunch += 2;
        } else {
            dim3 grid((hx + 127) / 128, (A.g.ny + 1) / 2, (A.g.nz + 1) / 2);
            for (int c = 0; c < 8; c++)
                k3_relax27<<<grid, 128, 0, s>>>(A, f, u, c);
            if (nlaunch)
                *nlaunch += 8;
        }
    }
}


// 27-point levels, colour-major copy: per colour c its sub-lattice
// points q = (kk*cy + jj)*cx + ii hold the full row, cf[e*Nc + q] = A[p, p+off_e]
// for e != 13 and cf[13*Nc + q] = rcp_pos(a_O), so a colour pass streams exactly its
// own coefficients once (the symmetric half would re-read every plane in all 8 passes).
struct Sub {
    int i0, j0, k0, cx, cy, cz;
};

__host__ __device__ inline Sub sub_of(const Grid3 &g, int c)
{
    Sub b;
    b.i0 = (c & 1) ? 1 : 2;
    b.j0 = (c & 2) ? 1 : 2;
    b.k0 = (c & 4) ? 1 : 2;
    b.cx = (c & 1) ? (g.nx + 1) / 2 : g.nx / 2;
    b.cy = (c & 2) ? (g.ny + 1) / 2 : g.ny / 2;
    b.cz = (c & 4) ? (g.nz + 1) / 2 : g.nz / 2;
    return b;
}

long long relax27_doubles(const Grid3 &g)
{
    long long n = 0;
    for (int c = 0; c < 8; c++) {
        const Sub b = sub_of(g, c);
        n += 27LL * b.cx * b.cy * b.cz;
    }
    return n;
}

__global__ void k3_build_relax27(Op3 A, Sub b, double *__restrict__ cf)
{
    const int ii = blockIdx.x * blockDim.x + threadIdx.x, jj = blockIdx.y, kk = blockIdx.z;
    if (ii >= b.cx)
        return;
    const long long Nc = (long long)b.cx * b.cy * b.cz, q = ((long long)kk * b.cy + jj) * b.cx + ii;
    const long long p = at3(A.g, b.i0 + 2 * ii, b.j0 + 2 * jj, b.k0 + 2 * kk);
    for (int e = 0; e < 27; e++)
        cf[e * Nc + q] = e == 13 ? rcp_pos(A.O[p]) : row_entry(A, p, e);
}

void launch3_build_relax27(const Op3 &A, double *cf, cudaStream_t s)
{
    for (int c = 0; c < 8; c++) {
        const Sub b = sub_of(A.g, c);
        if (b.cx * b.cy * b.cz == 0)
            continue;
        k3_build_relax27<<<dim3((b.cx + 127) / 128, b.cy, b.cz), 128, 0, s>>>(A, b, cf);
        cf += 27LL * b.cx * b.cy * b.cz;
    }
}

__global__ void __launch_bounds__(128) k3_relax27c(Grid3 g, Sub b, const double *__restrict__ cf,
                                                   const double *__restrict__ f, double *__restrict__ u)
{
    const int ii = blockIdx.x * 32 + threadIdx.x, jj = blockIdx.y * 4 + threadIdx.y, kk = blockIdx.z;
    if (ii >= b.cx || jj >= b.cy)
        return;
    const long long Nc = (long long)b.cx * b.cy * b.cz, q = ((long long)kk * b.cy + jj) * b.cx + ii;
    const long long p = at3(g, b.i0 + 2 * ii, b.j0 + 2 * jj, b.k0 + 2 * kk);
    const long long Y = g.px, Z = g.ps;
    double s = 0.0;
#pragma unroll
    for (int e = 0; e < 27; e++) {
        if (e == 13)
            continue;
        const long long o = (long long)(e / 9 - 1) * Z + (long long)((e / 3) % 3 - 1) * Y + (e % 3 - 1);
        s += __ldg(cf + e * Nc + q) * u[p + o];
    }
    u[p] = (f[p] - s) * __ldg(cf + 13 * Nc + q);
}

void launch3_relax27c(const Grid3 &g, const double *cf, const double *f, double *u, int nsweeps, cudaStream_t s)
{
    for (int sw = 0; sw < nsweeps; sw++) {
        const double *c = cf;
        for (int col = 0; col < 8; col++) {
            const Sub b = sub_of(g, col);
            if (b.cx * b.cy * b.cz == 0)
                continue;
            k3_relax27c<<<dim3((b.cx + 31) / 32, (b.cy + 3) / 4, b.cz), dim3(32, 4), 0, s>>>(g, b, c, f, u);
            c += 27LL * b.cx * b.cy * b.cz;
        }
    }
}


// ---------------------------------------------------------------- C1 on 7-point levels: one pass per sweep
// A red-black sweep u_out = GS(u_in) in ONE kernel.  A CTA owns a
// 64 x 8 column tile and a chunk of RB_KC planes and marches in z: at step k it
// updates the red points of plane k on the tile plus a one-point ring (their
// neighbours are old black values, read from u_in, which nobody writes), keeps
// them in a 4-plane shared ring, and after one barrier updates the black points of
// plane k-1 on the tile from the red values of planes k-2, k-1, k.  Ring red points
// are recomputed by every CTA that needs them, so no CTA waits for another; u_in
// is read-only and u_out written once, i.e. one pass over the level per sweep
// (the two colour launches read every array twice).  Same per-point expression as
// k3_relax7, so the iterate is that of the two-launch sweep.
constexpr int RB_TX = 64;

__device__ __forceinline__ double gs7(const Op3 &A, long long p, double f, double uw, double ue, double us, double un,
                                      double ub, double ut)
{
    const long long X = 1, Y = A.g.px, Z = A.g.ps;
    const double *W = A.a[12], *S = A.a[10], *B = A.a[4];
    const double s = W[p] * uw + W[p + X] * ue + S[p] * us + S[p + Y] * un + B[p] * ub + B[p + Z] * ut;
    return (f - s) * rcp_pos(A.O[p]);
}

template <int RB_TY, int RB_KC>
__global__ void __launch_bounds__(32 * RB_TY) k3_rb7(Op3 A, const double *__restrict__ f, const double *__restrict__ uin,
                                              double *__restrict__ uout)
{
    constexpr int RB_RX = RB_TX + 2, RB_RY = RB_TY + 2, NT = 32 * RB_TY;
    __shared__ double red[4][RB_RY][RB_RX];
    const int nx = A.g.nx, ny = A.g.ny, nz = A.g.nz;
    const long long Y = A.g.px, Z = A.g.ps;
    const int i0 = blockIdx.x * RB_TX + 1, j0 = blockIdx.y * RB_TY + 1;
    const int kb = blockIdx.z * RB_KC + 1, ke = min(kb + RB_KC, nz + 1);
    const int tid = threadIdx.y * 32 + threadIdx.x;
    for (int k = kb - 1; k <= ke; k++) {
        // red points of plane k on the tile + ring: 10 rows x 33 per row
        double(*rk)[RB_RX] = red[k & 3];
        for (int t = tid; t < RB_RY * (RB_RX / 2); t += NT) {
            const int row = t / (RB_RX / 2), c = t % (RB_RX / 2);
            const int j = j0 - 1 + row;
            const int ib = i0 - 1;
            const int i = ib + 2 * c + ((ib + j + k) & 1);
            double v = 0.0;
            if (k >= 1 && k <= nz && j >= 1 && j <= ny && i >= 1 && i <= nx) {
                const long long p = (long long)k * Z + (long long)j * Y + i;
                v = gs7(A, p, f[p], uin[p - 1], uin[p + 1], uin[p - Y], uin[p + Y], uin[p - Z], uin[p + Z]);
                if (k >= kb && k < ke && j >= j0 && j < j0 + RB_TY && i >= i0 && i < i0 + RB_TX)
                    uout[p] = v;
            }
            rk[row][i - ib] = v;  // black slots are never read
        }
        __syncthreads();
        const int kk = k - 1;
        if (kk >= kb && kk < ke) {
            const int j = j0 + threadIdx.y;
            const int ia = i0 + 2 * threadIdx.x;
            const int i = ia + ((ia + j + kk + 1) & 1);  // the black point of the pair (ia, ia+1)
            if (j <= ny && i <= nx) {
                const long long p = (long long)kk * Z + (long long)j * Y + i;
                const int r = threadIdx.y + 1, c = i - (i0 - 1);
                const double(*rm)[RB_RX] = red[kk & 3];
                uout[p] = gs7(A, p, f[p], rm[r][c - 1], rm[r][c + 1], rm[r - 1][c], rm[r + 1][c],
                              red[(kk - 1) & 3][r][c], red[(kk + 1) & 3][r][c]);
            }
        }
    }
}


// ---------------------------------------------------------------- k3_rb7t: the one-pass sweep fed by TMA
// k3_rb7's schedule with every input plane staged ONCE per CTA in shared memory by
// the tensor engine: one thread issues, per step, six 2-D tile boxes of (3-D tensor
// maps; out-of-range rows/columns/planes zero-filled) -- u_in(k+2), f/O/W/S(k+1),
// B(k+2) -- that land one step ahead on an mbarrier (complete_tx), so the 256 threads
// only compute (k3_rb7 re-read halo and next-plane data through L1/L2, 1.42x the
// arrays from DRAM; the cp.async variant was issue-bound, tools/archive/k3_rb7s.cu.txt).
namespace rbt {
constexpr int TX = 64, TY = 6, NT = 32 * TY;  // z-chunk (planes per CTA): planned per launch
constexpr int UX = TX + 6, UY = TY + 4;  // u_in box: origin (i0-3, j0-2) (TMA needs a 16-B aligned x start)
constexpr int RX = TX + 2, RY = TY + 2;  // f, O, B, red: origin (i0-1, j0-1)
constexpr int WX = TX + 4;               // W box: 68 wide (16-B multiple), origin (i0-1, j0-1)
constexpr int SY = TY + 3;               // S box: RX x 11
constexpr int al(int n) { return (n + 15) / 16 * 16; }  // 128-byte slots
constexpr int SU = al(UX * UY), SF = al(RX * RY), SW = al(WX * RY), SS = al(RX * SY), SR = RX * RY;
constexpr int OFF_U = 0, OFF_F = OFF_U + 4 * SU, OFF_O = OFF_F + 3 * SF, OFF_W = OFF_O + 3 * SF,
              OFF_S = OFF_W + 3 * SW, OFF_B = OFF_S + 3 * SS, OFF_R = OFF_B + 4 * SF, TOTAL = OFF_R + 4 * SR;
constexpr unsigned BU = UX * UY * 8, BF = RX * RY * 8, BW = WX * RY * 8, BS = RX * SY * 8;
}  // namespace rbt

struct Maps7 {
    CUtensorMap u, f, o, w, s, b;
};

__device__ __forceinline__ unsigned s32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void tma3(double *dst, const CUtensorMap *m, int x, int y, int z, unsigned long long *bar)
{
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];" ::"r"(s32(dst)),
        "l"(reinterpret_cast<unsigned long long>(m)), "r"(x), "r"(y), "r"(z), "r"(s32(bar))
        : "memory");
}

__device__ __forceinline__ void mb_expect(unsigned long long *bar, unsigned bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(bar)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mb_wait(unsigned long long *bar, unsigned parity)
{
    asm volatile(
        "{\n .reg .pred P1;\n RB7W:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        " @!P1 bra RB7W;\n}\n" ::"r"(s32(bar)),
        "r"(parity)
        : "memory");
}

template <bool RCP>
__global__ void __launch_bounds__(rbt::NT, 2) k3_rb7t(Op3 A, double *__restrict__ uout,
                                                      const __grid_constant__ Maps7 M, int KC)
{
    using namespace rbt;
    extern __shared__ __align__(1024) double sm[];
    unsigned long long *bar = reinterpret_cast<unsigned long long *>(sm + TOTAL);  // no static smem: slots stay 128-B aligned
    const Grid3 &G = A.g;
    const int nx = G.nx, ny = G.ny, nz = G.nz;
    const int i0 = blockIdx.x * TX + 1, j0 = blockIdx.y * TY + 1;
    const int kb = blockIdx.z * KC + 1, ke = min(kb + KC, nz + 1);
    const int tid = threadIdx.y * 32 + threadIdx.x;
    auto U_ = [&](int k) { return sm + OFF_U + (k & 3) * SU; };
    auto F_ = [&](int k) { return sm + OFF_F + ((k + 3) % 3) * SF; };
    auto O_ = [&](int k) { return sm + OFF_O + ((k + 3) % 3) * SF; };
    auto W_ = [&](int k) { return sm + OFF_W + ((k + 3) % 3) * SW; };
    auto S_ = [&](int k) { return sm + OFF_S + ((k + 3) % 3) * SS; };
    auto B_ = [&](int k) { return sm + OFF_B + (k & 3) * SF; };
    auto R_ = [&](int k) { return sm + OFF_R + (k & 3) * SR; };
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&bar[0])) : "memory");
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&bar[1])) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int xu = i0 - 3, yu = j0 - 2, xr = i0 - 1, yr = j0 - 1;  // even x starts (i0 = 64 bx + 1)
    if (tid == 0) {  // prologue: what step kb-1 reads (planes < 0 are zero-filled boxes)
        mb_expect(&bar[0], 3 * BU + 3 * BF + BW + BS + BF);
        for (int k = kb - 2; k <= kb; k++)
            tma3(U_(k), &M.u, xu, yu, k, &bar[0]);
        tma3(F_(kb - 1), &M.f, xr, yr, kb - 1, &bar[0]);
        tma3(O_(kb - 1), &M.o, xr, yr, kb - 1, &bar[0]);
        tma3(W_(kb - 1), &M.w, xr, yr, kb - 1, &bar[0]);
        tma3(S_(kb - 1), &M.s, xr, yr, kb - 1, &bar[0]);
        tma3(B_(kb - 1), &M.b, xr, yr, kb - 1, &bar[0]);
        tma3(B_(kb), &M.b, xr, yr, kb, &bar[0]);
    }
    mb_wait(&bar[0], 0);
    for (int k = kb - 1, st = 0; k <= ke; k++, st++) {
        if (tid == 0 && k < ke) {  // step st+1's new planes, one step ahead
            unsigned long long *b = &bar[(st + 1) & 1];
            mb_expect(b, BU + 3 * BF + BW + BS);
            tma3(U_(k + 2), &M.u, xu, yu, k + 2, b);
            tma3(F_(k + 1), &M.f, xr, yr, k + 1, b);
            tma3(O_(k + 1), &M.o, xr, yr, k + 1, b);
            tma3(W_(k + 1), &M.w, xr, yr, k + 1, b);
            tma3(S_(k + 1), &M.s, xr, yr, k + 1, b);
            tma3(B_(k + 2), &M.b, xr, yr, k + 2, b);
        }
        double *rk = R_(k);
        {
            const double *u0 = U_(k), *um = U_(k - 1), *up = U_(k + 1), *fk = F_(k), *ok = O_(k), *wk = W_(k),
                         *sk = S_(k), *bk = B_(k), *bp = B_(k + 1);
            const bool kin = k >= 1 && k <= nz;
            for (int t = tid; t < RY * (RX / 2); t += NT) {
                const int r = t / (RX / 2), cc = t % (RX / 2);
                const int j = j0 - 1 + r;
                const int c = 2 * cc + ((i0 - 1 + j + k) & 1), i = i0 - 1 + c;
                double v = 0.0;
                if (kin && j >= 1 && j <= ny && i >= 1 && i <= nx) {
                    const int q = r * RX + c, qc = (r + 1) * UX + (c + 2);  // (r+1, c+2) in u_in's box
                    const double s = wk[r * WX + c] * u0[qc - 1] + wk[r * WX + c + 1] * u0[qc + 1] +
                                     sk[r * RX + c] * u0[qc - UX] + sk[(r + 1) * RX + c] * u0[qc + UX] +
                                     bk[q] * um[qc] + bp[q] * up[qc];
                    v = (fk[q] - s) * (RCP ? ok[q] : rcp_pos(ok[q]));
                }
                rk[r * RX + c] = v;
            }
        }
        __syncthreads();
        const int kk = k - 1;
        if (kk >= kb && kk < ke) {
            const int j = j0 + threadIdx.y, r = threadIdx.y + 1;
            const int ia = i0 + 2 * threadIdx.x;
            const int par = (ia + j + kk + 1) & 1;  // 0: ia is black
            const int ib = ia + par, c = ib - (i0 - 1);
            const double *rm = R_(kk), *rl = R_(kk - 1), *rh = R_(kk + 1), *fk = F_(kk), *ok = O_(kk), *wk = W_(kk),
                         *sk = S_(kk), *bk = B_(kk), *bp = B_(kk + 1);
            const int q = r * RX + c;
            double vb = 0.0;
            if (j <= ny && ib <= nx) {
                const double s = wk[r * WX + c] * rm[q - 1] + wk[r * WX + c + 1] * rm[q + 1] +
                                 sk[r * RX + c] * rm[q - RX] + sk[(r + 1) * RX + c] * rm[q + RX] + bk[q] * rl[q] +
                                 bp[q] * rh[q];
                vb = (fk[q] - s) * (RCP ? ok[q] : rcp_pos(ok[q]));
            }
            if (j <= ny) {
                const long long p = (long long)kk * G.ps + (long long)j * G.px + ia;
                const int cr = ia - (i0 - 1);
                const double va = par ? rm[r * RX + cr] : vb, vn = par ? vb : rm[r * RX + cr + 1];
                if (ia <= nx)
                    uout[p] = va;
                if (ia + 1 <= nx)
                    uout[p + 1] = vn;
            }
        }
        if (k < ke)
            mb_wait(&bar[(st + 1) & 1], ((st + 1) >> 1) & 1);
        __syncthreads();
    }
}

static PFN_cuTensorMapEncodeTiled_v12000 encode3()
{
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
        cudaGetLastError();
    });
    return fn;
}

static bool map3(CUtensorMap *m, const double *base, const Grid3 &g, int bx, int by)
{
    auto fn = encode3();
    if (!fn)
        return false;
    cuuint64_t dims[3] = {(cuuint64_t)g.px, (cuuint64_t)(g.ny + 2), (cuuint64_t)(g.nz + 2)};
    cuuint64_t strides[2] = {(cuuint64_t)g.px * 8, (cuuint64_t)g.ps * 8};
    cuuint32_t box[3] = {(cuuint32_t)bx, (cuuint32_t)by, 1};
    cuuint32_t es[3] = {1, 1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, (void *)base, dims, strides, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// false: a tensor map could not be encoded (the caller falls back to k3_rb7)
bool launch3_rb7t(const Op3 &A, const double *f, const double *uin, double *uout, const double *ro, cudaStream_t s)
{
    using namespace rbt;
    Maps7 M;
    if (((uintptr_t)uin | (uintptr_t)f | (uintptr_t)(ro ? ro : A.O) | (uintptr_t)A.a[12] | (uintptr_t)A.a[10] |
         (uintptr_t)A.a[4]) & 15 || (A.g.px * 8) % 16 || (A.g.ps * 8) % 16)
        return false;
    if (!map3(&M.u, uin, A.g, UX, UY) || !map3(&M.f, f, A.g, RX, RY) || !map3(&M.o, ro ? ro : A.O, A.g, RX, RY) ||
        !map3(&M.w, A.a[12], A.g, WX, RY) || !map3(&M.s, A.a[10], A.g, RX, SY) || !map3(&M.b, A.a[4], A.g, RX, RY))
        return false;
    const size_t smem = sizeof(double) * TOTAL + 16;
    // z-chunk: the fewest waves x (planes + 2 warm-up) over 2 CTAs per SM (the 2-D planner's
    // model, DESIGN §5.2/§5.8): at 255^3 172 column tiles x 5 chunks of 51 planes = 3 waves
    // (a fixed 32 planes gave 8 chunks = 4.65 waves; measured 1.865 -> 1.831 ms per cycle)
    int sms = 148;
    {
        int dev = 0, v = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && v > 0)
            sms = v;
    }
    const long long cols = (long long)((A.g.nx + TX - 1) / TX) * ((A.g.ny + TY - 1) / TY), slots = 2LL * sms;
    int KC = A.g.nz, best_cost = INT_MAX;
    for (int nzc = 1; nzc <= A.g.nz; nzc++) {
        const int kc = (A.g.nz + nzc - 1) / nzc;
        const long long waves = (cols * ((A.g.nz + kc - 1) / kc) + slots - 1) / slots;
        const long long cost = waves * (kc + 2);
        if (cost < best_cost) {
            best_cost = (int)cost;
            KC = kc;
        }
    }
    dim3 grid((A.g.nx + TX - 1) / TX, (A.g.ny + TY - 1) / TY, (A.g.nz + KC - 1) / KC);
    if (ro) {
        cudaFuncSetAttribute(k3_rb7t<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k3_rb7t<true><<<grid, dim3(32, TY), smem, s>>>(A, uout, M, KC);
    } else {
        cudaFuncSetAttribute(k3_rb7t<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k3_rb7t<false><<<grid, dim3(32, TY), smem, s>>>(A, uout, M, KC);
    }
    return true;
}

// tile height x z-chunk: BMG3_RB="TY,KC" (a tuning knob read once; default measured)
static int rb_variant()
{
    static int v = -1;
    if (v < 0) {
        v = 7;  // the TMA-fed sweep (k3_rb7t); k3_rb7 16 x 32 if a tensor map cannot be encoded
        if (const char *e = getenv("BMG3_RB")) {
            int ty = 0, kc = 0;
            if (e[0] == 't')
                v = 7;
            else if (sscanf(e, "%d,%d", &ty, &kc) == 2)
                v = ty == 4 ? (kc == 32 ? 0 : 6) : ty == 8 ? (kc == 32 ? 1 : kc == 64 ? 2 : 3) : (kc == 32 ? 4 : 5);
        }
    }
    return v;
}

template <int TY, int KC>
static void rb7_launch(const Op3 &A, const double *f, const double *uin, double *uout, cudaStream_t s)
{
    dim3 grid((A.g.nx + RB_TX - 1) / RB_TX, (A.g.ny + TY - 1) / TY, (A.g.nz + KC - 1) / KC);
    k3_rb7<TY, KC><<<grid, dim3(32, TY), 0, s>>>(A, f, uin, uout);
}

// the reciprocal plane ro = rcp_pos(a_O) of a 7-point level (same value the sweeps form)
__global__ void k3_recip(Grid3 g, const double *__restrict__ O, double *__restrict__ ro)
{
    const int i = blockIdx.x * 32 + threadIdx.x + 1, j = blockIdx.y * 4 + threadIdx.y + 1, k = blockIdx.z + 1;
    if (i <= g.nx && j <= g.ny)
        ro[at3(g, i, j, k)] = rcp_pos(O[at3(g, i, j, k)]);
}

void launch3_recip(const Op3 &A, double *ro, cudaStream_t s)
{
    k3_recip<<<dim3((A.g.nx + 31) / 32, (A.g.ny + 3) / 4, A.g.nz), dim3(32, 4), 0, s>>>(A.g, A.O, ro);
}

void launch3_rb7(const Op3 &A, const double *f, const double *uin, double *uout, cudaStream_t s, const double *ro)
{
    if (rb_variant() == 7 && launch3_rb7t(A, f, uin, uout, ro, s))
        return;
    switch (rb_variant()) {
    case 0: rb7_launch<4, 32>(A, f, uin, uout, s); break;
    case 6: rb7_launch<4, 64>(A, f, uin, uout, s); break;
    case 2: rb7_launch<8, 64>(A, f, uin, uout, s); break;
    case 3: rb7_launch<8, 128>(A, f, uin, uout, s); break;
    case 4: rb7_launch<16, 32>(A, f, uin, uout, s); break;
    case 5: rb7_launch<16, 64>(A, f, uin, uout, s); break;
    case 1: rb7_launch<8, 32>(A, f, uin, uout, s); break;
    default: rb7_launch<16, 32>(A, f, uin, uout, s); break;  // 4, and 7's fallback
    }
}


// ---------------------------------------------------------------- C2 residual
template <int KIND>
__global__ void k3_residual(Op3 A, const double *__restrict__ f, const double *__restrict__ u, double *__restrict__ r)
{
    const int i = blockIdx.x * 32 + threadIdx.x + 1, j = blockIdx.y * 4 + threadIdx.y + 1, k = blockIdx.z + 1;
    if (i > A.g.nx || j > A.g.ny)
        return;
    const long long p = at3(A.g, i, j, k);
    r[p] = f[p] - (A.O[p] * u[p] + offdiag<KIND>(A, u, p));
}

void launch3_residual(const Op3 &A, const double *f, const double *u, double *r, cudaStream_t s)
{
    dim3 grid((A.g.nx + 31) / 32, (A.g.ny + 3) / 4, A.g.nz);
    if (A.kind == 7)
        k3_residual<7><<<grid, dim3(32, 4), 0, s>>>(A, f, u, r);
    else
        k3_residual<27><<<grid, dim3(32, 4), 0, s>>>(A, f, u, r);
}

// ---------------------------------------------------------------- C3 restriction (c21) + C4
// Gather at coarse C over the 27 fine points f = 2C + o: the weight of f toward C
// sits at coarse index Q = C + [o == +1] in slot slot_base(mask(o != 0)) + corner,
// corner bit = [o_d == -1] on each odd axis -- all compile-time per o.  Fine points
// on the ring contribute r = 0 (the ring of r is never written).
template <int E>
struct ROff {
    static constexpr int dx = E % 3 - 1, dy = (E / 3) % 3 - 1, dz = E / 9 - 1;
    static constexpr int m = (dx != 0) | (dy != 0) << 1 | (dz != 0) << 2;
    static constexpr int c0 = dx != 0 ? (dx == -1) : 0;
    static constexpr int nb0 = dx != 0;
    static constexpr int c1 = dy != 0 ? (dy == -1) << nb0 : 0;
    static constexpr int nb1 = nb0 + (dy != 0);
    static constexpr int c2 = dz != 0 ? (dz == -1) << nb1 : 0;
    static constexpr int slot = m == 0 ? -1 : slot_base(m) + c0 + c1 + c2;
};

template <int E>
__device__ __forceinline__ double rterm(const CI3 &ci, const Grid3 &fg, const double *__restrict__ r, int Ci, int Cj,
                                        int Ck)
{
    using O = ROff<E>;
    const double rv = r[at3(fg, 2 * Ci + O::dx, 2 * Cj + O::dy, 2 * Ck + O::dz)];
    if (O::m == 0)
        return rv;
    const double w = ci.w[O::slot][at3(ci.c, Ci + (O::dx == 1), Cj + (O::dy == 1), Ck + (O::dz == 1))];
    return w * rv;
}

template <int... Es>
__device__ __forceinline__ double rsum(const CI3 &ci, const Grid3 &fg, const double *__restrict__ r, int Ci, int Cj,
                                       int Ck, std::integer_sequence<int, Es...>)
{
    double s = 0.0;
    ((s += rterm<Es>(ci, fg, r, Ci, Cj, Ck)), ...);
    return s;
}

__global__ void k3_restrict(Grid3 fg, CI3 ci, const double *__restrict__ r, double *__restrict__ fc,
                            double *__restrict__ uc)
{
    const int Ci = blockIdx.x * 32 + threadIdx.x + 1, Cj = blockIdx.y * 4 + threadIdx.y + 1, Ck = blockIdx.z + 1;
    if (Ci > ci.c.nx || Cj > ci.c.ny)
        return;
    const double s = rsum(ci, fg, r, Ci, Cj, Ck, std::make_integer_sequence<int, 27>{});
    const long long pc = at3(ci.c, Ci, Cj, Ck);
    fc[pc] = s;
    if (uc)
        uc[pc] = 0.0;
}

void launch3_restrict(const Op3 &A, const CI3 &ci, const double *r, double *fc, double *uc, cudaStream_t s)
{
    dim3 grid((ci.c.nx + 31) / 32, (ci.c.ny + 3) / 4, ci.c.nz);
    k3_restrict<<<grid, dim3(32, 4), 0, s>>>(A.g, ci, r, fc, uc);
}

// ---------------------------------------------------------------- C6 interpolation + correction (c21)
// One thread per coarse cell (I,J,K): the eight fine points (2I-1..2I) x (2J-1..2J) x
// (2K-1..2K) share the weight index Q = (I,J,K) and the eight coarse corners, so every
// e value and weight is loaded once.  u(f) += sum_c w_c e(C_c), corners in the
// oracle's order (x fastest), no contraction -> bitwise the oracle's update.
template <int M>
__device__ __forceinline__ void iterm(const CI3 &ci, const double (&e)[8], long long q, const double *uin,
                                      double *u, long long p)
{
    constexpr int ox = M & 1, oy = (M >> 1) & 1, oz = (M >> 2) & 1;
    double s;
    if (M == 0) {
        s = __dmul_rn(1.0, e[7]);
    } else {
        constexpr int nc = 1 << (ox + oy + oz);
        s = 0.0;
#pragma unroll
        for (int c = 0; c < nc; c++) {
            int b = 0, cx = 1, cy = 1, cz = 1;  // corner coordinate: 1 = upper (I), 0 = lower (I-1)
            if (ox)
                cx = (c >> b++) & 1;
            if (oy)
                cy = (c >> b++) & 1;
            if (oz)
                cz = (c >> b++) & 1;
            s = __dadd_rn(s, __dmul_rn(ci.w[slot_base(M) + c][q], e[cz * 4 + cy * 2 + cx]));
        }
    }
    u[p] = __dadd_rn(uin[p], s);
}

__device__ __forceinline__ void interp_cell(const Grid3 &fg, const CI3 &ci, const double *__restrict__ ec,
                                            const double *uin, double *u, int I, int J, int K)
{
    const long long q = at3(ci.c, I, J, K);
    const long long X = 1, Y = ci.c.px, Z = ci.c.ps;
    const double e[8] = {ec[q - Z - Y - X], ec[q - Z - Y], ec[q - Z - X], ec[q - Z],
                         ec[q - Y - X],     ec[q - Y],     ec[q - X],     ec[q]};
    const int i1 = 2 * I - 1, j1 = 2 * J - 1, k1 = 2 * K - 1;
    const bool xe = 2 * I <= fg.nx, ye = 2 * J <= fg.ny, ze = 2 * K <= fg.nz;
    const long long p = at3(fg, i1, j1, k1), FY = fg.px, FZ = fg.ps;
    // fine (i1 + a, j1 + b, k1 + c): odd coordinate where the offset is 0
    iterm<7>(ci, e, q, uin, u, p);
    if (xe)
        iterm<6>(ci, e, q, uin, u, p + 1);
    if (ye)
        iterm<5>(ci, e, q, uin, u, p + FY);
    if (xe && ye)
        iterm<4>(ci, e, q, uin, u, p + FY + 1);
    if (ze) {
        iterm<3>(ci, e, q, uin, u, p + FZ);
        if (xe)
            iterm<2>(ci, e, q, uin, u, p + FZ + 1);
        if (ye)
            iterm<1>(ci, e, q, uin, u, p + FZ + FY);
        if (xe && ye)
            iterm<0>(ci, e, q, uin, u, p + FZ + FY + 1);
    }
}

__global__ void k3_interp_add(Grid3 fg, CI3 ci, const double *__restrict__ ec, const double *uin, double *u)
{
    const int I = blockIdx.x * 32 + threadIdx.x + 1, J = blockIdx.y * 4 + threadIdx.y + 1, K = blockIdx.z + 1;
    if (2 * I - 1 > fg.nx || 2 * J - 1 > fg.ny)
        return;
    interp_cell(fg, ci, ec, uin, u, I, J, K);
}

void launch3_interp_add(const Grid3 &fine, const CI3 &ci, const double *ec, const double *uin, double *u,
                        cudaStream_t s)
{
    const int hx = (fine.nx + 1) / 2, hy = (fine.ny + 1) / 2, hz = (fine.nz + 1) / 2;
    dim3 grid((hx + 31) / 32, (hy + 3) / 4, hz);
    k3_interp_add<<<grid, dim3(32, 4), 0, s>>>(fine, ci, ec, uin, u);
}


// ---------------------------------------------------------------- C7 residual norm (fixed-tree, deterministic)
constexpr int NT3 = 256;

int norm3_partials(const Grid3 &g)
{
    const long long n = (long long)g.nx * g.ny * g.nz;
    long long b = (n + NT3 - 1) / NT3;
    return (int)(b < 1024 ? (b < 1 ? 1 : b) : 1024);
}

template <int KIND>
__global__ void k3_norm_partial(Op3 A, Grid3 g, const double *__restrict__ f, const double *__restrict__ u,
                                double *__restrict__ partials)
{
    __shared__ double sh[NT3];
    const long long n = (long long)g.nx * g.ny * g.nz;
    double acc = 0.0;
    for (long long t = (long long)blockIdx.x * NT3 + threadIdx.x; t < n; t += (long long)gridDim.x * NT3) {
        const int i = (int)(t % g.nx) + 1, j = (int)((t / g.nx) % g.ny) + 1, k = (int)(t / ((long long)g.nx * g.ny)) + 1;
        const long long p = at3(g, i, j, k);
        double v = f[p];
        if (KIND != 0)
            v -= A.O[p] * u[p] + offdiag<KIND>(A, u, p);
        acc += v * v;
    }
    sh[threadIdx.x] = acc;
    __syncthreads();
    for (int w = NT3 / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w)
            sh[threadIdx.x] += sh[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0)
        partials[blockIdx.x] = sh[0];
}

__global__ void k3_norm_final(const double *__restrict__ partials, int n, double *result)
{
    __shared__ double sh[1024];
    sh[threadIdx.x] = threadIdx.x < n ? partials[threadIdx.x] : 0.0;
    __syncthreads();
    for (int w = 512; w > 0; w >>= 1) {
        if (threadIdx.x < w)
            sh[threadIdx.x] += sh[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0)
        *result = sqrt(sh[0]);
}

void launch3_resid_norm(const Op3 *A, const Grid3 &g, const double *f, const double *u, double *partials,
                        double *result, cudaStream_t s)
{
    const int nb = norm3_partials(g);
    Op3 dummy{};
    if (!A)
        k3_norm_partial<0><<<nb, NT3, 0, s>>>(dummy, g, f, u, partials);
    else if (A->kind == 7)
        k3_norm_partial<7><<<nb, NT3, 0, s>>>(*A, g, f, u, partials);
    else
        k3_norm_partial<27><<<nb, NT3, 0, s>>>(*A, g, f, u, partials);
    k3_norm_final<<<1, 1024, 0, s>>>(partials, nb, result);
}

__global__ void k3_zero_interior(Grid3 g, double *x)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x + 1, j = blockIdx.y + 1, k = blockIdx.z + 1;
    if (i <= g.nx)
        x[at3(g, i, j, k)] = 0.0;
}

void launch3_zero_interior(const Grid3 &g, double *x, cudaStream_t s)
{
    dim3 grid((g.nx + 127) / 128, g.ny, g.nz);
    k3_zero_interior<<<grid, 128, 0, s>>>(g, x);
}

}  // namespace bmg3
