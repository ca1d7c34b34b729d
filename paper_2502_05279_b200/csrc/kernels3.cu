// kernels3.cu -- the 3-D BoxMG kernels (DESIGN.md §3
// c16-c24, §5.8): stencil ingest, operator-induced interpolation, Galerkin
// RAP, coarsest dense factor/solve, multicolour point Gauss-Seidel, residual,
// restriction, interpolation-correction and the residual norm.  One thread per
// point (x fastest, so every warp reads consecutive doubles of a row).
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

// ---------------------------------------------------------------- C2 residual
template <int KIND>
__global__ void k3_residual(Op3 A, const double *__restrict__ f, const double *__restrict__ u, double *__restrict__ r)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x + 1, j = blockIdx.y + 1, k = blockIdx.z + 1;
    if (i > A.g.nx)
        return;
    const long long p = at3(A.g, i, j, k);
    r[p] = f[p] - (A.O[p] * u[p] + offdiag<KIND>(A, u, p));
}

void launch3_residual(const Op3 &A, const double *f, const double *u, double *r, cudaStream_t s)
{
    dim3 grid((A.g.nx + 127) / 128, A.g.ny, A.g.nz);
    if (A.kind == 7)
        k3_residual<7><<<grid, 128, 0, s>>>(A, f, u, r);
    else
        k3_residual<27><<<grid, 128, 0, s>>>(A, f, u, r);
}

// ---------------------------------------------------------------- C3 restriction (c21) + C4
__global__ void k3_restrict(Grid3 fg, CI3 ci, const double *__restrict__ r, double *__restrict__ fc,
                            double *__restrict__ uc)
{
    const int Ci = blockIdx.x * blockDim.x + threadIdx.x + 1, Cj = blockIdx.y + 1, Ck = blockIdx.z + 1;
    if (Ci > ci.c.nx)
        return;
    double s = 0.0;
    for (int e = 0; e < 27; e++) {
        const int fi = 2 * Ci + e % 3 - 1, fj = 2 * Cj + (e / 3) % 3 - 1, fk = 2 * Ck + e / 9 - 1;
        if (!inside3(fg, fi, fj, fk))
            continue;
        s += pw3(ci, fi, fj, fk, Ci, Cj, Ck) * r[at3(fg, fi, fj, fk)];
    }
    const long long pc = at3(ci.c, Ci, Cj, Ck);
    fc[pc] = s;
    if (uc)
        uc[pc] = 0.0;
}

void launch3_restrict(const Op3 &A, const CI3 &ci, const double *r, double *fc, double *uc, cudaStream_t s)
{
    dim3 grid((ci.c.nx + 127) / 128, ci.c.ny, ci.c.nz);
    k3_restrict<<<grid, 128, 0, s>>>(A.g, ci, r, fc, uc);
}

// ---------------------------------------------------------------- C6 interpolation + correction (c21)
// u(f) += sum_c w_c e(C_c), corners in the oracle's order (x fastest), no contraction
__global__ void k3_interp_add(Grid3 fg, CI3 ci, const double *__restrict__ ec, double *__restrict__ u)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x + 1, j = blockIdx.y + 1, k = blockIdx.z + 1;
    if (i > fg.nx)
        return;
    const int odd[3] = {i & 1, j & 1, k & 1};
    const int m = odd[0] | odd[1] << 1 | odd[2] << 2;
    const long long p = at3(fg, i, j, k);
    double s;
    if (m == 0) {
        s = __dmul_rn(1.0, ec[at3(ci.c, i >> 1, j >> 1, k >> 1)]);
    } else {
        const int Q[3] = {odd[0] ? (i + 1) >> 1 : i >> 1, odd[1] ? (j + 1) >> 1 : j >> 1,
                          odd[2] ? (k + 1) >> 1 : k >> 1};
        const long long q = at3(ci.c, Q[0], Q[1], Q[2]);
        const int base = slot_base(m), nc = 1 << __popc(m);
        s = 0.0;
        for (int c = 0; c < nc; c++) {
            int C[3] = {Q[0], Q[1], Q[2]}, nb = 0;
#pragma unroll
            for (int d = 0; d < 3; d++)
                if (odd[d]) {
                    if (!((c >> nb) & 1))
                        C[d] -= 1;
                    nb++;
                }
            s = __dadd_rn(s, __dmul_rn(ci.w[base + c][q], ec[at3(ci.c, C[0], C[1], C[2])]));
        }
    }
    u[p] = __dadd_rn(u[p], s);
}

void launch3_interp_add(const Grid3 &fine, const CI3 &ci, const double *ec, double *u, cudaStream_t s)
{
    dim3 grid((fine.nx + 127) / 128, fine.ny, fine.nz);
    k3_interp_add<<<grid, 128, 0, s>>>(fine, ci, ec, u);
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
