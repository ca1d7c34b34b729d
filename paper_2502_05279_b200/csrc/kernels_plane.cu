// kernels_plane.cu -- zebra xy-plane relaxation of the 3-D path (DESIGN.md §3
// c23, §5.8; fig:vcycle_flowchart's "Plane" box; "performance
// optimizations for operations such as plane relaxation").
//
// The planes of one colour (k = k0, k0+2, ...) are independent 2-D problems
// A_kk u_k = f_k - sum_{dz = +-1} A u: every kernel here works on the whole
// batch at once (blockIdx.z = plane), so a 2-D level of all planes is one
// launch however small each plane is.  The 2-D method is the repo's 2-D
// reading (c3 interpolation, c4 Galerkin, c6 colours, c5/c7 transfers, c8
// Cholesky) on the in-plane 9-point part of the 3-D operator.
#include "bmg3.cuh"
#include "bmg_internal.cuh"

namespace bmg3 {

using bmg::rcp_pos;

__device__ __forceinline__ bool inside2(const Grid3 &g, int i, int j) { return i >= 1 && i <= g.nx && j >= 1 && j <= g.ny; }

// the full 9-entry in-plane row at p
struct R9 {
    double sw, s, se, w, o, e, nw, n, ne;
};

__device__ __forceinline__ R9 rowP(const OpP &A, long long p)
{
    const long long Y = A.g.px;
    R9 a;
    a.o = A.O[p];
    a.w = A.W[p];
    a.e = A.W[p + 1];
    a.s = A.S[p];
    a.n = A.S[p + Y];
    if (A.kind == 9) {
        a.sw = A.SW[p];
        a.se = A.SE[p];
        a.nw = A.SE[p + Y - 1];
        a.ne = A.SW[p + Y + 1];
    } else {
        a.sw = a.se = a.nw = a.ne = 0.0;
    }
    return a;
}

__device__ __forceinline__ double offP(const R9 &a, const double *__restrict__ u, long long p, long long Y)
{
    return a.sw * u[p - Y - 1] + a.s * u[p - Y] + a.se * u[p - Y + 1] + a.w * u[p - 1] + a.e * u[p + 1] +
           a.nw * u[p + Y - 1] + a.n * u[p + Y] + a.ne * u[p + Y + 1];
}


// The two substitutions by ONE warp for n <= 32 unknowns (lane i holds b_i, x_k
// broadcast by a shuffle): the CTA loops pay two barriers per unknown.  Same
// operations in the same order as the CTA loops, so the same result.
__device__ __forceinline__ double warp_chol_solve(const double *__restrict__ L, int n, double b)
{
    const int i = threadIdx.x & 31;
    for (int k = 0; k < n; k++) {
        const double bk = __shfl_sync(0xffffffffu, b, k) / L[(long long)k * n + k];
        if (i == k)
            b = bk;
        else if (i > k && i < n)
            b -= L[(long long)i * n + k] * bk;
    }
    for (int k = n - 1; k >= 0; k--) {
        const double bk = __shfl_sync(0xffffffffu, b, k) / L[(long long)k * n + k];
        if (i == k)
            b = bk;
        else if (i < k)
            b -= L[(long long)k * n + i] * bk;
    }
    return b;
}

// ---------------------------------------------------------------- plane right-hand side (3-D)
// g = f - sum over the dz = -1, +1 couplings of A u, on the planes of the batch
template <int KIND>
__global__ void k3_plane_rhs(Op3 A, const double *__restrict__ f, const double *__restrict__ u, double *__restrict__ g,
                             Batch bt)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x + 1, j = blockIdx.y + 1, k = bt.k0 + 2 * blockIdx.z;
    if (i > A.g.nx)
        return;
    const long long Y = A.g.px, Z = A.g.ps;
    const long long p = (long long)k * Z + (long long)j * Y + i;
    double s;
    if (KIND == 7) {
        s = A.a[4][p] * u[p - Z] + A.a[4][p + Z] * u[p + Z];
    } else {
        s = 0.0;
#pragma unroll
        for (int e = 0; e < 9; e++) {
            const long long o = -Z + (long long)((e / 3) - 1) * Y + (e % 3 - 1);
            s += A.a[e][p] * u[p + o] + A.a[e][p - o] * u[p - o];
        }
    }
    g[p] = f[p] - s;
}

void launch3_plane_rhs(const Op3 &A, const double *f, const double *u, double *g, Batch b, cudaStream_t s)
{
    dim3 grid((A.g.nx + 127) / 128, A.g.ny, b.nb);
    if (A.kind == 7)
        k3_plane_rhs<7><<<grid, 128, 0, s>>>(A, f, u, g, b);
    else
        k3_plane_rhs<27><<<grid, 128, 0, s>>>(A, f, u, g, b);
}

// ---------------------------------------------------------------- c3 on every plane (setup)
// the 2-D oracle's expressions in its order, no contraction
__global__ void kP_interp(OpP A, CIP ci, double *w0, double *w1, double *w2, double *w3, double *w4, double *w5,
                          double *w6, double *w7, int phase, int *err)
{
    double *const wo[8] = {w0, w1, w2, w3, w4, w5, w6, w7};
    const int I = blockIdx.x * blockDim.x + threadIdx.x + 1, J = blockIdx.y + 1, k = blockIdx.z + 1;
    const long long Y = A.g.px;
    for (int t = 0; t < (phase == 1 ? 2 : 1); t++) {
        int i, j;
        if (phase == 1) {
            if (t == 0) {  // X at (2I-1, 2J)
                i = 2 * I - 1;
                j = 2 * J;
            } else {  // Y at (2I, 2J-1)
                i = 2 * I;
                j = 2 * J - 1;
            }
        } else {  // Z at (2I-1, 2J-1)
            i = 2 * I - 1;
            j = 2 * J - 1;
        }
        if (i > A.g.nx || j > A.g.ny)
            continue;
        const long long p = (long long)k * A.g.ps + (long long)j * Y + i;
        const R9 a = rowP(A, p);
        const double cW = -__dadd_rn(__dadd_rn(a.w, a.nw), a.sw);
        const double cE = -__dadd_rn(__dadd_rn(a.e, a.ne), a.se);
        const double cS = -__dadd_rn(__dadd_rn(a.s, a.sw), a.se);
        const double cN = -__dadd_rn(__dadd_rn(a.n, a.nw), a.ne);
        double sg = __dadd_rn(a.sw, a.s);
        sg = __dadd_rn(sg, a.se);
        sg = __dadd_rn(sg, a.w);
        sg = __dadd_rn(sg, a.e);
        sg = __dadd_rn(sg, a.nw);
        sg = __dadd_rn(sg, a.n);
        sg = __dadd_rn(sg, a.ne);
        const double sig = -sg;
        const double R = __dsub_rn(a.o, sig);
        const long long c = (long long)k * ci.c.ps;
        if (phase == 1 && t == 0) {
            const double eps = __ddiv_rn(fmin(fabs(cW), fabs(cE)), a.o);
            const double den = __dadd_rn(__dadd_rn(cW, cE), R > __dmul_rn(eps, sig) ? R : 0.0);
            if (!(den > 0.0)) {
                atomicOr(err, bmg::ERR_DEN);
                continue;
            }
            const long long q = c + (long long)J * ci.c.px + I;
            wo[P_LL][q] = __ddiv_rn(cW, den);
            wo[P_LR][q] = __ddiv_rn(cE, den);
        } else if (phase == 1) {
            const double eps = __ddiv_rn(fmin(fabs(cS), fabs(cN)), a.o);
            const double den = __dadd_rn(__dadd_rn(cS, cN), R > __dmul_rn(eps, sig) ? R : 0.0);
            if (!(den > 0.0)) {
                atomicOr(err, bmg::ERR_DEN);
                continue;
            }
            const long long q = c + (long long)J * ci.c.px + I;
            wo[P_LB][q] = __ddiv_rn(cS, den);
            wo[P_LA][q] = __ddiv_rn(cN, den);
        } else {
            const double eps = __ddiv_rn(fmin(fmin(fabs(cW), fabs(cE)), fmin(fabs(cS), fabs(cN))), a.o);
            const double den = __dadd_rn(sig, R > __dmul_rn(eps, sig) ? R : 0.0);
            if (!(den > 0.0)) {
                atomicOr(err, bmg::ERR_DEN);
                continue;
            }
            const long long qIJ = c + (long long)J * ci.c.px + I, qIm = qIJ - 1, qJm = qIJ - ci.c.px;
            const double lne = __ddiv_rn(
                __dsub_rn(__dsub_rn(-a.ne, __dmul_rn(a.n, ci.w[P_LR][qIJ])), __dmul_rn(a.e, ci.w[P_LA][qIJ])), den);
            const double lnw = __ddiv_rn(
                __dsub_rn(__dsub_rn(-a.nw, __dmul_rn(a.n, ci.w[P_LL][qIJ])), __dmul_rn(a.w, ci.w[P_LA][qIm])), den);
            const double lse = __ddiv_rn(
                __dsub_rn(__dsub_rn(-a.se, __dmul_rn(a.s, ci.w[P_LR][qJm])), __dmul_rn(a.e, ci.w[P_LB][qIJ])), den);
            const double lsw = __ddiv_rn(
                __dsub_rn(__dsub_rn(-a.sw, __dmul_rn(a.s, ci.w[P_LL][qJm])), __dmul_rn(a.w, ci.w[P_LB][qIm])), den);
            wo[P_LNE][qIJ] = lne;
            wo[P_LNW][qIJ] = lnw;
            wo[P_LSE][qIJ] = lse;
            wo[P_LSW][qIJ] = lsw;
        }
    }
}

void launchP_interp(const OpP &A, double *const ci[8], const Grid3 &cg, int *err, cudaStream_t s)
{
    CIP v;
    v.c = cg;
    for (int q = 0; q < 8; q++)
        v.w[q] = ci[q];
    const int hx = (A.g.nx + 1) / 2, hy = (A.g.ny + 1) / 2;
    dim3 grid((hx + 63) / 64, hy, A.g.nz);
    for (int phase = 1; phase <= 2; phase++)
        kP_interp<<<grid, 64, 0, s>>>(A, v, ci[0], ci[1], ci[2], ci[3], ci[4], ci[5], ci[6], ci[7], phase, err);
}

// P(q, C) on a plane (c7 naming: LL/LR toward I-1/I for X, LB/LA toward J-1/J for Y,
// LSW/LSE/LNW/LNE for Z)
__device__ __forceinline__ double pwP(const CIP &ci, long long ck, int qi, int qj, int Ci, int Cj)
{
    const int oi = qi & 1, oj = qj & 1;
    if (!oi && !oj)
        return (qi >> 1) == Ci && (qj >> 1) == Cj ? 1.0 : 0.0;
    const int I = oi ? (qi + 1) >> 1 : qi >> 1, J = oj ? (qj + 1) >> 1 : qj >> 1;
    const long long q = ck + (long long)J * ci.c.px + I;
    if (oi && !oj) {
        if (Cj != J)
            return 0.0;
        return Ci == I - 1 ? ci.w[P_LL][q] : Ci == I ? ci.w[P_LR][q] : 0.0;
    }
    if (!oi && oj) {
        if (Ci != I)
            return 0.0;
        return Cj == J - 1 ? ci.w[P_LB][q] : Cj == J ? ci.w[P_LA][q] : 0.0;
    }
    if (Ci == I - 1 && Cj == J - 1)
        return ci.w[P_LSW][q];
    if (Ci == I && Cj == J - 1)
        return ci.w[P_LSE][q];
    if (Ci == I - 1 && Cj == J)
        return ci.w[P_LNW][q];
    if (Ci == I && Cj == J)
        return ci.w[P_LNE][q];
    return 0.0;
}

// ---------------------------------------------------------------- c4 on every plane (setup)
// coarse stored entries: O (0,0), W (-1,0), S (0,-1), SW (-1,-1), SE (+1,-1)
__global__ void kP_rap(OpP A, CIP ci, double *dO, double *dW, double *dS, double *dSW, double *dSE)
{
    const int Ci = blockIdx.x * blockDim.x + threadIdx.x + 1, Cj = blockIdx.y + 1, k = blockIdx.z + 1;
    if (Ci > ci.c.nx)
        return;
    const long long Y = A.g.px, fk = (long long)k * A.g.ps, ck = (long long)k * ci.c.ps;
    double aO = 0.0, aW = 0.0, aS = 0.0, aSW = 0.0, aSE = 0.0;
    for (int o1 = 0; o1 < 9; o1++) {
        const int fi = 2 * Ci + o1 % 3 - 1, fj = 2 * Cj + o1 / 3 - 1;
        if (!inside2(A.g, fi, fj))
            continue;
        const double w1 = pwP(ci, ck, fi, fj, Ci, Cj);
        if (w1 == 0.0)
            continue;
        const long long pf = fk + (long long)fj * Y + fi;
        const R9 a = rowP(A, pf);
        const double av[9] = {a.sw, a.s, a.se, a.w, a.o, a.e, a.nw, a.n, a.ne};
        for (int e = 0; e < 9; e++) {
            const int gi = fi + e % 3 - 1, gj = fj + e / 3 - 1;
            if (av[e] == 0.0 || !inside2(A.g, gi, gj))
                continue;
            const double wa = w1 * av[e];
            const int lo0 = (gi & 1) ? (gi + 1) / 2 - 1 : gi / 2, hi0 = (gi & 1) ? (gi + 1) / 2 : gi / 2;
            const int lo1 = (gj & 1) ? (gj + 1) / 2 - 1 : gj / 2, hi1 = (gj & 1) ? (gj + 1) / 2 : gj / 2;
            for (int Dj = lo1; Dj <= hi1; Dj++)
                for (int Di = lo0; Di <= hi0; Di++) {
                    if (!inside2(ci.c, Di, Dj))
                        continue;
                    const int dx = Di - Ci, dy = Dj - Cj;
                    double *acc = nullptr;
                    if (dy == 0 && dx == 0)
                        acc = &aO;
                    else if (dy == 0 && dx == -1)
                        acc = &aW;
                    else if (dy == -1 && dx == 0)
                        acc = &aS;
                    else if (dy == -1 && dx == -1)
                        acc = &aSW;
                    else if (dy == -1 && dx == 1)
                        acc = &aSE;
                    if (!acc)
                        continue;
                    *acc += wa * pwP(ci, ck, gi, gj, Di, Dj);
                }
        }
    }
    const long long pc = ck + (long long)Cj * ci.c.px + Ci;
    dO[pc] = aO;
    dW[pc] = aW;
    dS[pc] = aS;
    dSW[pc] = aSW;
    dSE[pc] = aSE;
}

void launchP_rap(const OpP &A, const CIP &ci, double *const dst[5], cudaStream_t s)
{
    dim3 grid((ci.c.nx + 63) / 64, ci.c.ny, A.g.nz);
    kP_rap<<<grid, 64, 0, s>>>(A, ci, dst[0], dst[1], dst[2], dst[3], dst[4]);
}

// ---------------------------------------------------------------- c8 per plane: dense Cholesky (setup)
// one CTA per plane k = 1..nz: assemble (lexicographic, x fastest) then factor in place
__global__ void kP_assemble_chol(OpP A, double *Lall, int *err)
{
    const int k = blockIdx.x + 1, nx = A.g.nx, n = nx * A.g.ny;
    double *M = Lall + (long long)(k - 1) * n * n;
    for (long long t = threadIdx.x; t < (long long)n * n; t += blockDim.x)
        M[t] = 0.0;
    __syncthreads();
    for (int r = threadIdx.x; r < n; r += blockDim.x) {
        const int i = r % nx + 1, j = r / nx + 1;
        const R9 a = rowP(A, (long long)k * A.g.ps + (long long)j * A.g.px + i);
        const double av[9] = {a.sw, a.s, a.se, a.w, a.o, a.e, a.nw, a.n, a.ne};
        for (int e = 0; e < 9; e++) {
            const int qi = i + e % 3 - 1, qj = j + e / 3 - 1;
            if (inside2(A.g, qi, qj))
                M[(long long)r * n + (qj - 1) * nx + (qi - 1)] = av[e];
        }
    }
    __syncthreads();
    __shared__ double piv;
    for (int c = 0; c < n; c++) {
        if (threadIdx.x == 0) {
            double d = M[(long long)c * n + c];
            if (!(d > 0.0)) {
                atomicOr(err, bmg::ERR_PIVOT);
                d = 1.0;
            }
            piv = sqrt(d);
            M[(long long)c * n + c] = piv;
        }
        __syncthreads();
        for (int r = c + 1 + threadIdx.x; r < n; r += blockDim.x)
            M[(long long)r * n + c] /= piv;
        __syncthreads();
        const long long m = n - c - 1;
        for (long long t = threadIdx.x; t < m * m; t += blockDim.x) {
            const int r = c + 1 + (int)(t / m), q = c + 1 + (int)(t % m);
            if (q <= r)
                M[(long long)r * n + q] -= M[(long long)r * n + c] * M[(long long)q * n + c];
        }
        __syncthreads();
    }
}

void launchP_assemble_chol(const OpP &A, double *L, int *err, cudaStream_t s)
{
    kP_assemble_chol<<<A.g.nz, 256, 0, s>>>(A, L, err);
}

// ---------------------------------------------------------------- c6 on the planes of a batch
template <int KIND>
__global__ void kP_relax(OpP A, const double *__restrict__ f, double *__restrict__ u, Batch bt, int colour)
{
    const int k = bt.k0 + 2 * blockIdx.z;
    int i, j;
    if (KIND == 5) {
        j = blockIdx.y + 1;
        i = (((colour + j) & 1) ? 1 : 2) + 2 * (blockIdx.x * blockDim.x + threadIdx.x);
    } else {
        i = ((colour & 1) ? 1 : 2) + 2 * (blockIdx.x * blockDim.x + threadIdx.x);
        j = ((colour & 2) ? 1 : 2) + 2 * blockIdx.y;
    }
    if (i > A.g.nx || j > A.g.ny)
        return;
    const long long p = (long long)k * A.g.ps + (long long)j * A.g.px + i;
    const R9 a = rowP(A, p);
    u[p] = (f[p] - offP(a, u, p, A.g.px)) * rcp_pos(a.o);
}

// 5-point plane levels (the in-plane part of a 7-point level): a red-black sweep
// uout = GS(uin) in ONE pass over the colour's planes -- the 2-D form of k3_rb7: a CTA
// owns a strip of 256 points, 32 rows and one plane, marches up the rows (red of row j
// on the strip plus a one-point ring from uin, a barrier, black of row j-1 from the
// 4-row shared ring, row j-1 written out whole).  Same per-point expression as
// kP_relax<5> (offP with the zero corner terms).
constexpr int PRB_NT = 128, PRB_TX = 2 * PRB_NT, PRB_RC = 32;

__device__ __forceinline__ double offP_v(const R9 &a, double sw, double s, double se, double w, double e, double nw,
                                         double n, double ne)
{
    return a.sw * sw + a.s * s + a.se * se + a.w * w + a.e * e + a.nw * nw + a.n * n + a.ne * ne;
}

__global__ void __launch_bounds__(PRB_NT) kP_rb5(OpP A, const double *__restrict__ f, const double *__restrict__ uin,
                                                 double *__restrict__ uout, Batch bt)
{
    __shared__ double red[4][PRB_TX + 2];
    const int k = bt.k0 + 2 * blockIdx.z, nx = A.g.nx, ny = A.g.ny;
    const long long Y = A.g.px, base = (long long)k * A.g.ps;
    const int i0 = blockIdx.x * PRB_TX + 1, jb = blockIdx.y * PRB_RC + 1, je = min(jb + PRB_RC, ny + 1);
    const int tid = threadIdx.x;
    for (int j = jb - 1; j <= je; j++) {
        double *rj = red[j & 3];
        for (int t = tid; t <= PRB_NT; t += PRB_NT) {
            const int i = i0 - 1 + 2 * t + ((i0 - 1 + j) & 1);
            double v = 0.0;
            if (j >= 1 && j <= ny && i >= 1 && i <= nx) {
                const long long p = base + (long long)j * Y + i;
                const R9 a = rowP(A, p);
                v = (f[p] - offP_v(a, uin[p - Y - 1], uin[p - Y], uin[p - Y + 1], uin[p - 1], uin[p + 1],
                                   uin[p + Y - 1], uin[p + Y], uin[p + Y + 1])) *
                    rcp_pos(a.o);
            }
            if (i - (i0 - 1) < PRB_TX + 2)
                rj[i - (i0 - 1)] = v;
        }
        __syncthreads();
        const int jj = j - 1;
        if (jj >= jb && jj < je) {
            const int ia = i0 + 2 * tid;
            const int ib = ia + (((ia + jj) & 1) ? 0 : 1), ir = ib == ia ? ia + 1 : ia;  // black, red of the pair
            const double *rl = red[(jj - 1) & 3], *rm = red[jj & 3], *rh = red[j & 3];
            const long long row = base + (long long)jj * Y;
            if (ib <= nx) {
                const long long p = row + ib;
                const int x = ib - (i0 - 1);
                const R9 a = rowP(A, p);
                uout[p] = (f[p] - offP_v(a, 0.0, rl[x], 0.0, rm[x - 1], rm[x + 1], 0.0, rh[x], 0.0)) * rcp_pos(a.o);
            }
            if (ir <= nx)
                uout[row + ir] = rm[ir - (i0 - 1)];
        }
    }
}

void launchP_rb5(const OpP &A, const double *f, const double *uin, double *uout, Batch b, cudaStream_t s)
{
    dim3 grid((A.g.nx + PRB_TX - 1) / PRB_TX, (A.g.ny + PRB_RC - 1) / PRB_RC, b.nb);
    kP_rb5<<<grid, PRB_NT, 0, s>>>(A, f, uin, uout, b);
}

// 9-point plane levels: a sweep in two launches.  Colours 0, 1 live on the even rows
// and colour 1 depends only on colour 0 of its own row and on the (untouched) odd
// rows, colours 2, 3 likewise on the odd rows, so one CTA per (row, plane) runs the
// row's first colour, a barrier, its second colour -- in place, since no other CTA
// touches that row -- and a sweep is two launches instead of four.  Same per-point
// expression as kP_relax: the same iterate.
__global__ void kP_relax9_rows(OpP A, const double *__restrict__ f, double *__restrict__ u, Batch bt, int odd)
{
    const int k = bt.k0 + 2 * blockIdx.z, j = 2 * blockIdx.x + (odd ? 1 : 2);
    if (j > A.g.ny)
        return;
    const long long Y = A.g.px, base = (long long)k * A.g.ps + (long long)j * Y;
    for (int c = 0; c < 2; c++) {  // i even, then i odd
        for (int i = (c ? 1 : 2) + 2 * threadIdx.x; i <= A.g.nx; i += 2 * blockDim.x) {
            const long long p = base + i;
            const R9 a = rowP(A, p);
            u[p] = (f[p] - offP(a, u, p, Y)) * rcp_pos(a.o);
        }
        __syncthreads();
    }
}

void launchP_relax(const OpP &A, const double *f, double *u, Batch b, cudaStream_t s)
{
    const int hx = (A.g.nx + 1) / 2;
    if (A.kind == 5) {
        dim3 grid((hx + 127) / 128, A.g.ny, b.nb);
        for (int c = 0; c < 2; c++)
            kP_relax<5><<<grid, 128, 0, s>>>(A, f, u, b, c);
    } else {
        const int nt = hx <= 32 ? 32 : hx <= 64 ? 64 : 128;
        kP_relax9_rows<<<dim3(A.g.ny / 2, 1, b.nb), nt, 0, s>>>(A, f, u, b, 0);
        kP_relax9_rows<<<dim3((A.g.ny + 1) / 2, 1, b.nb), nt, 0, s>>>(A, f, u, b, 1);
    }
}

__global__ void kP_residual(OpP A, const double *__restrict__ f, const double *__restrict__ u, double *__restrict__ r,
                            Batch bt)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x + 1, j = blockIdx.y + 1, k = bt.k0 + 2 * blockIdx.z;
    if (i > A.g.nx)
        return;
    const long long p = (long long)k * A.g.ps + (long long)j * A.g.px + i;
    const R9 a = rowP(A, p);
    r[p] = f[p] - (a.o * u[p] + offP(a, u, p, A.g.px));
}

void launchP_residual(const OpP &A, const double *f, const double *u, double *r, Batch b, cudaStream_t s)
{
    dim3 grid((A.g.nx + 127) / 128, A.g.ny, b.nb);
    kP_residual<<<grid, 128, 0, s>>>(A, f, u, r, b);
}

// f_c = P^T r over the 3x3 fine box, u_c = 0
__global__ void kP_restrict(Grid3 fg, CIP ci, const double *__restrict__ r, double *__restrict__ fc,
                            double *__restrict__ uc, Batch bt)
{
    const int Ci = blockIdx.x * blockDim.x + threadIdx.x + 1, Cj = blockIdx.y + 1, k = bt.k0 + 2 * blockIdx.z;
    if (Ci > ci.c.nx)
        return;
    const long long fk = (long long)k * fg.ps, ck = (long long)k * ci.c.ps;
    double s = 0.0;
    for (int e = 0; e < 9; e++) {
        const int fi = 2 * Ci + e % 3 - 1, fj = 2 * Cj + e / 3 - 1;
        if (!inside2(fg, fi, fj))
            continue;
        s += pwP(ci, ck, fi, fj, Ci, Cj) * r[fk + (long long)fj * fg.px + fi];
    }
    const long long pc = ck + (long long)Cj * ci.c.px + Ci;
    fc[pc] = s;
    uc[pc] = 0.0;
}

void launchP_restrict(const OpP &A, const CIP &ci, const double *r, double *fc, double *uc, Batch b, cudaStream_t s)
{
    dim3 grid((ci.c.nx + 127) / 128, ci.c.ny, b.nb);
    kP_restrict<<<grid, 128, 0, s>>>(A.g, ci, r, fc, uc, b);
}

// u += P e_c (c7)
__global__ void kP_interp_add(Grid3 fg, CIP ci, const double *__restrict__ ec, double *__restrict__ u, Batch bt)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x + 1, j = blockIdx.y + 1, k = bt.k0 + 2 * blockIdx.z;
    if (i > fg.nx)
        return;
    const long long ck = (long long)k * ci.c.ps, Y = ci.c.px;
    const int oi = i & 1, oj = j & 1;
    double s;
    if (!oi && !oj) {
        s = ec[ck + (long long)(j >> 1) * Y + (i >> 1)];
    } else if (oi && !oj) {
        const int I = (i + 1) >> 1, J = j >> 1;
        const long long q = ck + (long long)J * Y + I;
        s = ci.w[P_LL][q] * ec[q - 1] + ci.w[P_LR][q] * ec[q];
    } else if (!oi && oj) {
        const int I = i >> 1, J = (j + 1) >> 1;
        const long long q = ck + (long long)J * Y + I;
        s = ci.w[P_LB][q] * ec[q - Y] + ci.w[P_LA][q] * ec[q];
    } else {
        const int I = (i + 1) >> 1, J = (j + 1) >> 1;
        const long long q = ck + (long long)J * Y + I;
        s = ci.w[P_LSW][q] * ec[q - Y - 1] + ci.w[P_LSE][q] * ec[q - Y] + ci.w[P_LNW][q] * ec[q - 1] +
            ci.w[P_LNE][q] * ec[q];
    }
    u[(long long)k * fg.ps + (long long)j * fg.px + i] += s;
}

void launchP_interp_add(const Grid3 &fine, const CIP &ci, const double *ec, double *u, Batch b, cudaStream_t s)
{
    dim3 grid((fine.nx + 127) / 128, fine.ny, b.nb);
    kP_interp_add<<<grid, 128, 0, s>>>(fine, ci, ec, u, b);
}

// per plane: u = L^-T L^-1 f on the coarsest plane level, one CTA per plane
__global__ void kP_coarse_solve(OpP A, const double *__restrict__ Lall, const double *__restrict__ f,
                                double *__restrict__ u, Batch bt)
{
    extern __shared__ double b[];
    const int k = bt.k0 + 2 * blockIdx.x, nx = A.g.nx, n = nx * A.g.ny;
    const double *L = Lall + (long long)(k - 1) * n * n;
    const long long base = (long long)k * A.g.ps;
    if (n <= 32) {
        if (threadIdx.x < 32) {
            const int i = threadIdx.x;
            const long long q = base + (long long)(i / nx + 1) * A.g.px + i % nx + 1;
            const double x = warp_chol_solve(L, n, i < n ? f[q] : 0.0);
            if (i < n)
                u[q] = x;
        }
        return;
    }
    for (int t = threadIdx.x; t < n; t += blockDim.x)
        b[t] = f[base + (long long)(t / nx + 1) * A.g.px + t % nx + 1];
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
        u[base + (long long)(t / nx + 1) * A.g.px + t % nx + 1] = b[t];
}

void launchP_coarse_solve(const OpP &A, const double *L, const double *f, double *u, Batch b, cudaStream_t s)
{
    const int n = A.g.nx * A.g.ny;
    const int threads = n < 256 ? ((n + 31) / 32) * 32 : 256;
    kP_coarse_solve<<<b.nb, threads, sizeof(double) * n, s>>>(A, L, f, u, b);
}

}  // namespace bmg3

namespace bmg3 {

// ---------------------------------------------------------------- the plane tail
// The small 2-D levels m0..M-1 of a plane V(1,1) cycle (each plane at most
// PTAIL_MAX unknowns) in ONE launch, one CTA per plane of the batch: the steps
// are the batched kernels' per-point expressions, ordered by __syncthreads
// instead of launch boundaries (within a colour the updates are independent), so
// the plane iterate is that of the batched path.  The levels are a few KB each and
// stay in L2; ~12 launches per level become barriers.
__device__ void pt_relax(const OpP &A, const double *f, double *u, long long base)
{
    const int nx = A.g.nx, ny = A.g.ny, ncol = A.kind == 5 ? 2 : 4;
    if (A.kind == 9) {
        // a warp per row: colours 0, 1 of the even rows (the second only after the first
        // within the row: __syncwarp), one barrier, colours 2, 3 of the odd rows -- two CTA
        // barriers per sweep instead of four (same updates, same order per point)
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
        for (int odd = 0; odd < 2; odd++) {
            for (int j = (odd ? 1 : 2) + 2 * warp; j <= ny; j += 2 * nw) {
                for (int c = 0; c < 2; c++) {
                    for (int i = (c ? 1 : 2) + 2 * lane; i <= nx; i += 64) {
                        const long long p = base + (long long)j * A.g.px + i;
                        const R9 a = rowP(A, p);
                        u[p] = (f[p] - offP(a, u, p, A.g.px)) * rcp_pos(a.o);
                    }
                    __syncwarp();
                }
            }
            __syncthreads();
        }
        return;
    }
    for (int c = 0; c < ncol; c++) {
        const int hx = (nx + 1) / 2;
        const int rows = A.kind == 5 ? ny : (ny + 1) / 2;
        for (int t = threadIdx.x; t < hx * rows; t += blockDim.x) {
            int i, j;
            if (A.kind == 5) {
                j = t / hx + 1;
                i = (((c + j) & 1) ? 1 : 2) + 2 * (t % hx);
            } else {
                i = ((c & 1) ? 1 : 2) + 2 * (t % hx);
                j = ((c & 2) ? 1 : 2) + 2 * (t / hx);
            }
            if (i > nx || j > ny)
                continue;
            const long long p = base + (long long)j * A.g.px + i;
            const R9 a = rowP(A, p);
            u[p] = (f[p] - offP(a, u, p, A.g.px)) * rcp_pos(a.o);
        }
        __syncthreads();
    }
}

__device__ void pt_residual(const OpP &A, const double *f, const double *u, double *r, long long base)
{
    const int nx = A.g.nx, n = nx * A.g.ny;
    for (int t = threadIdx.x; t < n; t += blockDim.x) {
        const long long p = base + (long long)(t / nx + 1) * A.g.px + t % nx + 1;
        const R9 a = rowP(A, p);
        r[p] = f[p] - (a.o * u[p] + offP(a, u, p, A.g.px));
    }
    __syncthreads();
}

__device__ void pt_restrict(const Grid3 &fg, const CIP &ci, const double *r, double *fc, double *uc, int k)
{
    const int nx = ci.c.nx, n = nx * ci.c.ny;
    const long long fk = (long long)k * fg.ps, ck = (long long)k * ci.c.ps;
    for (int t = threadIdx.x; t < n; t += blockDim.x) {
        const int Ci = t % nx + 1, Cj = t / nx + 1;
        double s = 0.0;
        for (int e = 0; e < 9; e++) {
            const int fi = 2 * Ci + e % 3 - 1, fj = 2 * Cj + e / 3 - 1;
            if (!inside2(fg, fi, fj))
                continue;
            s += pwP(ci, ck, fi, fj, Ci, Cj) * r[fk + (long long)fj * fg.px + fi];
        }
        const long long pc = ck + (long long)Cj * ci.c.px + Ci;
        fc[pc] = s;
        uc[pc] = 0.0;
    }
    __syncthreads();
}

__device__ void pt_interp_add(const Grid3 &fg, const CIP &ci, const double *ec, double *u, int k)
{
    const int nx = fg.nx, n = nx * fg.ny;
    const long long ck = (long long)k * ci.c.ps, Y = ci.c.px;
    for (int t = threadIdx.x; t < n; t += blockDim.x) {
        const int i = t % nx + 1, j = t / nx + 1;
        const int oi = i & 1, oj = j & 1;
        double s;
        if (!oi && !oj) {
            s = ec[ck + (long long)(j >> 1) * Y + (i >> 1)];
        } else if (oi && !oj) {
            const long long q = ck + (long long)(j >> 1) * Y + ((i + 1) >> 1);
            s = ci.w[P_LL][q] * ec[q - 1] + ci.w[P_LR][q] * ec[q];
        } else if (!oi && oj) {
            const long long q = ck + (long long)((j + 1) >> 1) * Y + (i >> 1);
            s = ci.w[P_LB][q] * ec[q - Y] + ci.w[P_LA][q] * ec[q];
        } else {
            const long long q = ck + (long long)((j + 1) >> 1) * Y + ((i + 1) >> 1);
            s = ci.w[P_LSW][q] * ec[q - Y - 1] + ci.w[P_LSE][q] * ec[q - Y] + ci.w[P_LNW][q] * ec[q - 1] +
                ci.w[P_LNE][q] * ec[q];
        }
        u[(long long)k * fg.ps + (long long)j * fg.px + i] += s;
    }
    __syncthreads();
}

__device__ void pt_coarse(const OpP &A, const double *Lall, const double *f, double *u, int k, double *b)
{
    const int nx = A.g.nx, n = nx * A.g.ny;
    const double *L = Lall + (long long)(k - 1) * n * n;
    const long long base = (long long)k * A.g.ps;
    if (n <= 32) {  // one warp, no barriers inside
        if (threadIdx.x < 32) {
            const int i = threadIdx.x;
            const long long q = base + (long long)(i / nx + 1) * A.g.px + i % nx + 1;
            const double x = warp_chol_solve(L, n, i < n ? f[q] : 0.0);
            if (i < n)
                u[q] = x;
        }
        __syncthreads();
        return;
    }
    for (int t = threadIdx.x; t < n; t += blockDim.x)
        b[t] = f[base + (long long)(t / nx + 1) * A.g.px + t % nx + 1];
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
        u[base + (long long)(t / nx + 1) * A.g.px + t % nx + 1] = b[t];
    __syncthreads();
}

__global__ void __launch_bounds__(256) kP_tail(PTail T, Batch bt)
{
    extern __shared__ double sb[];
    const int k = bt.k0 + 2 * blockIdx.x;
    const int M = T.nlev;
    // down: relax, residual, restrict on levels 0..M-2 of the tail
    for (int m = 0; m + 1 < M; m++) {
        const PTailLevel &a = T.lv[m];
        const long long base = (long long)k * a.op.g.ps;
        pt_relax(a.op, a.f, a.u, base);
        pt_residual(a.op, a.f, a.u, a.r, base);
        pt_restrict(a.op.g, a.ci, a.r, T.lv[m + 1].f, T.lv[m + 1].u, k);
    }
    pt_coarse(T.lv[M - 1].op, T.chol, T.lv[M - 1].f, T.lv[M - 1].u, k, sb);
    for (int m = M - 2; m >= 0; m--) {
        const PTailLevel &a = T.lv[m];
        pt_interp_add(a.op.g, a.ci, T.lv[m + 1].u, a.u, k);
        pt_relax(a.op, a.f, a.u, (long long)k * a.op.g.ps);
    }
}

void launchP_tail(const PTail &T, Batch b, cudaStream_t s)
{
    const OpP &c = T.lv[T.nlev - 1].op;
    const int n = c.g.nx * c.g.ny;
    kP_tail<<<b.nb, 256, sizeof(double) * n, s>>>(T, b);
}

}  // namespace bmg3
