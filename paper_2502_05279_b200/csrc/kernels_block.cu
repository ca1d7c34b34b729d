// kernels_block.cu -- block multi-RHS V-cycle kernels (DESIGN §3 c15; SURVEY
// §8(f) row 2; §5: "solve several initial vectors in block
// fashion").
//
// K right-hand sides (and K iterates) are stored interleaved: element (j, i, c)
// at (j*pitch + i)*K + c.  A thread loads the operator row / interpolation
// weights of its point ONCE and applies them to the K columns, whose values
// sit in K consecutive doubles (16-byte vector loads for even K).  The stencil
// and weight planes -- the dominant bytes of a cycle -- are thus read
// once per block instead of once per right-hand side.
//
// Per column every kernel performs the per-step kernels' operations
// (kernels_cycle.cu) in the same source order, with every product-sum pinned
// to that order (__dmul_rn/__fma_rn); column c of a block cycle is the
// single-RHS cycle on column c up to the FMA contractions nvcc picks there.
#include "bmg_internal.cuh"

namespace bmg {

namespace {

// K consecutive doubles (16-byte aligned for even K: cudaMalloc'd bases and an
// even element offset)
template <int K>
__device__ __forceinline__ void ldk(const double *__restrict__ p, double (&v)[K])
{
    if constexpr (K % 2 == 0) {
#pragma unroll
        for (int c = 0; c < K / 2; c++) {
            const double2 t = reinterpret_cast<const double2 *>(p)[c];
            v[2 * c] = t.x;
            v[2 * c + 1] = t.y;
        }
    } else {
#pragma unroll
        for (int c = 0; c < K; c++)
            v[c] = p[c];
    }
}

template <int K>
__device__ __forceinline__ void stk(double *__restrict__ p, const double (&v)[K])
{
    if constexpr (K % 2 == 0) {
#pragma unroll
        for (int c = 0; c < K / 2; c++)
            reinterpret_cast<double2 *>(p)[c] = make_double2(v[2 * c], v[2 * c + 1]);
    } else {
#pragma unroll
        for (int c = 0; c < K; c++)
            p[c] = v[c];
    }
}

template <int K>
__device__ __forceinline__ void setk(double *__restrict__ p, double x)
{
    double v[K];
#pragma unroll
    for (int c = 0; c < K; c++)
        v[c] = x;
    stk<K>(p, v);
}

// Work split: a thread owns W = 2 columns of its point (one 16-byte access per
// neighbour) for even K, W = 1 for odd K, and TP = K / W threads share a point
// (consecutive lanes: a warp touches 32/TP points' contiguous column blocks).
// The operator row / weights are loaded by each of the TP threads (same address,
// one L1 transaction).
template <int K>
struct Split {
    static constexpr int W = (K % 2 == 0) ? 2 : 1;
    static constexpr int TP = K / W;
};

// (off-diagonal part of A u)_p for W columns at element stride K (u already
// offset to the first of them), fig:stencil_operator order SW,S,SE,W,E,NW,N,NE
// (offdiag() of kernels_cycle.cu per column)
template <int W, int K>
__device__ __forceinline__ void offdiag_w(const Row9 &a, const double *__restrict__ u, long long p, long long P,
                                          double (&s)[W])
{
    double t[W];
    ldk<W>(u + (p - P - 1) * K, t);
#pragma unroll
    for (int c = 0; c < W; c++)
        s[c] = __dmul_rn(a.sw, t[c]);
    ldk<W>(u + (p - P) * K, t);
#pragma unroll
    for (int c = 0; c < W; c++)
        s[c] = __fma_rn(a.s, t[c], s[c]);
    ldk<W>(u + (p - P + 1) * K, t);
#pragma unroll
    for (int c = 0; c < W; c++)
        s[c] = __fma_rn(a.se, t[c], s[c]);
    ldk<W>(u + (p - 1) * K, t);
#pragma unroll
    for (int c = 0; c < W; c++)
        s[c] = __fma_rn(a.w, t[c], s[c]);
    ldk<W>(u + (p + 1) * K, t);
#pragma unroll
    for (int c = 0; c < W; c++)
        s[c] = __fma_rn(a.e, t[c], s[c]);
    ldk<W>(u + (p + P - 1) * K, t);
#pragma unroll
    for (int c = 0; c < W; c++)
        s[c] = __fma_rn(a.nw, t[c], s[c]);
    ldk<W>(u + (p + P) * K, t);
#pragma unroll
    for (int c = 0; c < W; c++)
        s[c] = __fma_rn(a.n, t[c], s[c]);
    ldk<W>(u + (p + P + 1) * K, t);
#pragma unroll
    for (int c = 0; c < W; c++)
        s[c] = __fma_rn(a.ne, t[c], s[c]);
}

// v[c] = w * q[c] / v[c] += w * q[c] / v[c] += q[c].  Every product-sum chain in
// this file is written with __dmul_rn / __fma_rn in source order: left to the
// compiler, a*b + c*d may contract to either fma(c,d,a*b) or fma(a,b,c*d), and
// the block kernels' rounding is pinned to the source order instead.
template <int W, int K>
__device__ __forceinline__ void wset(double (&v)[W], double w, const double *__restrict__ q, long long qi)
{
    double t[W];
    ldk<W>(q + qi * K, t);
#pragma unroll
    for (int c = 0; c < W; c++)
        v[c] = __dmul_rn(w, t[c]);
}

template <int W, int K>
__device__ __forceinline__ void wadd(double (&v)[W], double w, const double *__restrict__ q, long long qi)
{
    double t[W];
    ldk<W>(q + qi * K, t);
#pragma unroll
    for (int c = 0; c < W; c++)
        v[c] = __fma_rn(w, t[c], v[c]);
}

template <int W, int K>
__device__ __forceinline__ void add1(double (&v)[W], const double *__restrict__ q, long long qi)
{
    double t[W];
    ldk<W>(q + qi * K, t);
#pragma unroll
    for (int c = 0; c < W; c++)
        v[c] += t[c];
}

// ------------------------------------------------------------------ relaxation (c6)
template <int K>
__global__ void kb_relax5(Op A, const double *__restrict__ f, double *__restrict__ u, int colour)
{
    constexpr int W = Split<K>::W, TP = Split<K>::TP;
    const int j = blockIdx.y * blockDim.y + threadIdx.y + 1;
    if (j > A.ny)
        return;
    const int gx = blockIdx.x * blockDim.x + threadIdx.x, sub = gx % TP;
    const int i = ((((1 + j) & 1) == colour) ? 1 : 2) + 2 * (gx / TP);
    if (i > A.nx)
        return;
    const long long P = A.pitch, p = j * P + i;
    const double o = A.O[p], w = A.W[p], e = A.W[p + 1], s = A.S[p], n = A.S[p + P];
    const double rc = rcp_pos(o);
    const double *ub = u + sub * W;
    double us[W], uw[W], ue[W], un[W], fp[W], out[W];
    ldk<W>(ub + (p - P) * K, us);
    ldk<W>(ub + (p - 1) * K, uw);
    ldk<W>(ub + (p + 1) * K, ue);
    ldk<W>(ub + (p + P) * K, un);
    ldk<W>(f + sub * W + p * K, fp);
#pragma unroll
    for (int c = 0; c < W; c++) {
        double acc = __dmul_rn(s, us[c]);
        acc = __fma_rn(w, uw[c], acc);
        acc = __fma_rn(e, ue[c], acc);
        acc = __fma_rn(n, un[c], acc);
        out[c] = (fp[c] - acc) * rc;
    }
    stk<W>(u + sub * W + p * K, out);
}

template <int K>
__global__ void kb_relax9(Op A, const double *__restrict__ f, double *__restrict__ u, int colour)
{
    constexpr int W = Split<K>::W, TP = Split<K>::TP;
    const int j = 2 * (blockIdx.y * blockDim.y + threadIdx.y) + ((colour >> 1) ? 1 : 2);
    if (j > A.ny)
        return;
    const int gx = blockIdx.x * blockDim.x + threadIdx.x, sub = gx % TP;
    const int i = 2 * (gx / TP) + ((colour & 1) ? 1 : 2);
    if (i > A.nx)
        return;
    const long long P = A.pitch, p = j * P + i;
    const Row9 a = load_row9(A, p);
    const double rc = rcp_pos(a.o);
    double sm[W], fp[W];
    offdiag_w<W, K>(a, u + sub * W, p, P, sm);
    ldk<W>(f + sub * W + p * K, fp);
#pragma unroll
    for (int c = 0; c < W; c++)
        sm[c] = (fp[c] - sm[c]) * rc;
    stk<W>(u + sub * W + p * K, sm);
}

// ------------------------------------------------------------------ one-pass red-black sweep (5-point levels)
// uout = GS(uin), both colours in ONE pass over the level (kb_relax5 makes two, each
// reading every K-column block).  A CTA owns a strip of TX points and RC rows and
// marches up the rows: the red points of row j on the strip plus a one-point ring
// (their neighbours are old black values in uin, which nobody writes) go to a 4-row
// shared ring; one barrier later the black points of row j-1 take their neighbours
// from the ring, and row j-1 is written out whole.  Ring points are recomputed by
// each CTA that needs them (no inter-CTA waits).  Per point and column the
// expression is kb_relax5's, pinned (__dmul_rn/__fma_rn): bitwise its result.
template <int K>
struct RB5 {
    static constexpr int W = Split<K>::W, TP = Split<K>::TP, NT = 256, NPT = NT / TP;
    static constexpr int TX = 2 * NPT, RX = TX + 2, RC = 32;
};

template <int W>
__device__ __forceinline__ void gs5w(const double *__restrict__ A_O, const double *__restrict__ A_W,
                                     const double *__restrict__ A_S, long long p, long long P, const double (&us)[W],
                                     const double (&uw)[W], const double (&ue)[W], const double (&un)[W],
                                     const double (&fp)[W], double (&out)[W])
{
    const double o = A_O[p], w = A_W[p], e = A_W[p + 1], s = A_S[p], n = A_S[p + P];
    const double rc = rcp_pos(o);
#pragma unroll
    for (int c = 0; c < W; c++) {
        double acc = __dmul_rn(s, us[c]);
        acc = __fma_rn(w, uw[c], acc);
        acc = __fma_rn(e, ue[c], acc);
        acc = __fma_rn(n, un[c], acc);
        out[c] = (fp[c] - acc) * rc;
    }
}

template <int K>
__global__ void __launch_bounds__(256) kb_rb5(Op A, const double *__restrict__ f, const double *__restrict__ uin,
                                              double *__restrict__ uout)
{
    using R = RB5<K>;
    constexpr int W = R::W, TP = R::TP, NT = R::NT, NPT = R::NPT, RX = R::RX;
    __shared__ __align__(16) double red[4][RX * K];
    const long long P = A.pitch;
    const int i0 = blockIdx.x * R::TX + 1, jb = blockIdx.y * R::RC + 1, je = min(jb + R::RC, A.ny + 1);
    const int tid = threadIdx.x;
    for (int j = jb - 1; j <= je; j++) {
        double *rj = red[j & 3];
        const int base = i0 - 1;
        for (int t = tid; t < (NPT + 1) * TP; t += NT) {
            const int pt = t / TP, sb = t % TP;
            const int i = base + 2 * pt + ((base + j) & 1);
            double v[W];
#pragma unroll
            for (int c = 0; c < W; c++)
                v[c] = 0.0;
            if (j >= 1 && j <= A.ny && i >= 1 && i <= A.nx) {
                const long long p = j * P + i;
                const double *ub = uin + sb * W;
                double us[W], uw[W], ue[W], un[W], fp[W];
                ldk<W>(ub + (p - P) * K, us);
                ldk<W>(ub + (p - 1) * K, uw);
                ldk<W>(ub + (p + 1) * K, ue);
                ldk<W>(ub + (p + P) * K, un);
                ldk<W>(f + sb * W + p * K, fp);
                gs5w<W>(A.O, A.W, A.S, p, P, us, uw, ue, un, fp, v);
            }
            if (i - base < RX)
                stk<W>(rj + (i - base) * K + sb * W, v);
        }
        __syncthreads();
        const int jj = j - 1;
        if (jj >= jb && jj < je && tid < NPT * TP) {
            const int pt = tid / TP, sb = tid % TP;
            const int ia = i0 + 2 * pt;
            const int odd_a = (ia + jj) & 1;  // 1: ia is black
            const int ib = odd_a ? ia : ia + 1, ir = odd_a ? ia + 1 : ia;
            const double *rl = red[(jj - 1) & 3], *rm = red[jj & 3], *rh = red[j & 3];
            double vb[W];
            if (ib <= A.nx) {
                const long long p = jj * P + ib;
                const int cb = ib - base;
                double us[W], uw[W], ue[W], un[W], fp[W];
                ldk<W>(rl + cb * K + sb * W, us);
                ldk<W>(rm + (cb - 1) * K + sb * W, uw);
                ldk<W>(rm + (cb + 1) * K + sb * W, ue);
                ldk<W>(rh + cb * K + sb * W, un);
                ldk<W>(f + sb * W + p * K, fp);
                gs5w<W>(A.O, A.W, A.S, p, P, us, uw, ue, un, fp, vb);
                stk<W>(uout + sb * W + p * K, vb);
            }
            if (ir <= A.nx) {
                double vr[W];
                ldk<W>(rm + (ir - base) * K + sb * W, vr);
                stk<W>(uout + sb * W + (jj * P + ir) * K, vr);
            }
        }
    }
}

// one point, W columns: u = (f - sum_{q != p} a_pq u_q) * rcp(a_pp), neighbour values
// given in fig:stencil_operator order SW,S,SE,W,E,NW,N,NE (offdiag_w's order)
template <int W>
__device__ __forceinline__ void gs9w(const Row9 &a, const double (&n)[8][W], const double (&fp)[W], double (&out)[W])
{
    const double rc = rcp_pos(a.o);
#pragma unroll
    for (int c = 0; c < W; c++) {
        double s = __dmul_rn(a.sw, n[0][c]);
        s = __fma_rn(a.s, n[1][c], s);
        s = __fma_rn(a.se, n[2][c], s);
        s = __fma_rn(a.w, n[3][c], s);
        s = __fma_rn(a.e, n[4][c], s);
        s = __fma_rn(a.nw, n[5][c], s);
        s = __fma_rn(a.n, n[6][c], s);
        s = __fma_rn(a.ne, n[7][c], s);
        out[c] = (fp[c] - s) * rc;
    }
}

// ------------------------------------------------------------------ 9-point levels: a sweep in two launches
// The four colours of a 9-point level pair up by rows: colours 0, 1 live on the even
// rows and, within a row, 1 depends only on 0 (its x-neighbours) and on the odd rows
// (old); colours 2, 3 likewise on the odd rows given the even rows (new).  So a sweep
// uout = GS(uin) is two launches: even rows (neighbour rows from uin), then odd rows
// (neighbour rows from uout), each CTA a row segment whose first colour is recomputed
// on a one-point ring from uin (read-only), the second colour taking its x-neighbours
// from shared memory, both written out.  Per point kb_relax9's expression: bitwise.
template <int K>
struct R9P {
    static constexpr int W = Split<K>::W, TP = Split<K>::TP, NT = 256, NPT = NT / TP, TX = 2 * NPT;
};

template <int K>
__global__ void __launch_bounds__(256) kb_r9pair(Op A, const double *__restrict__ f, const double *__restrict__ uin,
                                                 double *uout, int odd)
{
    using R = R9P<K>;
    constexpr int W = R::W, TP = R::TP, NT = R::NT, NPT = R::NPT;
    __shared__ __align__(16) double c1[(NPT + 1) * K];  // the first colour, even i in [x0-1, x0+TX]
    const long long P = A.pitch;
    const int j = 2 * blockIdx.y + (odd ? 1 : 2);
    if (j > A.ny)
        return;
    const int x0 = blockIdx.x * R::TX + 1;
    const double *nb = odd ? uout : uin;  // rows j +- 1: old (even-row pass) or new (odd-row pass)
    const int tid = threadIdx.x;
    for (int t = tid; t < (NPT + 1) * TP; t += NT) {
        const int pt = t / TP, sb = t % TP, i = x0 - 1 + 2 * pt;
        double v[W];
#pragma unroll
        for (int c = 0; c < W; c++)
            v[c] = 0.0;
        if (i >= 1 && i <= A.nx) {
            const long long q = j * P + i;
            double n[8][W], fp[W];
            ldk<W>(nb + sb * W + (q - P - 1) * K, n[0]);
            ldk<W>(nb + sb * W + (q - P) * K, n[1]);
            ldk<W>(nb + sb * W + (q - P + 1) * K, n[2]);
            ldk<W>(uin + sb * W + (q - 1) * K, n[3]);
            ldk<W>(uin + sb * W + (q + 1) * K, n[4]);
            ldk<W>(nb + sb * W + (q + P - 1) * K, n[5]);
            ldk<W>(nb + sb * W + (q + P) * K, n[6]);
            ldk<W>(nb + sb * W + (q + P + 1) * K, n[7]);
            ldk<W>(f + sb * W + q * K, fp);
            gs9w<W>(load_row9(A, q), n, fp, v);
            if (i >= x0 && i < x0 + R::TX)
                stk<W>(uout + sb * W + q * K, v);
        }
        stk<W>(c1 + pt * K + sb * W, v);
    }
    __syncthreads();
    if (tid < NPT * TP) {
        const int pt = tid / TP, sb = tid % TP, i = x0 + 2 * pt;
        if (i <= A.nx) {
            const long long q = j * P + i;
            double n[8][W], fp[W], v[W];
            ldk<W>(nb + sb * W + (q - P - 1) * K, n[0]);
            ldk<W>(nb + sb * W + (q - P) * K, n[1]);
            ldk<W>(nb + sb * W + (q - P + 1) * K, n[2]);
            ldk<W>(c1 + pt * K + sb * W, n[3]);        // i-1 = x0-1+2pt
            ldk<W>(c1 + (pt + 1) * K + sb * W, n[4]);  // i+1
            ldk<W>(nb + sb * W + (q + P - 1) * K, n[5]);
            ldk<W>(nb + sb * W + (q + P) * K, n[6]);
            ldk<W>(nb + sb * W + (q + P + 1) * K, n[7]);
            ldk<W>(f + sb * W + q * K, fp);
            gs9w<W>(load_row9(A, q), n, fp, v);
            stk<W>(uout + sb * W + q * K, v);
        }
    }
}

// ------------------------------------------------------------------ residual
template <int K>
__global__ void kb_residual(Op A, const double *__restrict__ f, const double *__restrict__ u, double *__restrict__ r)
{
    constexpr int W = Split<K>::W, TP = Split<K>::TP;
    const int gx = blockIdx.x * blockDim.x + threadIdx.x, sub = gx % TP, i = gx / TP;
    const int j = blockIdx.y * blockDim.y + threadIdx.y;
    if (i > A.nx + 1 || j > A.ny + 1)
        return;
    const long long P = A.pitch, p = j * P + i;
    if (i == 0 || j == 0 || i > A.nx || j > A.ny) {
        setk<W>(r + sub * W + p * K, 0.0);
        return;
    }
    const Row9 a = load_row9(A, p);
    double sm[W], up[W], fp[W];
    offdiag_w<W, K>(a, u + sub * W, p, P, sm);
    ldk<W>(u + sub * W + p * K, up);
    ldk<W>(f + sub * W + p * K, fp);
#pragma unroll
    for (int c = 0; c < W; c++)
        sm[c] = fp[c] - __fma_rn(a.o, up[c], sm[c]);
    stk<W>(r + sub * W + p * K, sm);
}

// ------------------------------------------------------------------ restriction (fig:restrict_kernel)
template <int K>
__global__ void kb_restrict(Op A, CIv ci, const double *__restrict__ q, double *__restrict__ qc,
                            double *__restrict__ uc, bool vanish)
{
    constexpr int W = Split<K>::W, TP = Split<K>::TP;
    const int gx = blockIdx.x * blockDim.x + threadIdx.x, sub = gx % TP, I = gx / TP;
    const int J = blockIdx.y * blockDim.y + threadIdx.y;
    if (I > A.nx / 2 + 1 || J > A.ny / 2 + 1)
        return;
    const long long C = ci.pitch, c = J * C + I;
    if (uc)
        setk<W>(uc + sub * W + c * K, 0.0);
    if (I == 0 || J == 0 || I > A.nx / 2 || J > A.ny / 2) {
        setk<W>(qc + sub * W + c * K, 0.0);
        return;
    }
    const long long P = A.pitch, p = (2 * J) * P + 2 * I;
    const double *qb = q + sub * W;
    double v[W];
    if (vanish && A.kind == 5) {  // restrict_pt_vanish, 5-point: centre + Z terms
        wset<W, K>(v, ci.w[CI_LNE][c], qb, p - P - 1);
        wadd<W, K>(v, ci.w[CI_LNW][c + 1], qb, p - P + 1);
        add1<W, K>(v, qb, p);
        wadd<W, K>(v, ci.w[CI_LSE][c + C], qb, p + P - 1);
        wadd<W, K>(v, ci.w[CI_LSW][c + C + 1], qb, p + P + 1);
    } else if (vanish) {  // 9-point: centre + X/Y terms
        wset<W, K>(v, ci.w[CI_LA][c], qb, p - P);
        wadd<W, K>(v, ci.w[CI_LR][c], qb, p - 1);
        add1<W, K>(v, qb, p);
        wadd<W, K>(v, ci.w[CI_LL][c + 1], qb, p + 1);
        wadd<W, K>(v, ci.w[CI_LB][c + C], qb, p + P);
    } else {  // restrict_pt
        wset<W, K>(v, ci.w[CI_LNE][c], qb, p - P - 1);
        wadd<W, K>(v, ci.w[CI_LA][c], qb, p - P);
        wadd<W, K>(v, ci.w[CI_LNW][c + 1], qb, p - P + 1);
        wadd<W, K>(v, ci.w[CI_LR][c], qb, p - 1);
        add1<W, K>(v, qb, p);
        wadd<W, K>(v, ci.w[CI_LL][c + 1], qb, p + 1);
        wadd<W, K>(v, ci.w[CI_LSE][c + C], qb, p + P - 1);
        wadd<W, K>(v, ci.w[CI_LB][c + C], qb, p + P);
        wadd<W, K>(v, ci.w[CI_LSW][c + C + 1], qb, p + P + 1);
    }
    stk<W>(qc + sub * W + c * K, v);
}

// Residual and vanishing restriction in one pass (after nu1 >= 1 point-GS sweeps,
// DESIGN §5.2): r = f - A u is evaluated only at the fine points the restriction
// keeps -- 5-point: the centres and the Z corners; 9-point: the centres and the
// X/Y edge points -- and never stored in HBM.  Per column the residual is the
// per-step one (f - fma(a_O, u, offdiag)) and the sum is restrict_pt_vanish's,
// in source order.
template <int W, int K>
__device__ __forceinline__ void resid_w(const Op &A, const double *__restrict__ f, const double *__restrict__ u,
                                        int i, int j, double (&r)[W])
{
    const long long P = A.pitch, p = (long long)j * P + i;
    double sm[W], up[W], fp[W];
    if (A.kind == 5) {  // the zero corner terms of offdiag() contribute exact zeros
        const double o = A.O[p], w = A.W[p], e = A.W[p + 1], s = A.S[p], n = A.S[p + P];
        double t[W];
        ldk<W>(u + (p - P) * K, t);
#pragma unroll
        for (int c = 0; c < W; c++)
            sm[c] = __dmul_rn(s, t[c]);
        ldk<W>(u + (p - 1) * K, t);
#pragma unroll
        for (int c = 0; c < W; c++)
            sm[c] = __fma_rn(w, t[c], sm[c]);
        ldk<W>(u + (p + 1) * K, t);
#pragma unroll
        for (int c = 0; c < W; c++)
            sm[c] = __fma_rn(e, t[c], sm[c]);
        ldk<W>(u + (p + P) * K, t);
#pragma unroll
        for (int c = 0; c < W; c++)
            sm[c] = __fma_rn(n, t[c], sm[c]);
        ldk<W>(u + p * K, up);
        ldk<W>(f + p * K, fp);
#pragma unroll
        for (int c = 0; c < W; c++)
            r[c] = fp[c] - __fma_rn(o, up[c], sm[c]);
    } else {
        const Row9 a = load_row9(A, p);
        offdiag_w<W, K>(a, u, p, P, sm);
        ldk<W>(u + p * K, up);
        ldk<W>(f + p * K, fp);
#pragma unroll
        for (int c = 0; c < W; c++)
            r[c] = fp[c] - __fma_rn(a.o, up[c], sm[c]);
    }
}

template <int W>
__device__ __forceinline__ void racc(double (&v)[W], double w, const double (&r)[W], bool first)
{
#pragma unroll
    for (int c = 0; c < W; c++)
        v[c] = first ? __dmul_rn(w, r[c]) : __fma_rn(w, r[c], v[c]);
}

// Tiled so that every residual is evaluated once.  A CTA covers RT_CX x RT_CY coarse points; phase 1
// evaluates r at the fine points their restrictions keep -- the centres
// (2I, 2J) and the corners (odd, odd), a ring of corners included -- into
// shared memory; phase 2 forms each coarse value from there in
// restrict_pt_vanish's order.  (The untiled kernel evaluates each corner for
// all four coarse points that use it.)
#ifndef BMG_RT_CX
#define BMG_RT_CX 16
#endif
#ifndef BMG_RT_CY
#define BMG_RT_CY 8
#endif
constexpr int RT_CX = BMG_RT_CX, RT_CY = BMG_RT_CY;

// CTA shape of the per-colour GS kernels (tuning knob)
#ifndef BMG_KB_BX
#define BMG_KB_BX 128
#endif
#ifndef BMG_KB_BY
#define BMG_KB_BY 2
#endif
#ifndef BMG_KB9_BX
#define BMG_KB9_BX BMG_KB_BX
#endif
#ifndef BMG_KB9_BY
#define BMG_KB9_BY BMG_KB_BY
#endif
template <int K, int KIND>
__global__ void __launch_bounds__(256) kb_resid_restrict_tiled(Op A, CIv ci, const double *__restrict__ f,
                                                               const double *__restrict__ u, double *__restrict__ qc,
                                                               double *__restrict__ uc)
{
    constexpr int W = Split<K>::W, TP = Split<K>::TP;
    constexpr int FX = 2 * RT_CX + 1, FY = 2 * RT_CY + 1;  // fine region 2*I0-1 .. 2*(I0+CX-1)+1
    __shared__ __align__(16) double sr[FY * FX * K];
    const int I0 = 1 + blockIdx.x * RT_CX, J0 = 1 + blockIdx.y * RT_CY;
    const int ncx = A.nx / 2, ncy = A.ny / 2;
    const int x0 = 2 * I0 - 1, y0 = 2 * J0 - 1;
    // phase 1: residual at the kept points of the region -- 5-point: (x + y) even
    // (centres and corners); 9-point: all but (odd, odd) (centres and edges)
    constexpr int HALF = (FX + 1) / 2;  // 5-point: kept points per fine row (rows alternate odd/even)
    constexpr int PER_ROW = KIND == 5 ? HALF : FX;
    for (int it = threadIdx.x; it < FY * PER_ROW * TP; it += blockDim.x) {
        const int sub = it % TP, q = it / TP, ry = q / PER_ROW, k = q % PER_ROW;
        const int y = y0 + ry;
        const int x = KIND == 5 ? x0 + ((ry & 1) ? 1 : 0) + 2 * k : x0 + k;  // x0, y0 odd
        if (x - x0 >= FX || (KIND == 9 && (x & 1) && (y & 1)))
            continue;
        double r[W];
        if (x > A.nx || y > A.ny)  // the Dirichlet ring (and beyond): r = 0, as k_residual stores
#pragma unroll
            for (int k2 = 0; k2 < W; k2++)
                r[k2] = 0.0;
        else
            resid_w<W, K>(A, f + sub * W, u + sub * W, x, y, r);
        stk<W>(sr + ((ry * FX) + (x - x0)) * K + sub * W, r);
    }
    __syncthreads();
    // phase 2: one coarse point per item (ring points of the coarse grid: 0)
    for (int it = threadIdx.x; it < RT_CX * RT_CY * TP; it += blockDim.x) {
        const int sub = it % TP, q = it / TP, I = I0 + q % RT_CX, J = J0 + q / RT_CX;
        if (I > ncx + 1 || J > ncy + 1)
            continue;
        const long long C = ci.pitch, c = J * C + I;
        if (uc)
            setk<W>(uc + sub * W + c * K, 0.0);
        if (I > ncx || J > ncy) {
            setk<W>(qc + sub * W + c * K, 0.0);
            continue;
        }
        const int lx = 2 * I - x0, ly = 2 * J - y0;  // local fine coordinates of the centre
        auto at = [&](int dx, int dy) { return sr + (((ly + dy) * FX) + (lx + dx)) * K + sub * W; };
        double v[W], r[W];
        if (KIND == 5) {  // centre + Z terms
            ldk<W>(at(-1, -1), r);
            racc<W>(v, ci.w[CI_LNE][c], r, true);
            ldk<W>(at(1, -1), r);
            racc<W>(v, ci.w[CI_LNW][c + 1], r, false);
            ldk<W>(at(0, 0), r);
#pragma unroll
            for (int k2 = 0; k2 < W; k2++)
                v[k2] = __dadd_rn(v[k2], r[k2]);
            ldk<W>(at(-1, 1), r);
            racc<W>(v, ci.w[CI_LSE][c + C], r, false);
            ldk<W>(at(1, 1), r);
            racc<W>(v, ci.w[CI_LSW][c + C + 1], r, false);
        } else {  // centre + X/Y terms
            ldk<W>(at(0, -1), r);
            racc<W>(v, ci.w[CI_LA][c], r, true);
            ldk<W>(at(-1, 0), r);
            racc<W>(v, ci.w[CI_LR][c], r, false);
            ldk<W>(at(0, 0), r);
#pragma unroll
            for (int k2 = 0; k2 < W; k2++)
                v[k2] = __dadd_rn(v[k2], r[k2]);
            ldk<W>(at(1, 0), r);
            racc<W>(v, ci.w[CI_LL][c + 1], r, false);
            ldk<W>(at(0, 1), r);
            racc<W>(v, ci.w[CI_LB][c + C], r, false);
        }
        stk<W>(qc + sub * W + c * K, v);
    }
}

// the coarse ring row/column 0 (the tiled kernel's tiles start at I, J = 1)
template <int K>
__global__ void kb_coarse_ring0(int ncx, int ncy, long long C, double *__restrict__ qc, double *__restrict__ uc)
{
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    const int n0 = ncx + 2, n1 = ncy + 2;
    if (t >= n0 + n1)
        return;
    const long long c = t < n0 ? (long long)t : (long long)(t - n0) * C;  // row 0, then column 0
    setk<K>(qc + c * K, 0.0);
    if (uc)
        setk<K>(uc + c * K, 0.0);
}

// ------------------------------------------------------------------ interpolation + correction (c7, c14)
template <int K>
__global__ void kb_interp_add(Op A, CIv ci, const double *__restrict__ e, const double *__restrict__ r,
                              const double *u, double *uout, int skip)
{
    constexpr int W = Split<K>::W, TP = Split<K>::TP;
    const int j = blockIdx.y * blockDim.y + threadIdx.y + 1;
    int gx, i;
    if (skip && A.kind == 5) {
        // only the colour the post-smoother relaxes second is corrected: threads map
        // onto its points alone ((i + j) odd, reversed order (i + j) even)
        gx = blockIdx.x * blockDim.x + threadIdx.x;
        const int want = skip == 2 ? 0 : 1;
        i = ((((1 + j) & 1) == want) ? 1 : 2) + 2 * (gx / TP);
    } else {
        // the parity of i alternates with blockIdx.x, so that a warp (one j) takes one
        // branch below while the two parities of a strip run side by side (u read once)
        gx = (blockIdx.x >> 1) * blockDim.x + threadIdx.x;
        i = 2 * (gx / TP) + 1 + (blockIdx.x & 1);
    }
    const int sub = gx % TP;
    if (i > A.nx || j > A.ny)
        return;
    // skip = 1 (2: reversed colour order): the points the post-smoother's first
    // colour pass overwrites from their neighbours alone are not corrected (their
    // corrected value is never read) -- 5-point: (i + j) even (odd), handled by the
    // thread mapping above; 9-point: the C points (the Z points); as the fused up
    // leg does
    if (skip && A.kind == 9) {  // 9-point: the C points (reversed order: the Z points)
        const bool first = skip == 2 ? ((i & 1) && (j & 1)) : (!(i & 1) && !(j & 1));
        if (first)
            return;
    }
    const long long C = ci.pitch;
    const int I = (i + 1) >> 1, J = (j + 1) >> 1;
    const double *eb = e + sub * W;
    double s[W];
    if (!(i & 1) && !(j & 1)) {  // C point
        ldk<W>(eb + ((j >> 1) * C + (i >> 1)) * K, s);
    } else if ((i & 1) && !(j & 1)) {  // X
        const long long c = (j >> 1) * C + I;
        wset<W, K>(s, ci.w[CI_LL][c], eb, c - 1);
        wadd<W, K>(s, ci.w[CI_LR][c], eb, c);
    } else if (!(i & 1) && (j & 1)) {  // Y
        const long long c = J * C + (i >> 1);
        wset<W, K>(s, ci.w[CI_LB][c], eb, c - C);
        wadd<W, K>(s, ci.w[CI_LA][c], eb, c);
    } else {  // Z
        const long long c = J * C + I;
        wset<W, K>(s, ci.w[CI_LSW][c], eb, c - C - 1);
        wadd<W, K>(s, ci.w[CI_LSE][c], eb, c - C);
        wadd<W, K>(s, ci.w[CI_LNW][c], eb, c - 1);
        wadd<W, K>(s, ci.w[CI_LNE][c], eb, c);
    }
    const long long p = j * A.pitch + i;
    if (r && ((i & 1) || (j & 1))) {  // c14 affine term r / a_O at the non-coarse points
        double rp[W];
        ldk<W>(r + sub * W + p * K, rp);
        const double o = A.O[p];
#pragma unroll
        for (int c = 0; c < W; c++)
            s[c] += rp[c] / o;
    } else if (r) {  // affine_pt() is 0 at C points: s += 0.0, as the per-step kernel
#pragma unroll
        for (int c = 0; c < W; c++)
            s[c] += 0.0;
    }
    double up[W];
    ldk<W>(u + sub * W + p * K, up);
#pragma unroll
    for (int c = 0; c < W; c++)
        up[c] += s[c];
    stk<W>(uout + sub * W + p * K, up);
}

// ------------------------------------------------------------------ coarsest solve (c8)
// CTA c: column c, the substitutions of coarse_solve_cta.
template <int K>
__global__ void kb_coarse_solve(Op A, const double *__restrict__ Lf, const double *__restrict__ f,
                                double *__restrict__ u)
{
    extern __shared__ double b[];
    const int n = A.nx * A.ny, col = blockIdx.x;
    for (int p = threadIdx.x; p < n; p += blockDim.x)
        b[p] = f[((p / A.nx + 1) * A.pitch + p % A.nx + 1) * K + col];
    __syncthreads();
    for (int k = 0; k < n; k++) {  // L y = b
        double bk = b[k] / Lf[(long long)k * n + k];
        __syncthreads();
        if (threadIdx.x == 0)
            b[k] = bk;
        for (int i = k + 1 + threadIdx.x; i < n; i += blockDim.x)
            b[i] -= Lf[(long long)i * n + k] * bk;
        __syncthreads();
    }
    for (int k = n - 1; k >= 0; k--) {  // L^T x = y
        double bk = b[k] / Lf[(long long)k * n + k];
        __syncthreads();
        if (threadIdx.x == 0)
            b[k] = bk;
        for (int i = threadIdx.x; i < k; i += blockDim.x)
            b[i] -= Lf[(long long)k * n + i] * bk;
        __syncthreads();
    }
    for (int p = threadIdx.x; p < n; p += blockDim.x)
        u[((p / A.nx + 1) * A.pitch + p % A.nx + 1) * K + col] = b[p];
}

// ------------------------------------------------------------------ norms (per column, fixed trees)
template <int K, bool RESID>
__global__ void kb_norm_partial(Op A, const double *__restrict__ f, const double *__restrict__ u,
                                double *__restrict__ partials)
{
    // thread t: column slice sub = t % TP of the points 1 + t/TP, 1 + t/TP + 256/TP, ...
    // of the rows ylo + b, ylo + b + NORM_BLOCKS, ...; fixed trees per column
    constexpr int W = Split<K>::W, TP = Split<K>::TP;
    const int sub = threadIdx.x % TP, i0 = threadIdx.x / TP, di = blockDim.x / TP;
    double acc[W];
#pragma unroll
    for (int c = 0; c < W; c++)
        acc[c] = 0.0;
    const long long P = A.pitch;
    const bool idle = (int)threadIdx.x >= di * TP;  // TP need not divide blockDim.x
    for (int j = A.ylo + blockIdx.x; j < A.yhi && !idle; j += gridDim.x) {
        for (int i = 1 + i0; i <= A.nx; i += di) {
            double v[W];
            if (RESID)
                resid_w<W, K>(A, f + sub * W, u + sub * W, i, j, v);  // 5-point: no zero corner terms
            else
                ldk<W>(f + sub * W + (j * P + i) * K, v);
#pragma unroll
            for (int c = 0; c < W; c++)
                acc[c] = __fma_rn(v[c], v[c], acc[c]);
        }
    }
#pragma unroll
    for (int c = 0; c < K; c++) {
        double mine = 0.0;
#pragma unroll
        for (int w = 0; w < W; w++)
            if (sub * W + w == c)
                mine = acc[w];
        const double t = block_sum(mine);
        if (threadIdx.x == 0)
            partials[c * NORM_BLOCKS + blockIdx.x] = t;
    }
}

// CTA c: column c's partials, the tree of k_norm_final
__global__ void kb_norm_final(const double *__restrict__ partials, double *__restrict__ result)
{
    double acc = 0.0;
    const double *pc = partials + blockIdx.x * NORM_BLOCKS;
    for (int k = threadIdx.x; k < NORM_BLOCKS; k += blockDim.x)
        acc += pc[k];
    acc = block_sum(acc);
    if (threadIdx.x == 0)
        result[blockIdx.x] = sqrt(acc);
}

// ------------------------------------------------------------------ block PCG vectors (c13 x c15)
// <a_c, b_c> per column: the tree of k_dot_partial / k_sum_final per column
template <int K>
__global__ void kb_dot_partial(Op A, const double *__restrict__ a, const double *__restrict__ b,
                               double *__restrict__ partials)
{
    // the thread layout of kb_norm_partial (column slices, fixed trees per column)
    constexpr int W = Split<K>::W, TP = Split<K>::TP;
    const int sub = threadIdx.x % TP, i0 = threadIdx.x / TP, di = blockDim.x / TP;
    double acc[W];
#pragma unroll
    for (int c = 0; c < W; c++)
        acc[c] = 0.0;
    const long long P = A.pitch;
    const bool idle = (int)threadIdx.x >= di * TP;
    for (int j = A.ylo + blockIdx.x; j < A.yhi && !idle; j += gridDim.x)
        for (int i = 1 + i0; i <= A.nx; i += di) {
            const long long p = (j * P + i) * K + sub * W;
            double va[W], vb[W];
            ldk<W>(a + p, va);
            ldk<W>(b + p, vb);
#pragma unroll
            for (int c = 0; c < W; c++)
                acc[c] = __fma_rn(va[c], vb[c], acc[c]);
        }
#pragma unroll
    for (int c = 0; c < K; c++) {
        double mine = 0.0;
#pragma unroll
        for (int w = 0; w < W; w++)
            if (sub * W + w == c)
                mine = acc[w];
        const double t = block_sum(mine);
        if (threadIdx.x == 0)
            partials[c * NORM_BLOCKS + blockIdx.x] = t;
    }
}

__global__ void kb_sum_final(const double *__restrict__ partials, double *__restrict__ result)
{
    double acc = 0.0;
    const double *pc = partials + blockIdx.x * NORM_BLOCKS;
    for (int k = threadIdx.x; k < NORM_BLOCKS; k += blockDim.x)
        acc += pc[k];
    acc = block_sum(acc);
    if (threadIdx.x == 0)
        result[blockIdx.x] = acc;
}

// q = A p (interior), the single-RHS matvec (k_matvec_dot_partial) per column
template <int K>
__global__ void kb_matvec(Op A, const double *__restrict__ p, double *__restrict__ q)
{
    constexpr int W = Split<K>::W, TP = Split<K>::TP;
    const int gx = blockIdx.x * blockDim.x + threadIdx.x, sub = gx % TP, i = gx / TP + 1;
    const int j = blockIdx.y * blockDim.y + threadIdx.y + A.ylo;
    if (i > A.nx || j >= A.yhi)
        return;
    const long long P = A.pitch, k = j * P + i;
    const Row9 a = load_row9(A, k);
    double sm[W], pp[W];
    offdiag_w<W, K>(a, p + sub * W, k, P, sm);
    ldk<W>(p + sub * W + k * K, pp);
#pragma unroll
    for (int c = 0; c < W; c++)
        sm[c] = __fma_rn(a.o, pp[c], sm[c]);
    stk<W>(q + sub * W + k * K, sm);
}

// active columns (bit c of mask): x_c += alpha_c p_c, r_c -= alpha_c q_c with
// alpha_c = sc[inum + c] / sc[iden + c] (the single-RHS CG update per column); others untouched
template <int K>
__global__ void kb_cg_update(Op A, const double *__restrict__ sc, int inum, int iden, unsigned mask,
                             const double *__restrict__ p, const double *__restrict__ q, double *__restrict__ x,
                             double *__restrict__ r)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x + 1;
    const int j = blockIdx.y * blockDim.y + threadIdx.y + A.ylo;
    if (i > A.nx || j >= A.yhi)
        return;
    const long long k = (j * A.pitch + i) * K;
#pragma unroll
    for (int c = 0; c < K; c++)
        if ((mask >> c) & 1u) {
            const double alpha = sc[inum + c] / sc[iden + c];
            x[k + c] = __fma_rn(alpha, p[k + c], x[k + c]);
            r[k + c] = __fma_rn(-alpha, q[k + c], r[k + c]);
        }
}

// active columns: p_c = z_c + beta_c p_c, beta_c = sc[inum + c] / sc[iden + c]
template <int K>
__global__ void kb_cg_direction(Op A, const double *__restrict__ sc, int inum, int iden, unsigned mask,
                                const double *__restrict__ z, double *__restrict__ p)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x + 1;
    const int j = blockIdx.y * blockDim.y + threadIdx.y + A.ylo;
    if (i > A.nx || j >= A.yhi)
        return;
    const long long k = (j * A.pitch + i) * K;
#pragma unroll
    for (int c = 0; c < K; c++)
        if ((mask >> c) & 1u) {
            const double beta = sc[inum + c] / sc[iden + c];
            p[k + c] = __fma_rn(beta, p[k + c], z[k + c]);
        }
}

__global__ void kb_zero(long long n, double *x)
{
    const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (t < n)
        x[t] = 0.0;
}

// ------------------------------------------------------------------ launchers
template <int K>
struct Launch {
    static constexpr int TP = Split<K>::TP;
    static void relax(const Op &A, const double *f, double *u, int nsweeps, cudaStream_t s, int *nlaunch, bool rev)
    {
        const dim3 b(BMG_KB_BX, BMG_KB_BY);
        for (int sw = 0; sw < nsweeps; sw++) {
            if (A.kind == 5) {
                const dim3 g(((A.nx / 2 + 1) * TP + b.x - 1) / b.x, (A.ny + b.y - 1) / b.y);
                for (int c = 0; c < 2; c++)
                    kb_relax5<K><<<g, b, 0, s>>>(A, f, u, rev ? 1 - c : c);
                if (nlaunch)
                    *nlaunch += 2;
            } else {
                const dim3 b9(BMG_KB9_BX, BMG_KB9_BY);
                const dim3 g(((A.nx / 2 + 1) * TP + b9.x - 1) / b9.x, (A.ny / 2 + 1 + b9.y - 1) / b9.y);
                for (int c = 0; c < 4; c++)
                    kb_relax9<K><<<g, b9, 0, s>>>(A, f, u, rev ? 3 - c : c);
                if (nlaunch)
                    *nlaunch += 4;
            }
        }
    }
    static void residual(const Op &A, const double *f, const double *u, double *r, cudaStream_t s)
    {
        const dim3 b(32, 8), g(((A.nx + 2) * TP + 31) / 32, (A.ny + 2 + 7) / 8);
        kb_residual<K><<<g, b, 0, s>>>(A, f, u, r);
    }
    static void restrict_(const Op &A, const CIv &ci, const double *r, double *fc, double *uc, cudaStream_t s,
                          bool vanish)
    {
        const dim3 b(32, 8), g(((A.nx / 2 + 2) * TP + 31) / 32, (A.ny / 2 + 2 + 7) / 8);
        kb_restrict<K><<<g, b, 0, s>>>(A, ci, r, fc, uc, vanish);
    }
    static void resid_restrict(const Op &A, const CIv &ci, const double *f, const double *u, double *fc, double *uc,
                               cudaStream_t s)
    {
        // tiled: every residual evaluated once
        const int ncx = A.nx / 2, ncy = A.ny / 2;
        const dim3 g((ncx + 1 + RT_CX - 1) / RT_CX, (ncy + 1 + RT_CY - 1) / RT_CY);
        if (A.kind == 5)
            kb_resid_restrict_tiled<K, 5><<<g, 256, 0, s>>>(A, ci, f, u, fc, uc);
        else
            kb_resid_restrict_tiled<K, 9><<<g, 256, 0, s>>>(A, ci, f, u, fc, uc);
        kb_coarse_ring0<K><<<(ncx + ncy + 4 + 255) / 256, 256, 0, s>>>(ncx, ncy, ci.pitch, fc, uc);
    }
    static void interp_add(const Op &A, const CIv &ci, const double *ec, const double *u, double *uout, cudaStream_t s,
                           const double *r, int skip)
    {
        const int gxn = ((A.nx + 1) / 2 * TP + 31) / 32;  // CTAs per row for one parity of i
        const dim3 b(32, 8), g(skip && A.kind == 5 ? gxn : 2 * gxn, (A.ny + 7) / 8);
        kb_interp_add<K><<<g, b, 0, s>>>(A, ci, ec, r, u, uout, skip);
    }
    static void r9pair(const Op &A, const double *f, const double *uin, double *uout, cudaStream_t s)
    {
        using R = R9P<K>;
        const int gx = (A.nx + R::TX - 1) / R::TX;
        kb_r9pair<K><<<dim3(gx, A.ny / 2 + 1), R::NT, 0, s>>>(A, f, uin, uout, 0);
        kb_r9pair<K><<<dim3(gx, (A.ny + 1) / 2), R::NT, 0, s>>>(A, f, uin, uout, 1);
    }
    static void rb5(const Op &A, const double *f, const double *uin, double *uout, cudaStream_t s)
    {
        using R = RB5<K>;
        const dim3 g((A.nx + R::TX - 1) / R::TX, (A.ny + R::RC - 1) / R::RC);
        kb_rb5<K><<<g, R::NT, 0, s>>>(A, f, uin, uout);
    }
    static void coarse(const Op &A, const double *Lf, const double *f, double *u, cudaStream_t s)
    {
        const int n = A.nx * A.ny;
        const int threads = n < 32 ? 32 : (n < 1024 ? ((n + 31) / 32) * 32 : 1024);
        kb_coarse_solve<K><<<K, threads, sizeof(double) * n, s>>>(A, Lf, f, u);
    }
    static void dot(const Op &A, const double *a, const double *b, double *partials, double *result, cudaStream_t s)
    {
        kb_dot_partial<K><<<NORM_BLOCKS, 256, 0, s>>>(A, a, b, partials);
        kb_sum_final<<<K, 1024, 0, s>>>(partials, result);
    }
    static void matvec(const Op &A, const double *p, double *q, cudaStream_t s)
    {
        const dim3 b(32, 8), g((A.nx * TP + 31) / 32, (A.yhi - A.ylo + 7) / 8);
        kb_matvec<K><<<g, b, 0, s>>>(A, p, q);
    }
    static void cg_update(const Op &A, const double *sc, int inum, int iden, unsigned mask, const double *p,
                          const double *q, double *x, double *r, cudaStream_t s)
    {
        const dim3 b(32, 8), g((A.nx + 31) / 32, (A.yhi - A.ylo + 7) / 8);
        kb_cg_update<K><<<g, b, 0, s>>>(A, sc, inum, iden, mask, p, q, x, r);
    }
    static void cg_direction(const Op &A, const double *sc, int inum, int iden, unsigned mask, const double *z,
                             double *p, cudaStream_t s)
    {
        const dim3 b(32, 8), g((A.nx + 31) / 32, (A.yhi - A.ylo + 7) / 8);
        kb_cg_direction<K><<<g, b, 0, s>>>(A, sc, inum, iden, mask, z, p);
    }
    static void norm(const Op &A, const double *f, const double *u, double *partials, double *result, cudaStream_t s)
    {
        if (u)
            kb_norm_partial<K, true><<<NORM_BLOCKS, 256, 0, s>>>(A, f, u, partials);
        else
            kb_norm_partial<K, false><<<NORM_BLOCKS, 256, 0, s>>>(A, f, nullptr, partials);
        kb_norm_final<<<K, 1024, 0, s>>>(partials, result);
    }
};

#define BMG_BLOCK_DISPATCH(K, call)           \
    switch (K) {                              \
    case 1: Launch<1>::call; break;           \
    case 2: Launch<2>::call; break;           \
    case 3: Launch<3>::call; break;           \
    case 4: Launch<4>::call; break;           \
    case 5: Launch<5>::call; break;           \
    case 6: Launch<6>::call; break;           \
    case 7: Launch<7>::call; break;           \
    case 8: Launch<8>::call; break;           \
    default: break;                           \
    }

}  // namespace

void launch_relax_block(int K, const Op &A, const double *f, double *u, int nsweeps, cudaStream_t s, int *nlaunch,
                        bool rev)
{
    BMG_BLOCK_DISPATCH(K, relax(A, f, u, nsweeps, s, nlaunch, rev));
}

void launch_residual_block(int K, const Op &A, const double *f, const double *u, double *r, cudaStream_t s)
{
    BMG_BLOCK_DISPATCH(K, residual(A, f, u, r, s));
}

void launch_restrict_block(int K, const Op &A, const CIv &ci, const double *r, double *fc, double *uc,
                           cudaStream_t s, bool vanish)
{
    BMG_BLOCK_DISPATCH(K, restrict_(A, ci, r, fc, uc, s, vanish));
}

void launch_resid_restrict_block(int K, const Op &A, const CIv &ci, const double *f, const double *u, double *fc,
                                 double *uc, cudaStream_t s)
{
    BMG_BLOCK_DISPATCH(K, resid_restrict(A, ci, f, u, fc, uc, s));
}

void launch_interp_add_block(int K, const Op &A, const CIv &ci, const double *ec, double *u, cudaStream_t s,
                             const double *r, int skip, double *uout)
{
    BMG_BLOCK_DISPATCH(K, interp_add(A, ci, ec, u, uout ? uout : u, s, r, skip));
}

void launch_rb5_block(int K, const Op &A, const double *f, const double *uin, double *uout, cudaStream_t s)
{
    if (A.kind == 5) {
        BMG_BLOCK_DISPATCH(K, rb5(A, f, uin, uout, s));
    } else {
        BMG_BLOCK_DISPATCH(K, r9pair(A, f, uin, uout, s));
    }
}

void launch_coarse_solve_block(int K, const Op &A, const double *Lf, const double *f, double *u, cudaStream_t s)
{
    BMG_BLOCK_DISPATCH(K, coarse(A, Lf, f, u, s));
}

void launch_resid_norm_block(int K, const Op &A, const double *f, const double *u, double *partials, double *result,
                             cudaStream_t s)
{
    BMG_BLOCK_DISPATCH(K, norm(A, f, u, partials, result, s));
}

void launch_norm_block(int K, const Op &A, const double *g, double *partials, double *result, cudaStream_t s)
{
    BMG_BLOCK_DISPATCH(K, norm(A, g, nullptr, partials, result, s));
}

__global__ void kb_zero_col(long long n, int K, int col, double *x)
{
    const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (t < n)
        x[t * K + col] = 0.0;
}

void launch_zero_col_block(int K, const Op &A, double *x, int col, cudaStream_t s)
{
    const long long n = (A.ny + 2) * A.pitch;
    kb_zero_col<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(n, K, col, x);
}

void launch_dot_block(int K, const Op &A, const double *a, const double *b, double *partials, double *result,
                      cudaStream_t s)
{
    BMG_BLOCK_DISPATCH(K, dot(A, a, b, partials, result, s));
}

void launch_matvec_block(int K, const Op &A, const double *p, double *q, cudaStream_t s)
{
    BMG_BLOCK_DISPATCH(K, matvec(A, p, q, s));
}

void launch_cg_update_block(int K, const Op &A, const double *sc, int inum, int iden, unsigned mask, const double *p,
                            const double *q, double *x, double *r, cudaStream_t s)
{
    BMG_BLOCK_DISPATCH(K, cg_update(A, sc, inum, iden, mask, p, q, x, r, s));
}

void launch_cg_direction_block(int K, const Op &A, const double *sc, int inum, int iden, unsigned mask,
                               const double *z, double *p, cudaStream_t s)
{
    BMG_BLOCK_DISPATCH(K, cg_direction(A, sc, inum, iden, mask, z, p, s));
}

void launch_zero_block(int K, const Op &A, double *x, cudaStream_t s)
{
    const long long n = (A.ny + 2) * A.pitch * K;
    kb_zero<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(n, x);
}

}  // namespace bmg
