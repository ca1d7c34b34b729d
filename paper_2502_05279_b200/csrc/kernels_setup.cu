// kernels_setup.cu -- setup-phase kernels (S0-S3 of DESIGN.md §2):
// stencil ingest, operator-induced interpolation weights, Galerkin RAP,
// coarsest dense assembly + Cholesky.  fp64 throughout.
//
// Setup arithmetic uses __dmul_rn/__dadd_rn where the oracle evaluates a
// product followed by a sum, so that no FMA contraction changes a rounding:
// level-0 interpolation weights are then bitwise equal to the oracle's.
#include <stdlib.h>

#include <mutex>
#include <utility>

#include "bmg_internal.cuh"

namespace bmg {

// ---------------------------------------------------------------- S0 ingest
// Copy the caller's symmetric-half planes, dropping every coupling whose
// target is a ghost point and zeroing the ring (Dirichlet elimination, SPEC
// S:394; DESIGN §3 c0/c2).  Flags ERR_DIAG if an interior a_O <= 0.
__global__ void k_ingest(int nx, int ny, int kind, long long pitch, const double *__restrict__ sO,
                         const double *__restrict__ sW, const double *__restrict__ sS,
                         const double *__restrict__ sSW, const double *__restrict__ sNW, double *dO, double *dW,
                         double *dS, double *dSW, double *dNW, int *err, int j0)
{
    long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    int j = blockIdx.y + j0;  // global row
    if (i >= pitch)
        return;
    long long p = j * pitch + i;
    bool in = i >= 1 && i <= nx && j >= 1 && j <= ny;
    double o = 0, w = 0, s = 0, sw = 0, nw = 0;
    if (in) {
        o = sO[p];
        if (!(o > 0.0))
            atomicOr(err, ERR_DIAG);
        w = i == 1 ? 0.0 : sW[p];
        s = j == 1 ? 0.0 : sS[p];
        if (kind == 9) {
            sw = (i == 1 || j == 1) ? 0.0 : sSW[p];
            nw = (i == 1 || j == ny) ? 0.0 : sNW[p];
        }
    }
    dO[p] = o;
    dW[p] = w;
    dS[p] = s;
    if (kind == 9) {
        dSW[p] = sw;
        dNW[p] = nw;
    }
}

void launch_ingest(int nx, int ny, int kind, long long pitch, const double *const src[5], double *const dst[5],
                   int *err, cudaStream_t st, int j0, int j1)
{
    if (j1 <= j0)
        return;
    dim3 b(256), g((unsigned)((pitch + 255) / 256), j1 - j0);
    k_ingest<<<g, b, 0, st>>>(nx, ny, kind, pitch, src[0], src[1], src[2], src[3], src[4], dst[0], dst[1], dst[2],
                              dst[3], dst[4], err, j0);
}

// ---------------------------------------------------------------- S1 interpolation
// Operator-induced weights (DESIGN §3 c3: Dendy collapse + BoxMG row-sum
// switch, hard test).  Collapsed couplings of the fine point's row:
//   cW = -(a_W+a_NW+a_SW), cE = -(a_E+a_NE+a_SE), cS = -(a_S+a_SW+a_SE),
//   cN = -(a_N+a_NW+a_NE), sig = -(sum of the 8 off-diagonals), R = a_O - sig.
struct Collapsed {
    double cW, cE, cS, cN, sig, R;
};

__device__ __forceinline__ Collapsed collapse(const Row9 &a)
{
    Collapsed c;
    c.cW = -(a.w + a.nw + a.sw);
    c.cE = -(a.e + a.ne + a.se);
    c.cS = -(a.s + a.sw + a.se);
    c.cN = -(a.n + a.nw + a.ne);
    c.sig = -(a.sw + a.s + a.se + a.w + a.e + a.nw + a.n + a.ne);
    c.R = a.o - c.sig;
    return c;
}

// Phase 1: X points (2I-1,2J) -> LL, LR and Y points (2I,2J-1) -> LB, LA, all stored at (I,J).
__global__ void k_interp_xy(Op A, CIv ci, double *cLL, double *cLR, double *cLB, double *cLA, int ncx, int J0,
                            int J1, int *err)
{
    int I = blockIdx.x * blockDim.x + threadIdx.x + 1;
    int J = blockIdx.y * blockDim.y + threadIdx.y + J0;
    if (I > ncx + 1 || J > J1)
        return;
    long long q = J * ci.pitch + I;
    // X point
    {
        int i = 2 * I - 1, j = 2 * J;
        if (i <= A.nx && j <= A.ny) {
            Row9 a = load_row9(A, j * A.pitch + i);
            Collapsed c = collapse(a);
            double eps = fmin(fabs(c.cW), fabs(c.cE)) / a.o;
            double den = c.cW + c.cE + (c.R > __dmul_rn(eps, c.sig) ? c.R : 0.0);
            if (!(den > 0.0))
                atomicOr(err, ERR_DEN);
            cLL[q] = c.cW / den;
            cLR[q] = c.cE / den;
        }
    }
    // Y point
    {
        int i = 2 * I, j = 2 * J - 1;
        if (i <= A.nx && j <= A.ny) {
            Row9 a = load_row9(A, j * A.pitch + i);
            Collapsed c = collapse(a);
            double eps = fmin(fabs(c.cS), fabs(c.cN)) / a.o;
            double den = c.cS + c.cN + (c.R > __dmul_rn(eps, c.sig) ? c.R : 0.0);
            if (!(den > 0.0))
                atomicOr(err, ERR_DEN);
            cLB[q] = c.cS / den;
            cLA[q] = c.cN / den;
        }
    }
}

// Phase 2: Z points (2I-1,2J-1) -> LNE, LNW, LSE, LSW at (I,J), from the
// neighbouring edge weights X(I,J) north, X(I,J-1) south, Y(I,J) east, Y(I-1,J) west.
__global__ void k_interp_z(Op A, CIv ci, double *cLNE, double *cLNW, double *cLSE, double *cLSW, int ncx, int J0,
                           int J1, int *err)
{
    int I = blockIdx.x * blockDim.x + threadIdx.x + 1;
    int J = blockIdx.y * blockDim.y + threadIdx.y + J0;
    if (I > ncx + 1 || J > J1)
        return;
    int i = 2 * I - 1, j = 2 * J - 1;
    if (i > A.nx || j > A.ny)
        return;
    Row9 a = load_row9(A, j * A.pitch + i);
    Collapsed c = collapse(a);
    double eps = fmin(fmin(fabs(c.cW), fabs(c.cE)), fmin(fabs(c.cS), fabs(c.cN))) / a.o;
    double den = c.sig + (c.R > __dmul_rn(eps, c.sig) ? c.R : 0.0);
    if (!(den > 0.0))
        atomicOr(err, ERR_DEN);
    long long q = J * ci.pitch + I;
    double LR_ = ci.w[CI_LR][q], LL_ = ci.w[CI_LL][q], LA_ = ci.w[CI_LA][q], LB_ = ci.w[CI_LB][q];
    double LAw = ci.w[CI_LA][q - 1], LBw = ci.w[CI_LB][q - 1];
    double LRs = ci.w[CI_LR][q - ci.pitch], LLs = ci.w[CI_LL][q - ci.pitch];
    cLNE[q] = __dadd_rn(__dadd_rn(-a.ne, -__dmul_rn(a.n, LR_)), -__dmul_rn(a.e, LA_)) / den;
    cLNW[q] = __dadd_rn(__dadd_rn(-a.nw, -__dmul_rn(a.n, LL_)), -__dmul_rn(a.w, LAw)) / den;
    cLSE[q] = __dadd_rn(__dadd_rn(-a.se, -__dmul_rn(a.s, LRs)), -__dmul_rn(a.e, LB_)) / den;
    cLSW[q] = __dadd_rn(__dadd_rn(-a.sw, -__dmul_rn(a.s, LLs)), -__dmul_rn(a.w, LBw)) / den;
}

// Coarse rows [J0, J1] (inclusive; single GPU: [1, ncy+1]).  The Z phase reads
// edge weights of row J-1, so a slab computes phase 1 from one row lower.
void launch_setup_interp(const Op &A, double *const ci[8], long long cpitch, int *err, cudaStream_t s, int J0, int J1)
{
    int ncx = A.nx / 2;
    CIv v;
    v.pitch = cpitch;
    v.roff = 0;
    v.nrows = 0;
    for (int k = 0; k < 8; k++)
        v.w[k] = ci[k];
    dim3 b(32, 8);
    dim3 g1((ncx + 1 + 31) / 32, (J1 - J0 + 1 + 7) / 8);
    k_interp_xy<<<g1, b, 0, s>>>(A, v, ci[CI_LL], ci[CI_LR], ci[CI_LB], ci[CI_LA], ncx, J0, J1, err);
    k_interp_z<<<g1, b, 0, s>>>(A, v, ci[CI_LNE], ci[CI_LNW], ci[CI_LSE], ci[CI_LSW], ncx, J0, J1, err);
}

// ---------------------------------------------------------------- S2 Galerkin RAP
// P(g, D): the weight with which fine point g interpolates from coarse D
// (DESIGN §3 c7 row map).  Zero unless g lies in D's 3x3 fine window.
__device__ __forceinline__ double pweight(const CIv &ci, int gx, int gy, int Dx, int Dy)
{
    int dx = gx - 2 * Dx, dy = gy - 2 * Dy;
    if (dx < -1 || dx > 1 || dy < -1 || dy > 1)
        return 0.0;
    bool xo = gx & 1, yo = gy & 1;
    if (!xo && !yo)
        return (dx == 0 && dy == 0) ? 1.0 : 0.0;
    if (xo && !yo) {  // X point, stored at ((gx+1)/2, gy/2)
        if (dy != 0)
            return 0.0;
        long long q = (long long)(gy / 2) * ci.pitch + (gx + 1) / 2;
        return dx > 0 ? ci.w[CI_LL][q] : ci.w[CI_LR][q];
    }
    if (!xo && yo) {  // Y point, stored at (gx/2, (gy+1)/2)
        if (dx != 0)
            return 0.0;
        long long q = (long long)((gy + 1) / 2) * ci.pitch + gx / 2;
        return dy > 0 ? ci.w[CI_LB][q] : ci.w[CI_LA][q];
    }
    long long q = (long long)((gy + 1) / 2) * ci.pitch + (gx + 1) / 2;  // Z point
    if (dx > 0)
        return dy > 0 ? ci.w[CI_LSW][q] : ci.w[CI_LNW][q];
    return dy > 0 ? ci.w[CI_LSE][q] : ci.w[CI_LNE][q];
}

// One thread per interior coarse point C: gather
//   A_c(C,D) = sum_f P(f,C) sum_g A(f,g) P(g,D)   for D in {C, C-(1,0), C-(0,1), C-(1,1), C+(-1,1)}
// over interior fine f in C's 3x3 window and interior g in f's 3x3 window.
__global__ void k_rap(Op A, CIv ci, int ncx, int ncy, long long cpitch, double *cO, double *cW, double *cS,
                      double *cSW, double *cNW, int J0, int J1)
{
    int I = blockIdx.x * blockDim.x + threadIdx.x + 1;
    int J = blockIdx.y * blockDim.y + threadIdx.y + J0;
    if (I > ncx || J > J1)
        return;
    const int tx[5] = {0, -1, 0, -1, -1};
    const int ty[5] = {0, 0, -1, -1, 1};
    double acc[5] = {0, 0, 0, 0, 0};
    for (int fy = 2 * J - 1; fy <= 2 * J + 1; fy++) {
        if (fy < 1 || fy > A.ny)
            continue;
        for (int fx = 2 * I - 1; fx <= 2 * I + 1; fx++) {
            if (fx < 1 || fx > A.nx)
                continue;
            double wf = pweight(ci, fx, fy, I, J);
            if (wf == 0.0)
                continue;
            Row9 a = load_row9(A, fy * A.pitch + fx);
            const double av[9] = {a.sw, a.s, a.se, a.w, a.o, a.e, a.nw, a.n, a.ne};
#pragma unroll
            for (int d = 0; d < 9; d++) {
                int gx = fx + (d % 3) - 1, gy = fy + (d / 3) - 1;
                if (av[d] == 0.0 || gx < 1 || gx > A.nx || gy < 1 || gy > A.ny)
                    continue;
                double wa = wf * av[d];
#pragma unroll
                for (int k = 0; k < 5; k++) {
                    int Dx = I + tx[k], Dy = J + ty[k];
                    if (Dx < 1 || Dy < 1 || Dy > ncy)
                        continue;
                    acc[k] += wa * pweight(ci, gx, gy, Dx, Dy);
                }
            }
        }
    }
    long long q = J * cpitch + I;
    cO[q] = acc[0];
    cW[q] = acc[1];
    cS[q] = acc[2];
    cSW[q] = acc[3];
    cNW[q] = acc[4];
}

// ---- tiled RAP: the same gather, the same terms in the same order as k_rap (so the
// same bits), with the P lookups resolved at compile time and the operands staged
// in shared memory.  For coarse C = (I,J), fine f = (2I-1+UX, 2J-1+UY) and its
// stencil direction d (g = f + off_d), and target D = C + t_k, the weight P(g, D)
// is zero, one, or ONE interpolation weight at a FIXED offset from (I,J): g's
// position relative to (2I,2J) is (ex,ey) = (UX-1+ddx, UY-1+ddy) in [-2,2]^2.
struct PwSel {
    int kind;  // 0: zero, 1: one, 2: weight plane `plane` at coarse (I+oi, J+oj)
    int plane, oi, oj;
};
__host__ __device__ constexpr PwSel pw_sel(int ex, int ey, int tx, int ty)
{
    const int dx = ex - 2 * tx, dy = ey - 2 * ty;
    if (dx < -1 || dx > 1 || dy < -1 || dy > 1)
        return {0, 0, 0, 0};
    const bool xo = (ex & 1) != 0, yo = (ey & 1) != 0;
    if (!xo && !yo)
        return (dx == 0 && dy == 0) ? PwSel{1, 0, 0, 0} : PwSel{0, 0, 0, 0};
    if (xo && !yo)  // X point, stored at ((gx+1)/2, gy/2)
        return dy != 0 ? PwSel{0, 0, 0, 0} : PwSel{2, dx > 0 ? CI_LL : CI_LR, (ex + 1) / 2, ey / 2};
    if (!xo && yo)  // Y point, stored at (gx/2, (gy+1)/2)
        return dx != 0 ? PwSel{0, 0, 0, 0} : PwSel{2, dy > 0 ? CI_LB : CI_LA, ex / 2, (ey + 1) / 2};
    return {2, dx > 0 ? (dy > 0 ? CI_LSW : CI_LNW) : (dy > 0 ? CI_LSE : CI_LNE), (ex + 1) / 2, (ey + 1) / 2};
}

constexpr int RAP_TC = 32, RAP_TR = 8;                     // coarse tile
constexpr int RAP_FW = 2 * RAP_TC + 2, RAP_FH = 2 * RAP_TR + 3;  // fine planes: x in [2I0-1, 2I0+2TC], y in [2J0-2, 2J0+2TR]
constexpr int RAP_CW = RAP_TC + 2, RAP_CH = RAP_TR + 2;          // weights: I in [I0-1, I0+TC], J in [J0-1, J0+TR]
constexpr int RAP_TX[5] = {0, -1, 0, -1, -1}, RAP_TY[5] = {0, 0, -1, -1, 1};

struct RapSm {
    double pl[5][RAP_FH][RAP_FW];  // O W S SW NW
    double ci[8][RAP_CH][RAP_CW];
};

// weight P(g, D) for g at (EX,EY) from (2I,2J), D = C + t_K; cx, cy: thread's (I,J) in the weight tile
template <int EX, int EY, int K>
__device__ __forceinline__ double pw_tile(const RapSm &sm, int cx, int cy)
{
    constexpr PwSel q = pw_sel(EX, EY, RAP_TX[K], RAP_TY[K]);
    if constexpr (q.kind == 0)
        return 0.0;
    else if constexpr (q.kind == 1)
        return 1.0;
    else
        return sm.ci[q.plane][cy + q.oj][cx + q.oi];
}

// the k_rap contributions of stencil direction DD of fine point f = (2I-1+UX, 2J-1+UY)
template <int UX, int UY, int DD, int K>
__device__ __forceinline__ void rap_term(const RapSm &sm, int cx, int cy, double wa, const bool *vk, double *acc)
{
    constexpr int EX = UX - 1 + DD % 3 - 1, EY = UY - 1 + DD / 3 - 1;
    constexpr PwSel q = pw_sel(EX, EY, RAP_TX[K], RAP_TY[K]);
    if constexpr (q.kind != 0) {  // a structurally zero weight adds an exact 0 in k_rap
        if (vk[K])
            acc[K] = __fma_rn(wa, pw_tile<EX, EY, K>(sm, cx, cy), acc[K]);
    }
}

template <int UX, int UY, int DD>
__device__ __forceinline__ void rap_dir(const RapSm &sm, int cx, int cy, double wf, const double *av, const bool *vk,
                                        double *acc)
{
    const double wa = __dmul_rn(wf, av[DD]);
    rap_term<UX, UY, DD, 0>(sm, cx, cy, wa, vk, acc);
    rap_term<UX, UY, DD, 1>(sm, cx, cy, wa, vk, acc);
    rap_term<UX, UY, DD, 2>(sm, cx, cy, wa, vk, acc);
    rap_term<UX, UY, DD, 3>(sm, cx, cy, wa, vk, acc);
    rap_term<UX, UY, DD, 4>(sm, cx, cy, wa, vk, acc);
}

template <int UX, int UY, int... DD>
__device__ __forceinline__ void rap_fine(const RapSm &sm, int cx, int cy, int fxl, int fyl, const bool *vk, double *acc,
                                         std::integer_sequence<int, DD...>)
{
    constexpr PwSel wq = pw_sel(UX - 1, UY - 1, 0, 0);  // P(f, C)
    if constexpr (wq.kind != 0) {
        const double wf = pw_tile<UX - 1, UY - 1, 0>(sm, cx, cy);
        // f's full row (fig:stencil_operator order SW,S,SE,W,O,E,NW,N,NE) from the staged planes;
        // fxl, fyl: f's position in the plane tile
        const int x = fxl + UX, y = fyl + UY;
        const double av[9] = {sm.pl[3][y][x],     sm.pl[2][y][x],     sm.pl[4][y - 1][x + 1],
                              sm.pl[1][y][x],     sm.pl[0][y][x],     sm.pl[1][y][x + 1],
                              sm.pl[4][y][x],     sm.pl[2][y + 1][x], sm.pl[3][y + 1][x + 1]};
        (rap_dir<UX, UY, DD>(sm, cx, cy, wf, av, vk, acc), ...);
    }
}

// One CTA per RAP_TC x RAP_TR coarse tile, one thread per coarse point.  Same
// definition as k_rap: A_c(C,D) = sum_f P(f,C) sum_g A(f,g) P(g,D), terms in the order
// f (row-major over C's 3x3 window), stencil direction, target D.
__global__ void __launch_bounds__(RAP_TC *RAP_TR) k_rap_tiled(Op A, CIv ci, int ncx, int ncy, long long cpitch,
                                                             double *cO, double *cW, double *cS, double *cSW,
                                                             double *cNW, int J0, int J1)
{
    extern __shared__ __align__(16) unsigned char rap_raw[];
    RapSm &sm = *reinterpret_cast<RapSm *>(rap_raw);
    const int I0 = blockIdx.x * RAP_TC + 1, Jt = J0 + blockIdx.y * RAP_TR;
    const int tid = threadIdx.x;
    // stage the fine planes and the weights (zero outside the stored rows / the padded
    // grid): one warp per row, lanes along it -- no index divisions, constant plane indices
    const int fx0 = 2 * I0 - 1, fy0 = 2 * Jt - 2;
    const int ylo = max(A.roff, 0), yhi = min(A.ny + 1, A.roff + A.nrows - 1);
    const int warp = tid >> 5, lane = tid & 31, nw = blockDim.x >> 5;
    // cp.async with zero fill (source size 0 off the grid): every element of the tile in
    // flight at once -- element-by-element loads into registers left one DRAM round trip
    // per row chunk on each warp's critical path (ncu: 54 % long-scoreboard stalls)
    const double *dummy = A.O;  // a valid global address for the zero-fill copies (nothing is read)
    auto cp8 = [dummy](double *dst, const double *src, bool ok) {
        const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(ok ? src : dummy), "r"(ok ? 8 : 0)
                     : "memory");
    };
    auto stage_plane = [&](const double *src, double (*dst)[RAP_FW]) {
        for (int r = warp; r < RAP_FH; r += nw) {
            const int gy = fy0 + r;
            const bool rin = src && gy >= ylo && gy <= yhi;
            const double *row = rin ? src + (long long)gy * A.pitch : nullptr;
            for (int c = lane; c < RAP_FW; c += 32) {
                const int gx = fx0 + c;
                const bool ok = rin && gx <= A.nx + 1;
                cp8(&dst[r][c], ok ? row + gx : nullptr, ok);
            }
        }
    };
    stage_plane(A.O, sm.pl[0]);
    stage_plane(A.W, sm.pl[1]);
    stage_plane(A.S, sm.pl[2]);
    stage_plane(A.kind == 9 ? A.SW : nullptr, sm.pl[3]);
    stage_plane(A.kind == 9 ? A.NW : nullptr, sm.pl[4]);
    const int cylo = max(ci.roff, 0), cyhi = min(ncy + 1, ci.roff + ci.nrows - 1);
#pragma unroll
    for (int k = 0; k < 8; k++) {
        const double *src = ci.w[k];
        for (int r = warp; r < RAP_CH; r += nw) {
            const int cy = Jt - 1 + r;
            const bool rin = cy >= cylo && cy <= cyhi;
            for (int c = lane; c < RAP_CW; c += 32) {
                const int cx = I0 - 1 + c;
                const bool ok = rin && cx <= ncx + 1;
                cp8(&sm.ci[k][r][c], ok ? src + (long long)cy * ci.pitch + cx : nullptr, ok);
            }
        }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    const int tx = tid % RAP_TC, ty = tid / RAP_TC;
    const int I = I0 + tx, J = Jt + ty;
    if (I > ncx || J > J1)
        return;
    // target D = C + t_k exists (k_rap's test): t = (0,0), (-1,0), (0,-1), (-1,-1), (-1,+1)
    const bool vk[5] = {true, I > 1, J > 1, I > 1 && J > 1, I > 1 && J < ncy};
    double acc[5] = {0, 0, 0, 0, 0};
    const int cx = tx + 1, cy = ty + 1;          // (I,J) in the weight tile
    const int fxl = 2 * tx, fyl = 2 * ty + 1;    // f = (2I-1+UX, 2J-1+UY) -> tile (fxl+UX, fyl+UY)
    using Dirs = std::make_integer_sequence<int, 9>;
    rap_fine<0, 0>(sm, cx, cy, fxl, fyl, vk, acc, Dirs{});
    rap_fine<1, 0>(sm, cx, cy, fxl, fyl, vk, acc, Dirs{});
    rap_fine<2, 0>(sm, cx, cy, fxl, fyl, vk, acc, Dirs{});
    rap_fine<0, 1>(sm, cx, cy, fxl, fyl, vk, acc, Dirs{});
    rap_fine<1, 1>(sm, cx, cy, fxl, fyl, vk, acc, Dirs{});
    rap_fine<2, 1>(sm, cx, cy, fxl, fyl, vk, acc, Dirs{});
    rap_fine<0, 2>(sm, cx, cy, fxl, fyl, vk, acc, Dirs{});
    rap_fine<1, 2>(sm, cx, cy, fxl, fyl, vk, acc, Dirs{});
    rap_fine<2, 2>(sm, cx, cy, fxl, fyl, vk, acc, Dirs{});
    const long long q = J * cpitch + I;
    cO[q] = acc[0];
    cW[q] = acc[1];
    cS[q] = acc[2];
    cSW[q] = acc[3];
    cNW[q] = acc[4];
}

// Coarse rows [J0, J1] (inclusive; single GPU: [1, ncy]).
void launch_setup_rap(const Op &A, const CIv &ci, int ncx, int ncy, long long cpitch, double *const dst[5],
                      cudaStream_t s, int J0, int J1)
{
    if (J1 < J0)
        return;
    static const bool ref = getenv("BMG_RAP_REF") != nullptr;  // the untiled k_rap (A/B checks)
    if (ref) {
        dim3 b(32, 4), g((ncx + 31) / 32, (J1 - J0 + 1 + 3) / 4);
        k_rap<<<g, b, 0, s>>>(A, ci, ncx, ncy, cpitch, dst[0], dst[1], dst[2], dst[3], dst[4], J0, J1);
        return;
    }
    {  // the dynamic shared-memory limit of k_rap_tiled, once per device
        static std::once_flag once[64];
        int dev = 0;
        cudaGetDevice(&dev);
        std::call_once(once[dev & 63], []() {
            cudaFuncSetAttribute(k_rap_tiled, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(RapSm));
        });
    }
    dim3 g((ncx + RAP_TC - 1) / RAP_TC, (J1 - J0 + RAP_TR) / RAP_TR);
    k_rap_tiled<<<g, RAP_TC * RAP_TR, sizeof(RapSm), s>>>(A, ci, ncx, ncy, cpitch, dst[0], dst[1], dst[2], dst[3],
                                                         dst[4], J0, J1);
}

// ---------------------------------------------------------------- S3 coarsest factor
// Dense operator of the coarsest level, lexicographic order (x fastest).
__global__ void k_assemble_dense(Op A, double *M)
{
    int n = A.nx * A.ny;
    int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n)
        return;
    int i = p % A.nx + 1, j = p / A.nx + 1;
    Row9 a = load_row9(A, j * A.pitch + i);
    const double av[9] = {a.sw, a.s, a.se, a.w, a.o, a.e, a.nw, a.n, a.ne};
    for (int d = 0; d < 9; d++) {
        int qi = i + (d % 3) - 1, qj = j + (d / 3) - 1;
        if (qi < 1 || qi > A.nx || qj < 1 || qj > A.ny)
            continue;
        M[(long long)p * n + (qj - 1) * A.nx + (qi - 1)] = av[d];
    }
}

void launch_assemble_dense(const Op &A, double *M, cudaStream_t s)
{
    int n = A.nx * A.ny;
    cudaMemsetAsync(M, 0, sizeof(double) * (size_t)n * n, s);
    k_assemble_dense<<<(n + 127) / 128, 128, 0, s>>>(A, M);
}

// Right-looking dense Cholesky in one CTA (the coarsest system has 9-21
// unknowns on the BASELINE configs).  Lower triangle <- L, upper <- 0.
__global__ void k_chol_factor(int n, double *M, int *err)
{
    __shared__ double piv;
    for (int j = 0; j < n; j++) {
        if (threadIdx.x == 0) {
            double d = M[(long long)j * n + j];
            if (!(d > 0.0)) {
                atomicOr(err, ERR_PIVOT);
                d = 1.0;
            }
            piv = sqrt(d);
            M[(long long)j * n + j] = piv;
        }
        __syncthreads();
        for (int i = j + 1 + threadIdx.x; i < n; i += blockDim.x)
            M[(long long)i * n + j] /= piv;
        __syncthreads();
        long long m = n - j - 1;
        for (long long t = threadIdx.x; t < m * m; t += blockDim.x) {
            int i = j + 1 + (int)(t / m), k = j + 1 + (int)(t % m);
            if (k <= i)
                M[(long long)i * n + k] -= M[(long long)i * n + j] * M[(long long)k * n + j];
        }
        __syncthreads();
    }
    for (long long t = threadIdx.x; t < (long long)n * n; t += blockDim.x) {
        int i = (int)(t / n), k = (int)(t % n);
        if (k > i)
            M[t] = 0.0;
    }
}

void launch_chol_factor(int n, double *M, int *err, cudaStream_t s) { k_chol_factor<<<1, 1024, 0, s>>>(n, M, err); }

}  // namespace bmg
