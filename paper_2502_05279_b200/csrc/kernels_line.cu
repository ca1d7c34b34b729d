// kernels_line.cu -- zebra line Gauss-Seidel (DESIGN.md §3 c11; the "Line"
// relaxation box of fig:vcycle_flowchart, which the paper names but
// does not define).
//
// One colour pass solves every line of that colour exactly: x-lines are grid
// rows (unknowns i = 1..nx of row j, colour j mod 2), y-lines grid columns
// (unknowns j = 1..ny of column i, colour i mod 2); colour 0 first.  The line
// system is tridiagonal (lo = W or S, diagonal O, up = E or N); the couplings
// to the two neighbouring lines (the other colour) move to the right-hand
// side.  A 9-point stencil couples a line only to its neighbours, so the lines
// of one colour are independent -- the batch of tridiagonal solves is the
// data-parallel work.
//
// B200 mapping (HBM-bound: one pass reads ~10 doubles per point of the colour
// and writes one).  A line of n unknowns is cut into nch chunks
// of <= LINE_M points; a thread owns one (line, chunk), consecutive threads of
// a warp own the same chunk of consecutive lines (so the grid loads of a y-line
// warp are row-contiguous).  The chunked solve is the partition ("modified
// Thomas") method: each thread eliminates its chunk in registers down to
//     x_k = D'_k - A'_k x_first - C'_k x_last          (interior k)
// plus two reduced equations for its chunk ends, which couple only to the
// neighbouring chunks' ends: the reduced system of 2*nch unknowns per line is
// again tridiagonal with unit diagonal.  Three launches per colour:
//   k_line_elim    rhs + chunk elimination; chunk interiors (A',C',D') and the
//                  reduced rows go to a scratch buffer (coalesced [k][line]);
//   k_line_reduced one warp per line: the reduced system in shared memory,
//                  solved by the same partition method one level up (lane
//                  sub-chunks, then the 64 lane ends); writes the chunk-end
//                  unknowns into u;
//   k_line_back    interiors x_k = D' - A' x_first - C' x_last into u.
// A line that fits one chunk (n <= LINE_M) is solved completely by
// k_line_elim (no scratch).  Pivots use rcp_pos (FMA pipe, bmg_internal.cuh):
// the line blocks of an SPD operator are SPD, so every pivot is positive
// (checked once at setup by k_line_pivots -> BMG_ENOTSPD).
#include <mutex>
#include "bmg_internal.cuh"
#include "line.cuh"

namespace bmg {

namespace {

// Geometry of one colour pass.  Line l of colour c has line coordinate
// 2l + 2 (c = 0) or 2l + 1 (c = 1); position k in [0, n) along it.
struct LineGeo {
    int Y;       // 0: x-lines (rows), 1: y-lines (columns)
    int c;       // colour
    int n;       // unknowns per line
    int nl;      // lines of this colour
    int nlmax;   // scratch stride: max lines of a colour, (#lines + 1) / 2
    int nch;     // chunks per line
    __device__ __forceinline__ int line_coord(int l) const { return 2 * l + (c == 0 ? 2 : 1); }
    // p * n < 2^31: n <= LINE_NMAX = 32768, p <= nch <= 4096
    __device__ __forceinline__ int chunk_start(int p) const { return (p * n) / nch; }
};

// Thread -> (line l, chunk p).  y-lines: consecutive threads take consecutive
// lines (their points of a row are 16 B apart); x-lines: consecutive threads
// take consecutive chunks of one row (the row is read contiguously by the CTA).
template <int Y>
__device__ __forceinline__ void line_chunk(int &l, int &p)
{
    if (Y) {
        l = blockIdx.x * blockDim.x + threadIdx.x;
        p = blockIdx.y;
    } else {
        p = blockIdx.x * blockDim.x + threadIdx.x;
        l = blockIdx.y;
    }
}

// scratch slot of interior position k of line l: y-lines [k][line] (a warp's
// stores coalesce), x-lines [line][k]
template <int Y>
__device__ __forceinline__ long long scr_index(const LineGeo &g, int l, int k)
{
    return Y ? (long long)k * g.nlmax + l : (long long)l * g.n + k;
}

}  // namespace

struct LineScratch {
    double *a, *c, *d;          // chunk interiors: scr_index (y: [k][line], x: [line][k])
    double *rlo, *rup, *rrhs;   // reduced rows:    [l * 2nch + q], q = 2p (first), 2p+1 (last)
};

// Pass 1: right-hand side + partition elimination of one chunk (registers).
// x-lines stage the CTA's row segment (128 chunks) through shared memory: the
// per-point coefficients and right-hand side are formed by consecutive threads
// on consecutive points (coalesced), each thread then reads its chunk from the
// padded arrays, and the chunk interiors go back out through shared memory.
constexpr int XSEG = 128 * LINE_M;                 // points per x-line CTA
__device__ __forceinline__ int xpad(int x) { return x + x / LINE_M; }

template <int Y>
__global__ void __launch_bounds__(128) k_line_elim(Op A, const double *__restrict__ f, double *__restrict__ u,
                                                   LineGeo g, LineScratch sc)
{
    int l, p;
    line_chunk<Y>(l, p);
    __shared__ double xs[Y ? 1 : 4][Y ? 1 : XSEG + XSEG / LINE_M];
    int s_lo = 0, s_hi = 0;
    if (!Y) {  // whole CTA: same row l, chunks [p0, p0 + 128)
        const int p0 = blockIdx.x * blockDim.x;
        const int p1 = p0 + (int)blockDim.x < g.nch ? p0 + (int)blockDim.x : g.nch;
        s_lo = g.chunk_start(p0);
        s_hi = g.chunk_start(p1);
        const int lc0 = g.line_coord(l);
        for (int x = threadIdx.x; x < s_hi - s_lo; x += blockDim.x) {
            double lo_, di_, up_, d_;
            line_row<0>(A, f, u, lc0, s_lo + x, lo_, di_, up_, d_);
            const int i = xpad(x);
            xs[0][i] = lo_;
            xs[1][i] = di_;
            xs[2][i] = up_;
            xs[3][i] = d_;
        }
        __syncthreads();
    }
    const bool active = l < g.nl && p < g.nch;
    const int lc = g.line_coord(l);
    const int s0 = active ? g.chunk_start(p) : 0, m = active ? g.chunk_start(p + 1) - s0 : 0;
    double a[LINE_M], c[LINE_M], d[LINE_M];
    // forward, fused with the loads: rows 0, 1 normalised; rows k >= 2 lose
    // x_{k-1} and gain x_0 (coefficient kept in a[k])
#pragma unroll
    for (int k = 0; k < LINE_M; k++)
        if (k < m) {
            double b;
            if (Y) {
                line_row<Y>(A, f, u, lc, s0 + k, a[k], b, c[k], d[k]);
            } else {
                const int i = xpad(s0 - s_lo + k);
                a[k] = xs[0][i];
                b = xs[1][i];
                c[k] = xs[2][i];
                d[k] = xs[3][i];
            }
            if (k < 2) {
                const double r = rcp_pos(b);
                d[k] *= r;
                a[k] *= r;
                c[k] *= r;
            } else {
                const double r = rcp_pos(fma(-a[k], c[k - 1], b));
                d[k] = r * fma(-a[k], d[k - 1], d[k]);
                a[k] = -r * a[k] * a[k - 1];
                c[k] = r * c[k];
            }
        }
    // backward: rows m-3 .. 1 lose x_{k+1}, gain x_{m-1} (in c[k])
#pragma unroll
    for (int k = LINE_M - 3; k >= 1; k--)
        if (k <= m - 3) {
            d[k] = fma(-c[k], d[k + 1], d[k]);
            a[k] = fma(-c[k], a[k + 1], a[k]);
            c[k] = -c[k] * c[k + 1];
        }
    // row 0 loses x_1: a_0 x_{-1} + x_0 + c_0 x_{m-1} = d_0
    if (m >= 3) {
        const double r = rcp_pos(fma(-c[0], a[1], 1.0));
        d[0] = r * fma(-c[0], d[1], d[0]);
        a[0] = r * a[0];
        c[0] = -r * c[0] * c[1];
    }
    if (g.nch == 1 && active) {
        // whole line in this chunk: solve the 2x2 end system, then the interior
        double x0 = d[0], xl = d[0];
        if (m > 1) {
            double am = 0.0, dm = 0.0;  // row m-1: last write wins (no dynamic index)
#pragma unroll
            for (int k = 1; k < LINE_M; k++)
                if (k < m) {
                    am = a[k];
                    dm = d[k];
                }
            xl = fma(-am, d[0], dm) * rcp_pos(fma(-am, c[0], 1.0));
            x0 = fma(-c[0], xl, d[0]);
        }
#pragma unroll
        for (int k = 0; k < LINE_M; k++)
            if (k < m) {
                const double x = k == 0 ? x0 : (k == m - 1 ? xl : fma(-c[k], xl, fma(-a[k], x0, d[k])));
                u[grid_index<Y>(A, lc, s0 + k)] = x;
            }
        return;
    }
    if (g.nch == 1)
        return;  // (x-lines: the whole CTA, nothing staged out)
    if (Y) {
#pragma unroll
        for (int k = 1; k < LINE_M - 1; k++)
            if (k < m - 1) {
                const long long q = scr_index<Y>(g, l, s0 + k);
                sc.a[q] = a[k];
                sc.c[q] = c[k];
                sc.d[q] = d[k];
            }
    } else {
        __syncthreads();  // every thread has read its chunk
#pragma unroll
        for (int k = 1; k < LINE_M - 1; k++)
            if (k < m - 1) {
                const int i = xpad(s0 - s_lo + k);
                xs[0][i] = a[k];
                xs[2][i] = c[k];
                xs[3][i] = d[k];
            }
        __syncthreads();
        // coalesced copy of the segment (chunk-end slots carry stale values K3 never reads)
        for (int x = threadIdx.x; x < s_hi - s_lo; x += blockDim.x) {
            const long long q = scr_index<0>(g, l, s_lo + x);
            const int i = xpad(x);
            sc.a[q] = xs[0][i];
            sc.c[q] = xs[2][i];
            sc.d[q] = xs[3][i];
        }
    }
    if (!active)
        return;
    // reduced rows: first (lo -> last of chunk p-1, up -> own last), last (lo -> own first, up -> first of p+1)
    const long long q0 = (long long)l * (2 * g.nch) + 2 * p, q1 = q0 + 1;  // line-major
    double al = a[0], cl = c[0], dl = d[0];  // row m-1: last write wins (no dynamic index)
#pragma unroll
    for (int k = 1; k < LINE_M; k++)
        if (k < m) {
            al = a[k];
            cl = c[k];
            dl = d[k];
        }
    sc.rlo[q0] = a[0];
    sc.rup[q0] = c[0];
    sc.rrhs[q0] = d[0];
    sc.rlo[q1] = al;
    sc.rup[q1] = cl;
    sc.rrhs[q1] = dl;
}

// Pass 2: the reduced system of each line (2*nch unknowns, unit diagonal:
// lo_q x_{q-1} + x_q + up_q x_{q+1} = r_q), ONE WARP per line.  Short systems
// (nq < 96): lane 0 runs Thomas in shared memory.  Otherwise the partition
// method one level up: lane t owns rows [t*nq/32, (t+1)*nq/32) (shared memory,
// lane-interleaved: row k of lane t at k*32 + t, no bank conflicts) and
// eliminates them down to its two ends; the 64 lane-end equations (two per
// lane, in registers) are solved by parallel cyclic reduction over warp
// shuffles (6 steps); each lane then recovers its interior.  The serial chains
// use the correctly rounded __drcp_rn (latency, not throughput, bounds them).
// The chunk-end unknowns x_q go into u.
template <int Y>
__global__ void __launch_bounds__(128) k_line_reduced(Op A, double *__restrict__ u, LineGeo g, LineScratch sc)
{
    extern __shared__ double sm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int l = blockIdx.x * (blockDim.x >> 5) + warp;
    if (l >= g.nl)
        return;  // whole warp
    const int nq = 2 * g.nch;
    const int mmax = (nq + 31) / 32;
    double *lo = sm + (size_t)warp * 3 * 32 * mmax, *up = lo + 32 * mmax, *rh = up + 32 * mmax;
    const long long base = (long long)l * nq;
    const int lc = g.line_coord(l);
    if (nq < 96) {
        for (int q = lane; q < nq; q += 32) {
            lo[q] = sc.rlo[base + q];
            up[q] = sc.rup[base + q];
            rh[q] = sc.rrhs[base + q];
        }
        __syncwarp();
        if (lane == 0) {
            double gp = up[0], ep = rh[0];
            for (int q = 1; q < nq; q++) {
                const double r = __drcp_rn(fma(-lo[q], gp, 1.0));
                ep = r * fma(-lo[q], ep, rh[q]);
                gp = up[q] * r;
                up[q] = gp;
                rh[q] = ep;
            }
            double x = ep;
            for (int q = nq - 2; q >= 0; q--) {
                x = fma(-up[q], x, rh[q]);
                rh[q] = x;
            }
        }
        __syncwarp();
        for (int q = lane; q < nq; q += 32) {
            const int p = q >> 1;
            const int at = (q & 1) ? g.chunk_start(p + 1) - 1 : g.chunk_start(p);
            u[grid_index<Y>(A, lc, at)] = rh[q];
        }
        return;
    }
    const int s0 = (lane * nq) / 32, m = ((lane + 1) * nq) / 32 - s0;  // m >= 3
    double *a = lo + lane, *c = up + lane, *d = rh + lane;             // row k at [k*32]
    // coalesced loads (lane L reads rows it*32 + L), stored to the owner's slot;
    // batches of 16 rows per lane in flight (the loads, not the arithmetic, bound
    // this kernel otherwise)
    for (int q0 = 0; q0 < nq; q0 += 16 * 32) {
        double vl[16], vu[16], vr[16];
#pragma unroll
        for (int b = 0; b < 16; b++) {
            const int q = q0 + b * 32 + lane;
            if (q < nq) {
                vl[b] = sc.rlo[base + q];
                vu[b] = sc.rup[base + q];
                vr[b] = sc.rrhs[base + q];
            }
        }
#pragma unroll
        for (int b = 0; b < 16; b++) {
            const int q = q0 + b * 32 + lane;
            if (q < nq) {
                int t = (q * 32 + 31) / nq;  // owner: the t with t*nq/32 <= q < (t+1)*nq/32
                if ((t * nq) / 32 > q)
                    t--;
                const int i = (q - (t * nq) / 32) * 32 + t;
                lo[i] = vl[b];
                up[i] = vu[b];
                rh[i] = vr[b];
            }
        }
    }
    __syncwarp();
    for (int k = 2; k < m; k++) {
        const double r = __drcp_rn(fma(-a[32 * k], c[32 * (k - 1)], 1.0));
        d[32 * k] = r * fma(-a[32 * k], d[32 * (k - 1)], d[32 * k]);
        a[32 * k] = -r * a[32 * k] * a[32 * (k - 1)];
        c[32 * k] = r * c[32 * k];
    }
    for (int k = m - 3; k >= 1; k--) {
        d[32 * k] = fma(-c[32 * k], d[32 * (k + 1)], d[32 * k]);
        a[32 * k] = fma(-c[32 * k], a[32 * (k + 1)], a[32 * k]);
        c[32 * k] = -c[32 * k] * c[32 * (k + 1)];
    }
    {
        const double r = __drcp_rn(fma(-c[0], a[32], 1.0));
        d[0] = r * fma(-c[0], d[32], d[0]);
        a[0] = r * a[0];
        c[0] = -r * c[0] * c[32];
    }
    // lane ends: equation 2t = first row of lane t, 2t+1 = its last row
    Eq e0 = {a[0], 1.0, c[0], d[0]};
    Eq e1 = {a[32 * (m - 1)], 1.0, c[32 * (m - 1)], d[32 * (m - 1)]};
    pcr64(e0, e1, lane);
    const double x0 = e0.r * __drcp_rn(e0.d), xl = e1.r * __drcp_rn(e1.d);
    d[0] = x0;
    d[32 * (m - 1)] = xl;
    for (int k = 1; k < m - 1; k++)
        d[32 * k] = fma(-c[32 * k], xl, fma(-a[32 * k], x0, d[32 * k]));
    for (int k = 0; k < m; k++) {
        const int q = s0 + k, p = q >> 1;
        const int at = (q & 1) ? g.chunk_start(p + 1) - 1 : g.chunk_start(p);
        u[grid_index<Y>(A, lc, at)] = d[32 * k];
    }
}

// Pass 3: chunk interiors from the chunk ends.
template <int Y>
__global__ void __launch_bounds__(128) k_line_back(Op A, double *__restrict__ u, LineGeo g, LineScratch sc)
{
    int l, p;
    line_chunk<Y>(l, p);
    if (l >= g.nl || p >= g.nch)
        return;
    const int lc = g.line_coord(l);
    const int s0 = g.chunk_start(p), m = g.chunk_start(p + 1) - s0;
    const double x0 = u[grid_index<Y>(A, lc, s0)], xl = u[grid_index<Y>(A, lc, s0 + m - 1)];
#pragma unroll
    for (int k = 1; k < LINE_M - 1; k++)
        if (k < m - 1) {
            const long long q = scr_index<Y>(g, l, s0 + k);
            u[grid_index<Y>(A, lc, s0 + k)] = fma(-sc.c[q], xl, fma(-sc.a[q], x0, sc.d[q]));
        }
}

// Setup check (c11): Thomas pivots of every line (both colours) must be > 0.
template <int Y>
__global__ void k_line_pivots(Op A, int *err)
{
    const int line = blockIdx.x * blockDim.x + threadIdx.x + 1;
    const int nl = Y ? A.nx : A.ny, n = Y ? A.ny : A.nx;
    if (line > nl)
        return;
    const long long P = A.pitch, step = Y ? P : 1;
    long long p = Y ? P + line : line * P + 1;
    double beta = A.O[p];
    bool ok = beta > 0.0;
    for (int k = 1; k < n && ok; k++) {
        const double up_prev = Y ? A.S[p + P] : A.W[p + 1];
        p += step;
        const double lo = Y ? A.S[p] : A.W[p];
        beta = A.O[p] - lo * (up_prev / beta);
        ok = beta > 0.0;
    }
    if (!ok)
        atomicOr(err, ERR_LINE);
}

static LineGeo make_geo(const Op &A, int Y, int c)
{
    LineGeo g;
    g.Y = Y;
    g.c = c;
    const int lines = Y ? A.nx : A.ny;
    g.n = Y ? A.ny : A.nx;
    g.nl = c == 0 ? lines / 2 : (lines + 1) / 2;
    g.nlmax = (lines + 1) / 2;
    g.nch = (g.n + LINE_M - 1) / LINE_M;
    return g;
}

size_t line_scratch_doubles(int nx, int ny)
{
    size_t best = 0;
    for (int Y = 0; Y < 2; Y++) {
        const int lines = Y ? nx : ny, n = Y ? ny : nx;
        const size_t nlmax = (size_t)(lines + 1) / 2, nch = (size_t)(n + LINE_M - 1) / LINE_M;
        const size_t need = 3 * (size_t)n * nlmax + 3 * 2 * nch * nlmax;
        if (need > best)
            best = need;
    }
    return best;
}

static LineScratch carve(double *base, const Op &A, int Y)
{
    const int lines = Y ? A.nx : A.ny, n = Y ? A.ny : A.nx;
    const size_t nlmax = (size_t)(lines + 1) / 2, nch = (size_t)(n + LINE_M - 1) / LINE_M;
    const size_t big = (size_t)n * nlmax, red = 2 * nch * nlmax;
    LineScratch s;
    s.a = base;
    s.c = s.a + big;
    s.d = s.c + big;
    s.rlo = s.d + big;
    s.rup = s.rlo + red;
    s.rrhs = s.rup + red;
    return s;
}

template <int Y>
static void colour_pass(const Op &A, const double *f, double *u, double *scr, int c, cudaStream_t s, int *nlaunch)
{
    const LineGeo g = make_geo(A, Y, c);
    if (g.nl <= 0)
        return;
    const LineScratch sc = carve(scr, A, Y);
    const dim3 b(128), gr = Y ? dim3((g.nl + 127) / 128, g.nch) : dim3((g.nch + 127) / 128, g.nl);
    k_line_elim<Y><<<gr, b, 0, s>>>(A, f, u, g, sc);
    int n = 1;
    if (g.nch > 1) {
        // up to 4 lines (warps) per CTA, 3 reduced rows of 2*nch doubles each per line
        const size_t per_line = 3 * (size_t)32 * ((2 * g.nch + 31) / 32) * sizeof(double);
        int lpb = (int)((size_t)LINE_SMEM / per_line);
        lpb = lpb > 4 ? 4 : (lpb < 1 ? 1 : lpb);
        const size_t smem = lpb * per_line;
        {  // the attribute is per device (a handle may live on any GPU of the process)
            static std::once_flag once[64][2];
            int dev = 0;
            cudaGetDevice(&dev);
            std::call_once(once[dev & 63][Y], []() {
                cudaFuncSetAttribute(k_line_reduced<Y>, cudaFuncAttributeMaxDynamicSharedMemorySize, LINE_SMEM);
            });
        }
        k_line_reduced<Y><<<dim3((g.nl + lpb - 1) / lpb), dim3(32 * lpb), smem, s>>>(A, u, g, sc);
        k_line_back<Y><<<gr, b, 0, s>>>(A, u, g, sc);
        n += 2;
    }
    if (nlaunch)
        *nlaunch += n;
}

// rev (c12, the adjoint sweep): the (direction, colour) passes in reverse order
void launch_relax_lines(const Op &A, const double *f, double *u, int nsweeps, int mode, double *scr, cudaStream_t s,
                        int *nlaunch, bool rev)
{
    const bool X = mode == RELAX_XLINES || mode == RELAX_ALTLINES, Yd = mode == RELAX_YLINES || mode == RELAX_ALTLINES;
    for (int sw = 0; sw < nsweeps; sw++) {
        for (int pp = 0; pp < 2; pp++) {
            const int pass = rev ? 1 - pp : pp;
            if (pass == 0 && X)
                for (int c = 0; c < 2; c++)
                    colour_pass<0>(A, f, u, scr, rev ? 1 - c : c, s, nlaunch);
            if (pass == 1 && Yd)
                for (int c = 0; c < 2; c++)
                    colour_pass<1>(A, f, u, scr, rev ? 1 - c : c, s, nlaunch);
        }
    }
}

void launch_line_pivots(const Op &A, int mode, int *err, cudaStream_t s)
{
    if (mode == RELAX_XLINES || mode == RELAX_ALTLINES)
        k_line_pivots<0><<<(A.ny + 127) / 128, 128, 0, s>>>(A, err);
    if (mode == RELAX_YLINES || mode == RELAX_ALTLINES)
        k_line_pivots<1><<<(A.nx + 127) / 128, 128, 0, s>>>(A, err);
}

}  // namespace bmg
