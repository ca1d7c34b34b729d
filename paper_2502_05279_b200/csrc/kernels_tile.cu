// kernels_tile.cu -- the legs of the SMALL levels: one launch per
// leg, one CTA per 32x32 block of fine points, the level's data for the block
// plus a halo staged in shared memory, and every step of the leg done there,
// separated by __syncthreads only:
//   down leg: nu1 multicolour GS sweeps (c6), residual, restriction
//             (fig:restrict_kernel without the vanishing terms, c5a), zero start
//             of the next level (when it reads one);
//   up leg:   interpolation + correction (c7), nu2 sweeps.
// A CTA recomputes the halo its neighbours own (same per-point arithmetic as
// relax5_pt / relax9_pt / residual_pt / interp_pt, so the owners' values are
// reproduced exactly), so CTAs never synchronise with each other.  These levels
// (<= 511^2 at the bench size) sit in L2 and are bound by latency, not bytes:
// the streaming kernels of kernels_fused.cu need ~20 row steps of pipeline fill
// per chunk there (~20 us a leg); a tile leg is one load phase and ~10 shared-
// memory phases.
#include <mutex>

#include "bmg_internal.cuh"

namespace bmg {

constexpr int TL_TC = 16;        // coarse points per tile side (fine: 2*TL_TC owned)
constexpr int TL_THREADS = 1024;

template <int KIND>
struct TileOps {
    static constexpr int NPL = KIND == 9 ? 5 : 3;  // O W S [SW NW]
    static constexpr int NC = KIND == 9 ? 4 : 2;   // colours per sweep
};

// Shared-memory view of the window: arrays [u | f | planes...], each WW x WW.
template <int KIND, int WW>
struct Win {
    double *base;
    __device__ __forceinline__ double *arr(int q) const { return base + q * WW * WW; }
    __device__ __forceinline__ double &u(int b, int a) const { return base[b * WW + a]; }
    __device__ __forceinline__ double &f(int b, int a) const { return base[WW * WW + b * WW + a]; }
    __device__ __forceinline__ double pl(int k, int b, int a) const { return base[(2 + k) * WW * WW + b * WW + a]; }
};

// Load rows [wy0, wy0+WW) x cols [wx0, wx0+WW) of a level array (0 outside the padded grid)
// with asynchronous 8-byte copies (cp.async: every element in flight at once, no register
// round trip; out-of-grid elements zero-filled by a source size of 0).  Completed by
// tile_wait().  The loads of these L2-resident levels are latency-bound: issued one row at
// a time they cost ~0.7 us each.
__device__ __forceinline__ void cp_async8(double *dst, const double *src, bool valid)
{
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(src), "r"(valid ? 8 : 0) : "memory");
}
__device__ __forceinline__ void tile_wait()
{
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
}
// Rows to warps, columns to lanes: the row test and base address once per row (ncu: the
// divided linear index made the staging ~60 % of a tile leg's executed instructions; the
// leg's time did not move -- its staging waits on memory latency, not on issue).
template <int WW>
__device__ __forceinline__ void stage(double *dst, const double *src, long long pitch, int wx0, int wy0, int nx,
                                      int ny)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int b = warp; b < WW; b += nw) {
        const int gy = wy0 + b;
        const bool rok = src && gy >= 0 && gy <= ny + 1;
        const double *row = rok ? src + (long long)gy * pitch : nullptr;
        for (int a = lane; a < WW; a += 32) {
            const int gx = wx0 + a;
            const bool ok = rok && gx >= 0 && gx <= nx + 1;
            cp_async8(dst + b * WW + a, ok ? row + gx : (const double *)dst, ok);
        }
    }
}

// The points each thread relaxes, per colour: window index (b*WW + a) and 1/a_pp, formed
// once per launch.  The window origin's parity is fixed at compile time (PX0, PY0: parity
// of wx0, wy0), so colour c's points are the rows b = b0 + 2i and columns a = a0 + 2j of
// the updatable square [1, WW-2]^2: thread t takes points t, t + NT, ... of that grid.
// Colour of global (gx, gy): 5-point (gx+gy)&1, 9-point (gx&1) + 2(gy&1) (c6).
template <int KIND, int WW, int PX0, int PY0>
struct Points {
    static constexpr int NC = TileOps<KIND>::NC;
    static constexpr int NA = (WW - 1) / 2;  // column slots per row of one parity
    static constexpr int NSLOT = KIND == 9 ? NA * NA : NA * (WW - 2);
    static constexpr int PPT = (NSLOT + TL_THREADS - 1) / TL_THREADS;  // points per thread and colour
    int idx[NC][PPT];
    double rc[NC][PPT];

    __device__ __forceinline__ void build(const double *O, int wx0, int wy0, int nx, int ny)
    {
#pragma unroll
        for (int c = 0; c < NC; c++)
#pragma unroll
            for (int j = 0; j < PPT; j++) {
                const int k = threadIdx.x + j * TL_THREADS;
                int b, a;
                if (KIND == 9) {
                    // rows with gy parity (c>>1)&1, columns with gx parity c&1, starting at 1 or 2
                    const int b0 = ((((c >> 1) & 1) - PY0 - 1) & 1) + 1, a0 = (((c & 1) - PX0 - 1) & 1) + 1;
                    b = b0 + 2 * (k / NA);
                    a = a0 + 2 * (k % NA);
                } else {
                    // 5-point: per row about (WW-2)/2 points of parity (c - gy) & 1
                    b = 1 + k / NA;
                    const int px = (c - (PY0 + b)) & 1;
                    const int a0 = ((px - PX0 - 1) & 1) + 1;
                    a = a0 + 2 * (k % NA);
                }
                const int gx = wx0 + a, gy = wy0 + b;
                const bool ok = k < NSLOT && b <= WW - 2 && a <= WW - 2 && gx >= 1 && gx <= nx && gy >= 1 &&
                                gy <= ny;
                idx[c][j] = ok ? b * WW + a : -1;
                rc[c][j] = ok ? rcp_pos(O[b * WW + a]) : 0.0;
            }
    }
};

// (A u) off-diagonal part at window index q, fig:stencil_operator order SW,S,SE,W,E,NW,N,NE
// (the order of offdiag / relax5_pt in kernels_cycle.cu)
template <int KIND, int WW>
__device__ __forceinline__ double tile_offdiag_q(const Win<KIND, WW> &w, int q)
{
    const double *u = w.arr(0), *O = w.arr(2);
    const double *W = O + WW * WW, *S = O + 2 * WW * WW;
    if (KIND == 5) {
        double acc = S[q] * u[q - WW];
        acc += W[q] * u[q - 1];
        acc += W[q + 1] * u[q + 1];
        acc += S[q + WW] * u[q + WW];
        return acc;
    } else {
        const double *SW = O + 3 * WW * WW, *NW = O + 4 * WW * WW;
        double acc = SW[q] * u[q - WW - 1];
        acc += S[q] * u[q - WW];
        acc += NW[q - WW + 1] * u[q - WW + 1];
        acc += W[q] * u[q - 1];
        acc += W[q + 1] * u[q + 1];
        acc += NW[q] * u[q + WW - 1];
        acc += S[q + WW] * u[q + WW];
        acc += SW[q + WW + 1] * u[q + WW + 1];
        return acc;
    }
}

template <int KIND, int WW, int PX0, int PY0>
__device__ __forceinline__ void tile_sweeps(const Win<KIND, WW> &w, const Points<KIND, WW, PX0, PY0> &pt,
                                            int nsweeps, bool rev)
{
    constexpr int NC = TileOps<KIND>::NC, PPT = Points<KIND, WW, PX0, PY0>::PPT;
    double *u = w.arr(0);
    const double *f = w.arr(1);
    for (int sw = 0; sw < nsweeps; sw++)
#pragma unroll
        for (int cc = 0; cc < NC; cc++) {
            const int c = rev ? NC - 1 - cc : cc;
#pragma unroll
            for (int j = 0; j < PPT; j++) {
                const int q = pt.idx[c][j];
                if (q >= 0)
                    u[q] = (f[q] - tile_offdiag_q<KIND, WW>(w, q)) * pt.rc[c][j];
            }
            __syncthreads();
        }
}

// stage u (or zeros), f and the planes; rcp = 1/a_O (rcp_pos, as every relaxation path)
template <int KIND, int WW>
__device__ __forceinline__ void tile_load(const Win<KIND, WW> &w, const Op &A, const double *f, const double *uin,
                                          int wx0, int wy0)
{
    stage<WW>(w.arr(0), uin, A.pitch, wx0, wy0, A.nx, A.ny);  // uin == nullptr: zero start
    stage<WW>(w.arr(1), f, A.pitch, wx0, wy0, A.nx, A.ny);
    const double *pls[5] = {A.O, A.W, A.S, A.SW, A.NW};
#pragma unroll
    for (int k = 0; k < TileOps<KIND>::NPL; k++)
        stage<WW>(w.arr(2 + k), pls[k], A.pitch, wx0, wy0, A.nx, A.ny);
    tile_wait();
}

// ---------------------------------------------------------------- down leg
template <int KIND, int NU>
__global__ void __launch_bounds__(TL_THREADS) k_tile_down(TileArgs t)
{
    constexpr int P = NU * TileOps<KIND>::NC;          // colour passes
    constexpr int WW = 2 * TL_TC + 3 + 2 * P;          // r on [X0, X0+2TC], u valid one further
    extern __shared__ __align__(16) double tl_sm[];
    const Win<KIND, WW> w{tl_sm};
    const Op &A = t.A;
    const int I0 = 1 + blockIdx.x * TL_TC, J0 = 1 + blockIdx.y * TL_TC;
    const int X0 = 2 * I0 - 1, Y0 = 2 * J0 - 1;        // owned fine block [X0, X0+2TC)^2
    const int wx0 = X0 - 1 - P, wy0 = Y0 - 1 - P;
    tile_load<KIND, WW>(w, A, t.f, t.uzero ? nullptr : t.uin, wx0, wy0);
    // wx0 = 2 I0 - 2 - P: even (P is even)
    Points<KIND, WW, 0, 0> pt;
    pt.build(w.arr(2), wx0, wy0, A.nx, A.ny);
    tile_sweeps<KIND, WW, 0, 0>(w, pt, NU, false);
    // residual on [X0, X0+2TC]^2 into f (each point reads only its own f), skipping the colour
    // relaxed last (its residual vanishes, c5a): 5-point black, 9-point colour 3
    constexpr int RW = 2 * TL_TC + 1;
    for (int k = threadIdx.x; k < RW * RW; k += blockDim.x) {
        const int b = 1 + P + k / RW, a = 1 + P + k % RW, gx = wx0 + a, gy = wy0 + b;
        if (KIND == 5 ? ((gx + gy) & 1) : ((gx & 1) && (gy & 1)))
            continue;
        const bool in = gx >= 1 && gx <= A.nx && gy >= 1 && gy <= A.ny;
        const int q = b * WW + a;
        w.f(b, a) = in ? w.f(b, a) - (w.arr(2)[q] * w.arr(0)[q] + tile_offdiag_q<KIND, WW>(w, q)) : 0.0;
    }
    __syncthreads();
    // restriction of the tile's coarse points (restrict_pt_vanish's terms and order)
    const int ncx = A.nx / 2, ncy = A.ny / 2;
    const long long C = t.ci.pitch;
    for (int k = threadIdx.x; k < TL_TC * TL_TC; k += blockDim.x) {
        const int I = I0 + k % TL_TC, J = J0 + k / TL_TC;
        if (I > ncx || J > ncy)
            continue;
        const int a = 2 * I - wx0, b = 2 * J - wy0;  // window position of fine (2I, 2J)
        const long long c = J * C + I;
        double v;
        if (KIND == 5) {
            v = t.ci.w[CI_LNE][c] * w.f(b - 1, a - 1);
            v += t.ci.w[CI_LNW][c + 1] * w.f(b - 1, a + 1);
            v += w.f(b, a);
            v += t.ci.w[CI_LSE][c + C] * w.f(b + 1, a - 1);
            v += t.ci.w[CI_LSW][c + C + 1] * w.f(b + 1, a + 1);
        } else {
            v = t.ci.w[CI_LA][c] * w.f(b - 1, a);
            v += t.ci.w[CI_LR][c] * w.f(b, a - 1);
            v += w.f(b, a);
            v += t.ci.w[CI_LL][c + 1] * w.f(b, a + 1);
            v += t.ci.w[CI_LB][c + C] * w.f(b + 1, a);
        }
        t.fc[c] = v;
        if (t.uc)
            t.uc[c] = 0.0;
    }
    // the relaxed iterate on the owned block
    for (int k = threadIdx.x; k < 4 * TL_TC * TL_TC; k += blockDim.x) {
        const int b = 1 + P + k / (2 * TL_TC), a = 1 + P + k % (2 * TL_TC), gx = wx0 + a, gy = wy0 + b;
        if (gx <= A.nx && gy <= A.ny)
            t.uout[(long long)gy * A.pitch + gx] = w.u(b, a);
    }
}

// ---------------------------------------------------------------- up leg
template <int KIND, int NU, bool REV>
__global__ void __launch_bounds__(TL_THREADS) k_tile_up(TileArgs t)
{
    constexpr int P = NU * TileOps<KIND>::NC;
    constexpr int WW = 2 * TL_TC + 2 * P;
    constexpr int CW = WW / 2 + 3;  // coarse window of the fine window (e and the 8 weights)
    extern __shared__ __align__(16) double tl_sm[];
    const Win<KIND, WW> w{tl_sm};
    const Op &A = t.A;
    const int X0 = 1 + blockIdx.x * 2 * TL_TC, Y0 = 1 + blockIdx.y * 2 * TL_TC;
    const int wx0 = X0 - P, wy0 = Y0 - P;
    double *sc = tl_sm + (2 + TileOps<KIND>::NPL) * WW * WW;  // [e | 8 weights], CW x CW each
    const int cx0 = wx0 / 2 - 1, cy0 = wy0 / 2 - 1;             // (wx0 may be negative: floor not needed, -1 margin)
    {
        const int ncx = A.nx / 2, ncy = A.ny / 2;
        for (int q = 0; q < 9; q++) {
            const double *src = q == 0 ? t.ec : t.ci.w[q - 1];
            const long long cp = t.ci.pitch;
            const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
            for (int by = warp; by < CW; by += nw) {
                const int cy = cy0 + by;
                const bool rok = cy >= 0 && cy <= ncy + 1;
                for (int bx = lane; bx < CW; bx += 32) {
                    const int cx = cx0 + bx;
                    const bool ok = rok && cx >= 0 && cx <= ncx + 1;
                    cp_async8(sc + q * CW * CW + by * CW + bx, ok ? src + cy * cp + cx : (const double *)sc, ok);
                }
            }
        }
    }
    tile_load<KIND, WW>(w, A, t.f, t.uin, wx0, wy0);  // waits for every copy above too
    // views of the staged coarse arrays indexed by GLOBAL coarse (I, J), as interp_pt expects
    CIv cs;
    cs.pitch = CW;
    cs.roff = 0;
    cs.nrows = 0;
    const long long sh = (long long)cy0 * CW + cx0;
    for (int k = 0; k < 8; k++)
        cs.w[k] = sc + (1 + k) * CW * CW - sh;
    const double *es = sc - sh;
    // u += P e at the window's interior points (interp_pt: the per-step kernel's terms and order)
    for (int k = threadIdx.x; k < WW * WW; k += blockDim.x) {
        const int b = k / WW, a = k % WW, gx = wx0 + a, gy = wy0 + b;
        if (gx >= 1 && gx <= A.nx && gy >= 1 && gy <= A.ny)
            w.u(b, a) += interp_pt(cs, es, gx, gy);
    }
    // wx0 = X0 - P, X0 odd: odd
    Points<KIND, WW, 1, 1> pt;
    pt.build(w.arr(2), wx0, wy0, A.nx, A.ny);
    __syncthreads();
    tile_sweeps<KIND, WW, 1, 1>(w, pt, NU, REV);
    for (int k = threadIdx.x; k < 4 * TL_TC * TL_TC; k += blockDim.x) {
        const int b = P + k / (2 * TL_TC), a = P + k % (2 * TL_TC), gx = wx0 + a, gy = wy0 + b;
        if (gx <= A.nx && gy <= A.ny)
            t.uout[(long long)gy * A.pitch + gx] = w.u(b, a);
    }
}

template <int KIND, int NU>
constexpr size_t tile_smem(bool up)
{
    constexpr int P = NU * TileOps<KIND>::NC;
    const int WW = up ? 2 * TL_TC + 2 * P : 2 * TL_TC + 3 + 2 * P;
    const int CW = WW / 2 + 3;
    return ((size_t)(2 + TileOps<KIND>::NPL) * WW * WW + (up ? 9 * CW * CW : 0)) * sizeof(double);
}

// the dynamic shared-memory attribute, once per device; `once` is per kernel instance
template <typename K>
static void tile_attr(K kern, size_t smem, std::once_flag *once)
{
    int dev = 0;
    cudaGetDevice(&dev);
    std::call_once(once[dev & 63], [&]() { cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                                (int)smem); });
}

template <int KIND, int NU>
static void tile_down(const TileArgs &t, cudaStream_t s)
{
    static std::once_flag once[64];
    const size_t smem = tile_smem<KIND, NU>(false);
    tile_attr(k_tile_down<KIND, NU>, smem, once);
    dim3 g((t.A.nx + 2 * TL_TC - 1) / (2 * TL_TC), (t.A.ny + 2 * TL_TC - 1) / (2 * TL_TC));
    k_tile_down<KIND, NU><<<g, TL_THREADS, smem, s>>>(t);
}

template <int KIND, int NU, bool REV>
static void tile_up(const TileArgs &t, cudaStream_t s)
{
    static std::once_flag once[64];
    const size_t smem = tile_smem<KIND, NU>(true);
    tile_attr(k_tile_up<KIND, NU, REV>, smem, once);
    dim3 g((t.A.nx + 2 * TL_TC - 1) / (2 * TL_TC), (t.A.ny + 2 * TL_TC - 1) / (2 * TL_TC));
    k_tile_up<KIND, NU, REV><<<g, TL_THREADS, smem, s>>>(t);
}

bool tile_supported(int kind, int nu1, int nu2)
{
    return (kind == 5 || kind == 9) && (nu1 == 1 || nu1 == 2) && (nu2 == 1 || nu2 == 2);
}

void launch_tile_down(const TileArgs &t, int nu1, cudaStream_t s)
{
    if (t.A.kind == 9)
        nu1 == 1 ? tile_down<9, 1>(t, s) : tile_down<9, 2>(t, s);
    else
        nu1 == 1 ? tile_down<5, 1>(t, s) : tile_down<5, 2>(t, s);
}

void launch_tile_up(const TileArgs &t, int nu2, bool rev, cudaStream_t s)
{
    if (t.A.kind == 9) {
        if (rev)
            nu2 == 1 ? tile_up<9, 1, true>(t, s) : tile_up<9, 2, true>(t, s);
        else
            nu2 == 1 ? tile_up<9, 1, false>(t, s) : tile_up<9, 2, false>(t, s);
    } else {
        if (rev)
            nu2 == 1 ? tile_up<5, 1, true>(t, s) : tile_up<5, 2, true>(t, s);
        else
            nu2 == 1 ? tile_up<5, 1, false>(t, s) : tile_up<5, 2, false>(t, s);
    }
}

}  // namespace bmg
