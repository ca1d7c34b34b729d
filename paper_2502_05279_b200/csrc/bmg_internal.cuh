// bmg_internal.cuh -- device-side data views and launcher declarations of
// libbmg.so (product code; shares nothing with oracle/).
//
// Layout in HBM: every level stores its operator as the
// symmetric half in structure-of-arrays planes O, W, S (5-point) or
// O, W, S, SW, NW (9-point), each a pitched (ny+2) x pitch fp64 grid with the
// Dirichlet ring zero and couplings into the ring zeroed at ingest, so a
// kernel never branches on the boundary.  The interpolation weights from
// level l+1 to l are 8 planes (LNE, LA, LNW, LR, LL, LSE, LB, LSW) on the
// coarse index range with the coarse pitch.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace bmg {

// Storage order of the 8 weight planes: the Z-point (corner) weights first, then
// the X/Y (edge) weights, so that each half is one contiguous block (the fused
// down legs fetch only the half their restriction needs).
// bmg_export_level reorders to the API order LNE,LA,LNW,LR,LL,LSE,LB,LSW.
enum { CI_LNE = 0, CI_LNW = 1, CI_LSE = 2, CI_LSW = 3, CI_LR = 4, CI_LL = 5, CI_LA = 6, CI_LB = 7 };

// error bits raised by setup kernels (device int, OR-ed)
enum { ERR_DIAG = 1, ERR_DEN = 2, ERR_PIVOT = 4, ERR_LINE = 8, ERR_PEER = 16 };

// relaxation modes (bmg_params_t.relax): c6 point GS, c11 zebra line GS
enum { RELAX_POINT = 0, RELAX_XLINES = 1, RELAX_YLINES = 2, RELAX_ALTLINES = 3 };

// line relaxation: unknowns per chunk of a line (kernels_line.cu)
constexpr int LINE_M = 8;
// shared memory of the reduced-system kernel (one line's 3 x 2*ceil(n/LINE_M)
// doubles must fit): lines of at most LINE_NMAX unknowns
constexpr int LINE_SMEM = 227 * 1024;
constexpr int LINE_NMAX = 32768;

// One level's operator (read-only view).  SW/NW are nullptr on 5-point levels.
// Pointers are GLOBAL-row indexed: element (i, j) is at p[j*pitch + i] for the
// global row j.  A single-GPU level stores all rows (roff = 0, nrows = ny+2);
// a slab of a row-partitioned level (dist.cu) stores global rows
// [roff, roff+nrows) and owns interior rows [ylo, yhi) -- its pointers are the
// allocation shifted by -roff*pitch, so kernels index identically.
struct Op {
    int nx, ny, kind;  // GLOBAL interior sizes
    long long pitch;
    const double *O, *W, *S, *SW, *NW;
    int ylo, yhi;      // owned interior rows
    int roff, nrows;   // stored rows
};

// Interpolation weights between a level (fine) and the next (coarse); same
// row convention on the coarse grid.
struct CIv {
    long long pitch;  // coarse pitch
    const double *w[8];
    int roff, nrows;  // stored coarse rows
};

// Full 9-entry row of the operator at an interior point, reconstructed from
// the symmetric half (E=W(i+1,j), N=S(i,j+1), NE=SW(i+1,j+1), SE=NW(i+1,j-1)).
struct Row9 {
    double sw, s, se, w, o, e, nw, n, ne;
};

__device__ __forceinline__ Row9 load_row9(const Op &A, long long p)
{
    Row9 a;
    a.o = A.O[p];
    a.w = A.W[p];
    a.e = A.W[p + 1];
    a.s = A.S[p];
    a.n = A.S[p + A.pitch];
    if (A.kind == 9) {
        a.sw = A.SW[p];
        a.ne = A.SW[p + A.pitch + 1];
        a.nw = A.NW[p];
        a.se = A.NW[p - A.pitch + 1];
    } else {
        a.sw = a.ne = a.nw = a.se = 0.0;
    }
    return a;
}

// 1/b for b > 0 normal, entirely on the FP64 FMA pipe (no MUFU.RCP64H on the
// XU pipe, whose throughput bounded the streaming kernels).  Seed: exponent/
// mantissa reflection 0x7FE0...0 - bits(b), relative error <= 1/8; six Newton
// steps (2^-3 -> 2^-96, then a final one to settle rounding) give 1/b within
// 1 ulp.  Every GPU relaxation (per-step, tail and fused kernels) forms
// u = (f - sum) * rcp_pos(a_pp), so all paths agree bitwise; the oracle divides
// (difference <= ~2 ulp per update, inside the DESIGN §7 tolerances).
__device__ __forceinline__ double rcp_pos(double b)
{
    double r = __longlong_as_double(0x7FE0000000000000LL - __double_as_longlong(b));
#pragma unroll
    for (int i = 0; i < 5; i++)
        r = fma(r, fma(-b, r, 1.0), r);
    return fma(r, fma(-b, r, 1.0), r);
}

// (P e) at fine interior point (i, j) (DESIGN §3 c7); e's ring is 0.
__device__ __forceinline__ double interp_pt(const CIv &ci, const double *__restrict__ e, int i, int j)
{
    long long C = ci.pitch;
    int I = (i + 1) >> 1, J = (j + 1) >> 1;  // storage index of X/Y/Z weights; C point: (i/2, j/2)
    long long c = J * C + I;
    double s;
    if (!(i & 1) && !(j & 1)) {
        s = e[(j >> 1) * C + (i >> 1)];
    } else if ((i & 1) && !(j & 1)) {  // X at (2I-1, 2J): J = j/2
        c = (j >> 1) * C + I;
        s = ci.w[CI_LL][c] * e[c - 1];
        s += ci.w[CI_LR][c] * e[c];
    } else if (!(i & 1) && (j & 1)) {  // Y at (2I, 2J-1): I = i/2
        c = J * C + (i >> 1);
        s = ci.w[CI_LB][c] * e[c - C];
        s += ci.w[CI_LA][c] * e[c];
    } else {  // Z
        s = ci.w[CI_LSW][c] * e[c - C - 1];
        s += ci.w[CI_LSE][c] * e[c - C];
        s += ci.w[CI_LNW][c] * e[c - 1];
        s += ci.w[CI_LNE][c] * e[c];
    }
    return s;
}

// The legs of the small levels, by tiles in shared memory (kernels_tile.cu)
struct TileArgs {
    Op A;
    CIv ci;                       // weights to the next level
    const double *f, *uin, *ec;   // uin: start (down: nullptr with uzero), ec: coarse correction (up)
    double *uout, *fc, *uc;       // uc: the next level's zero start (nullptr: not read there)
    int uzero;
};
bool tile_supported(int kind, int nu1, int nu2);
void launch_tile_down(const TileArgs &t, int nu1, cudaStream_t s);
void launch_tile_up(const TileArgs &t, int nu2, bool rev, cudaStream_t s);

// CTA-wide sum in a fixed tree (warp shuffles, then one warp over the warp
// sums): the deterministic reduction of the norms and dot products.
__device__ __forceinline__ double block_sum(double v)
{
    __shared__ double sh[32];
    for (int o = 16; o > 0; o >>= 1)
        v += __shfl_down_sync(0xffffffffu, v, o);
    int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0)
        sh[wid] = v;
    __syncthreads();
    int nw = blockDim.x >> 5;
    v = (threadIdx.x < nw) ? sh[threadIdx.x] : 0.0;
    if (wid == 0)
        for (int o = 16; o > 0; o >>= 1)
            v += __shfl_down_sync(0xffffffffu, v, o);
    __syncthreads();
    return v;
}

// ---- launchers (kernels.cu) ----
void launch_ingest(int nx, int ny, int kind, long long pitch, const double *const src[5], double *const dst[5],
                   int *err, cudaStream_t s, int j0, int j1);
void launch_setup_interp(const Op &A, double *const ci[8], long long cpitch, int *err, cudaStream_t s, int J0,
                         int J1);
void launch_setup_rap(const Op &A, const CIv &ci, int ncx, int ncy, long long cpitch, double *const dst[5],
                      cudaStream_t s, int J0, int J1);
void launch_assemble_dense(const Op &A, double *M, cudaStream_t s);
void launch_chol_factor(int n, double *M, int *err, cudaStream_t s);
void launch_coarse_solve(const Op &A, const double *Lf, const double *f, double *u, cudaStream_t s);

// rev: colours in descending order (the adjoint smoother of the symmetric cycle, c12)
void launch_relax(const Op &A, const double *f, double *u, int nsweeps, cudaStream_t s, int *nlaunch,
                  bool rev = false);
void launch_residual(const Op &A, const double *f, const double *u, double *r, cudaStream_t s);
// vanish: r is the residual right after a point-GS sweep; the terms of the colour
// relaxed last (zero residual) are skipped, as in the fused down leg
void launch_restrict(const Op &A, const CIv &ci, const double *r, double *fc, double *uc, cudaStream_t s,
                     bool vanish = false);
// r != nullptr: BoxMG's affine term r/a_O at the non-coarse points (c14)
void launch_interp_add(const Op &A, const CIv &ci, const double *ec, double *u, cudaStream_t s,
                       const double *r = nullptr);
// c11 zebra line GS (kernels_line.cu): nsweeps sweeps in `mode`; scr holds
// line_scratch_doubles(nx, ny) doubles.  launch_line_pivots ORs ERR_LINE into
// *err if a line block has a pivot <= 0.
void launch_relax_lines(const Op &A, const double *f, double *u, int nsweeps, int mode, double *scr, cudaStream_t s,
                        int *nlaunch, bool rev = false);
void launch_line_pivots(const Op &A, int mode, int *err, cudaStream_t s);
size_t line_scratch_doubles(int nx, int ny);
void launch_resid_norm(const Op &A, const double *f, const double *u, double *r_out, double *partials,
                       double *result, cudaStream_t s);
void launch_norm(const Op &A, const double *g, double *partials, double *result, cudaStream_t s);
void launch_zero_interior(const Op &A, double *x, cudaStream_t s);
// c13 PCG vector kernels (owned interior rows of A)
void launch_dot(const Op &A, const double *a, const double *b, double *partials, double *result, cudaStream_t s);
// beta = sc[inum] / sc[iden], read on the device (no host round trip)
void launch_cg_direction(const Op &A, const double *sc, int inum, int iden, const double *z, double *p,
                         cudaStream_t s);
// fused: q = A p with <p, q> -> *result; the CG update with ||r|| -> *result
// (the same per-thread accumulation order as the separate dot / norm kernels)
void launch_matvec_dot(const Op &A, const double *p, double *q, double *partials, double *result, cudaStream_t s);
void launch_cg_update_norm(const Op &A, const double *sc, int inum, int iden, const double *p, const double *q,
                           double *x, double *r, double *partials, double *result, cudaStream_t s);

// c15 block multi-RHS kernels (kernels_block.cu): K = 1..BMG_MAX_NRHS columns
// stored interleaved, element (j, i, c) at (j*pitch + i)*K + c; per column the
// per-step kernels' arithmetic.  The norm launchers leave K results in result[0..K)
// and need K*NORM_BLOCKS partials.
void launch_relax_block(int K, const Op &A, const double *f, double *u, int nsweeps, cudaStream_t s, int *nlaunch,
                        bool rev = false);
void launch_residual_block(int K, const Op &A, const double *f, const double *u, double *r, cudaStream_t s);
void launch_restrict_block(int K, const Op &A, const CIv &ci, const double *r, double *fc, double *uc,
                           cudaStream_t s, bool vanish);
// residual + vanishing restriction fused (after nu1 >= 1 point-GS sweeps; r never stored)
void launch_resid_restrict_block(int K, const Op &A, const CIv &ci, const double *f, const double *u, double *fc,
                                 double *uc, cudaStream_t s);
// skip = 1 / 2: leave the points the post-smoother's first colour (forward / reversed
// order) overwrites uncorrected
void launch_interp_add_block(int K, const Op &A, const CIv &ci, const double *ec, double *u, cudaStream_t s,
                             const double *r, int skip, double *uout = nullptr);
// one GS sweep uout = GS(uin) of K columns (5-point: kb_rb5, one pass; 9-point: kb_r9pair, even then
// odd rows; uin != uout)
void launch_rb5_block(int K, const Op &A, const double *f, const double *uin, double *uout, cudaStream_t s);
void launch_coarse_solve_block(int K, const Op &A, const double *Lf, const double *f, double *u, cudaStream_t s);
void launch_resid_norm_block(int K, const Op &A, const double *f, const double *u, double *partials, double *result,
                             cudaStream_t s);
void launch_norm_block(int K, const Op &A, const double *g, double *partials, double *result, cudaStream_t s);
void launch_zero_block(int K, const Op &A, double *x, cudaStream_t s);
// block PCG (c13 x c15): per-column dot products (K results), q = A p, and the
// CG updates of the columns in `mask` with alpha/beta = sc[inum + c] / sc[iden + c]
void launch_dot_block(int K, const Op &A, const double *a, const double *b, double *partials, double *result,
                      cudaStream_t s);
void launch_matvec_block(int K, const Op &A, const double *p, double *q, cudaStream_t s);
void launch_cg_update_block(int K, const Op &A, const double *sc, int inum, int iden, unsigned mask, const double *p,
                            const double *q, double *x, double *r, cudaStream_t s);
void launch_cg_direction_block(int K, const Op &A, const double *sc, int inum, int iden, unsigned mask,
                               const double *z, double *p, cudaStream_t s);
void launch_zero_col_block(int K, const Op &A, double *x, int col, cudaStream_t s);

// Small levels l0..L-1 of the cycle in one single-CTA launch (k_tail).  Lives in
// device memory (filled once at setup); level 0's f/u are launch arguments.
// row pitch of a level's shared-memory copy in k_tail_sm (compact)
__host__ __device__ inline int tail_wp(int nx) { return nx + 2; }

struct TailLevel {
    Op A;
    CIv ci;                // weights to level l+1 (unused on L-1)
    double *f, *u, *r;     // level arrays (l > 0); r: residual scratch
    // shared-memory copy (k_tail_sm): compact pitch nx+2; offsets in doubles of u, f, r,
    // the plane block, the 8 weight planes (on level l+1's compact grid) and 1/a_pp
    int so_u, so_f, so_r, so_pl, so_ci, so_di;
};
struct TailPlan {
    int l0, L, nu1, nu2;
    int cycle_sym;         // 1: post-smoother colours reversed (c12)
    int affine;            // 1: affine interpolation-correction with the level's r (c14)
    const double *chol;    // coarsest Cholesky factor
    int sm_doubles;        // k_tail_sm: shared memory (0: the levels do not fit, k_tail runs)
    int so_chol, so_b;     // k_tail_sm: the Cholesky factor and the solve's scratch
    int so_part;           // k_tail_solve: the norms' NORM_BLOCKS partials
    TailLevel lv[32];
};
// fills the so_* fields and sm_doubles (host); returns false if they exceed `limit` doubles
bool tail_plan_smem(TailPlan &tp, int ncoarse, long long limit);
void launch_tail(const TailPlan *tp_dev, int ncoarse, const double *f0, double *u0, cudaStream_t s,
                 int sm_doubles = 0);

// Device-side solve loop (bmg_solve): state read and advanced by k_solve_step,
// the last node of the body of a conditional WHILE graph node.
struct SolveState {
    double fn, tol;   // ||rhs||, relative tolerance
    int k, maxiter;   // cycles done, cap
};
// k = ++st->k; hist[k] = *norm; continue while *norm > tol*fn and k < maxiter
void launch_solve_step(cudaGraphConditionalHandle hd, const double *norm, SolveState *st, double *hist,
                       cudaStream_t s);

// bmg_solve in ONE launch when the whole hierarchy is the shared-memory tail (tail from
// level 0): reads st->tol, st->maxiter; writes st->fn, st->k and hist[0..k]
void launch_tail_solve(const TailPlan *tp_dev, const double *f0, double *u0, SolveState *st, double *hist,
                       cudaStream_t s, int sm_doubles);

// the block solve's state (K columns): continue while any ||r_c|| > tol ||rhs_c||
struct SolveStateBlock {
    double fn[8], tol;
    int k, maxiter, K;
};
void launch_solve_step_block(cudaGraphConditionalHandle hd, const double *norms, SolveStateBlock *st, double *hist,
                             cudaStream_t s);

constexpr int NORM_BLOCKS = 592;  // 4 x 148 SMs; fixed so the reduction tree is fixed

}  // namespace bmg
