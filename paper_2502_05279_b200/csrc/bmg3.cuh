// bmg3.cuh -- device-side views, per-point helpers and launchers of the 3-D
// BoxMG path (DESIGN.md §3 c16-c24, §5.8).  Product code,
// shares nothing with oracle/.
//
// HBM layout: every 3-D grid function of a level is one pitched
// (nz+2) x (ny+2) x px fp64 array, element (i,j,k) at k*ps + j*px + i, ring 0.
// The operator is its symmetric half in structure-of-arrays planes: O plus the
// 13 entries that precede the centre (e = (dz+1)*9 + (dy+1)*3 + (dx+1)), of
// which a 7-point level stores only W (e = 12), S (10) and B (4).  Every plane
// is 0 on the ring and on couplings into it, so a kernel never branches on the
// boundary.  Interpolation weights from level l+1 to l are 26 planes on the
// coarse index grid (c19 slot order).  The plane solver of c23 keeps, per
// relaxed level, a batch of 2-D hierarchies: one (nz+2)-deep array per 2-D
// level and field, plane k of the batch belonging to xy-plane k of the level.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace bmg3 {

struct Grid3 {
    int nx, ny, nz;
    long long px, ps;  // row pitch, plane stride (elements)
};

// a level's operator (read-only view); a[e] == nullptr where a 7-point level has no entry
struct Op3 {
    Grid3 g;
    int kind;  // 7 or 27
    const double *O;
    const double *a[13];
};

// weights from the next coarser level: 26 planes over the coarse index grid
struct CI3 {
    Grid3 c;
    const double *w[26];
};

// c19 slot base per fine-point type (mask of odd coordinates x|y<<1|z<<2)
__host__ __device__ constexpr int slot_base(int m)
{
    return m == 1 ? 0 : m == 2 ? 2 : m == 4 ? 4 : m == 3 ? 6 : m == 5 ? 10 : m == 6 ? 14 : m == 7 ? 18 : -1;
}

__host__ __device__ __forceinline__ long long eoff(const Grid3 &g, int e)
{
    return (long long)(e / 9 - 1) * g.ps + (long long)((e / 3) % 3 - 1) * g.px + (e % 3 - 1);
}

__host__ __device__ __forceinline__ long long at3(const Grid3 &g, int i, int j, int k)
{
    return (long long)k * g.ps + (long long)j * g.px + i;
}

// ---------------------------------------------------------------- batched 2-D plane levels (c23)
// One 2-D level of the plane hierarchies of a 3-D level: nz+2 planes of
// (ny+2) x px, plane k = the 2-D problem of xy-plane k.  Symmetric half of
// the 9-point operator: W = (-1,0), S = (0,-1), SW = (-1,-1), SE = (+1,-1)
// (NW(i,j) = SE(i-1,j+1), NE = SW(i+1,j+1), E = W(i+1), N = S(j+1)).
struct OpP {
    Grid3 g;
    int kind;  // 5 (no corner entries) or 9
    const double *O, *W, *S, *SW, *SE;
};

// 2-D interpolation weights (c3), 8 planes over the coarse index grid, order
// of the 2-D ABI: LNE, LA, LNW, LR, LL, LSE, LB, LSW
enum { P_LNE = 0, P_LA = 1, P_LNW = 2, P_LR = 3, P_LL = 4, P_LSE = 5, P_LB = 6, P_LSW = 7 };
struct CIP {
    Grid3 c;
    const double *w[8];
};

// the batch of planes one launch works on: k = k0 + 2*b, b in [0, nb)
struct Batch {
    int k0, nb;
};

// ---------------------------------------------------------------- launchers (kernels3.cu)
void launch3_ingest(int kind, const Grid3 &g, const double *const src[14], double *const dst[14], int *err,
                    cudaStream_t s);
void launch3_interp(const Op3 &A, double *const ci[26], const Grid3 &cg, int *err, cudaStream_t s);
void launch3_rap(const Op3 &A, const CI3 &ci, double *const dst[14], int *err, cudaStream_t s);
void launch3_assemble_dense(const Op3 &A, double *M, cudaStream_t s);
void launch3_coarse_solve(const Op3 &A, const double *Lf, const double *f, double *u, cudaStream_t s);
void launch3_relax_point(const Op3 &A, const double *f, double *u, int nsweeps, cudaStream_t s, int *nlaunch);
// 27-point levels: colour-major full-row copy (relax27_doubles(g) doubles) and its sweeps
long long relax27_doubles(const Grid3 &g);
void launch3_build_relax27(const Op3 &A, double *cf, cudaStream_t s);
void launch3_relax27c(const Grid3 &g, const double *cf, const double *f, double *u, int nsweeps, cudaStream_t s);
void launch3_residual(const Op3 &A, const double *f, const double *u, double *r, cudaStream_t s);
void launch3_restrict(const Op3 &A, const CI3 &ci, const double *r, double *fc, double *uc, cudaStream_t s);
// u = uin + P ec (uin may equal u)
void launch3_interp_add(const Grid3 &fine, const CI3 &ci, const double *ec, const double *uin, double *u,
                        cudaStream_t s);
// 7-point levels: one red-black sweep uout = GS(uin) in one pass (uin != uout)
void launch3_rb7(const Op3 &A, const double *f, const double *uin, double *uout, cudaStream_t s,
                 const double *ro = nullptr);
// ro = rcp_pos(a_O) on the interior (the one-pass sweep's reciprocal plane)
void launch3_recip(const Op3 &A, double *ro, cudaStream_t s);
// ||f - A u||_2 (or ||g||_2 when A == nullptr: pass f = g, u = nullptr) into *result (device)
void launch3_resid_norm(const Op3 *A, const Grid3 &g, const double *f, const double *u, double *partials,
                        double *result, cudaStream_t s);
int norm3_partials(const Grid3 &g);
void launch3_zero_interior(const Grid3 &g, double *x, cudaStream_t s);

// plane relaxation (kernels_plane.cu)
void launch3_plane_rhs(const Op3 &A, const double *f, const double *u, double *g, Batch b, cudaStream_t s);
void launchP_interp(const OpP &A, double *const ci[8], const Grid3 &cg, int *err, cudaStream_t s);
void launchP_rap(const OpP &A, const CIP &ci, double *const dst[5], cudaStream_t s);
void launchP_assemble_chol(const OpP &A, double *L, int *err, cudaStream_t s);
void launchP_relax(const OpP &A, const double *f, double *u, Batch b, cudaStream_t s);
// 5-point plane levels: one red-black sweep uout = GS(uin) in one pass (uin != uout)
void launchP_rb5(const OpP &A, const double *f, const double *uin, double *uout, Batch b, cudaStream_t s);
void launchP_residual(const OpP &A, const double *f, const double *u, double *r, Batch b, cudaStream_t s);
void launchP_restrict(const OpP &A, const CIP &ci, const double *r, double *fc, double *uc, Batch b,
                      cudaStream_t s);
void launchP_interp_add(const Grid3 &fine, const CIP &ci, const double *ec, double *u, Batch b, cudaStream_t s);
void launchP_coarse_solve(const OpP &A, const double *L, const double *f, double *u, Batch b, cudaStream_t s);

// the plane tail: the small plane levels of one V(1,1) in one launch (one CTA per plane)
constexpr int PTAIL_MAX = 1024;  // unknowns per plane of a tail level
constexpr int PTAIL_LEVELS = 8;
struct PTailLevel {
    OpP op;
    CIP ci;  // to the next tail level (unused on the last)
    double *u, *f, *r;
};
struct PTail {
    int nlev;
    PTailLevel lv[PTAIL_LEVELS];
    const double *chol;
};
void launchP_tail(const PTail &T, Batch b, cudaStream_t s);

}  // namespace bmg3
