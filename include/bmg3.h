/*
 * include/bmg3.h -- C ABI of the 3-D BoxMG path of libbmg.so (SURVEY.md §8(f)
 * row 4: "3-D BoxMG (7/27-point) with plane relaxation").
 *
 * The problem is Eq. (1) on a structured 3-D grid with a
 * 7- or 27-point stencil; the solver is the V-cycle of fig:vcycle_flowchart
 * with its "Gauss Seidel" or "Plane" relaxation box (
 * "performance optimizations for operations such as plane relaxation",
 * P:104-107).  The paper gives no 3-D formula; the readings c16-c24 of
 * DESIGN.md §3 fix every step (each reduces to its 2-D reading of bmg.h when
 * the third dimension is trivial).
 *
 * Conventions: those of bmg.h (fp64, device pointers on the current device,
 * no aliasing, caller-owned inputs, status codes, bmg_last_error_detail(),
 * one host thread per handle).  A 3-D grid function g of an nx*ny*nz interior
 * has element (i,j,k) at g[k*plane_stride + j*pitch + i], i in [0,nx+1],
 * j in [0,ny+1], k in [0,nz+1]; the interior is [1,nx]x[1,ny]x[1,nz]; the ring
 * is the homogeneous Dirichlet ghost (an iterate's ring must be 0 and is
 * never written; a right-hand side's ring is ignored).
 */
#ifndef BMG3_H
#define BMG3_H

#include "bmg.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct bmg3_solver *bmg3_solver_t; /* opaque, library-owned */

/*
 * The fine operator as its symmetric half, matrix-entry signs (c16, c18):
 * plane[0] = O (diagonal); kind 7: plane[1] = W = A[p, p-(1,0,0)],
 * plane[2] = S = A[p, p-(0,1,0)], plane[3] = B = A[p, p-(0,0,1)];
 * kind 27: plane[1+e] = A[p, p+off_e] for the 13 offsets that precede the
 * centre, e = (dz+1)*9 + (dy+1)*3 + (dx+1) = 0..12 (dz = -1: all nine;
 * dz = 0: (-1,-1), (0,-1), (1,-1), (-1,0)).  The other half by symmetry:
 * A[p, p-off_e] = plane[1+e](p-off_e).  Couplings into the ring are dropped
 * (Dirichlet elimination).  Planes are read during bmg3_setup only (copied);
 * they and rhs/x share `pitch` and `plane_stride`.
 */
typedef struct {
    int kind;                /* 7 or 27 */
    int nx, ny, nz;          /* interior sizes, >= 1 */
    long long pitch;         /* elements per row, >= nx+2 */
    long long plane_stride;  /* elements per z-plane, >= pitch*(ny+2) */
    const double *plane[14];
} bmg3_stencil_t;

#define BMG3_RELAX_POINT 0  /* multicolour point GS: 2 colours on 7-point, 8 on 27-point levels (c22) */
#define BMG3_RELAX_PLANES 1 /* zebra xy-plane GS, one 2-D V(1,1) per plane (c23) */

typedef struct {
    int nu1, nu2;   /* pre-/post-smoothing sweeps, default 2, 1 */
    int coarsest;   /* stop coarsening when min(nx,ny,nz) <= coarsest; default 3 (c17) */
    int max_levels; /* 0 = unlimited */
    int relax;      /* BMG3_RELAX_POINT (default) or BMG3_RELAX_PLANES */
} bmg3_params_t;

void bmg3_params_default(bmg3_params_t *p);

/*
 * Setup (P:99-102 in 3-D): copy the stencil (c16), then per level l < L-1 the
 * operator-induced interpolation (c19) and the Galerkin operator
 * A_{l+1} = P^T A_l P (c20; coarse levels are 27-point); with plane
 * relaxation, every relaxed level's planes get a 2-D hierarchy (c23: the
 * in-plane part of the level's operator, c3/c4 on it, Cholesky on its
 * coarsest); the coarsest 3-D level is factored densely (c24; at most 4096
 * unknowns, as are the coarsest plane levels).  params may be NULL.
 * Errors: EINVAL (sizes, kind, pitch/stride, a_O <= 0, a denominator <= 0, a
 * coarsest system too large), ENOMEM, ENOTSPD (a Cholesky pivot <= 0), ECUDA.
 * Synchronises cuda_stream.
 */
bmg_status_t bmg3_setup(const bmg3_stencil_t *stencil, const bmg3_params_t *params, void *cuda_stream,
                        bmg3_solver_t *out);

/* ncycles V(nu1,nu2) cycles on the fine level (c9 in 3-D), x in/out; asynchronous; replayed as a
 * CUDA graph cached per (rhs, x). */
bmg_status_t bmg3_vcycle(bmg3_solver_t h, const double *rhs, double *x, int ncycles, void *cuda_stream);

/* Cycle until ||rhs - A x||_2 <= tol ||rhs||_2 or maxiter; hist_host: maxiter+1
 * doubles or NULL.  ||rhs|| = 0 sets x = 0, 0 iterations.  ENOTCONV at maxiter (x, hist valid). */
bmg_status_t bmg3_solve(bmg3_solver_t h, const double *rhs, double *x, double tol, int maxiter, int *iters_out,
                        double *hist_host, void *cuda_stream);

/* ||rhs - A x||_2 over the interior (synchronises). */
bmg_status_t bmg3_residual_norm(bmg3_solver_t h, const double *rhs, const double *x, double *norm_host,
                                void *cuda_stream);

/* nsweeps sweeps of the hierarchy's smoother (point or planes) on the fine level (tests). */
bmg_status_t bmg3_relax(bmg3_solver_t h, const double *rhs, double *x, int nsweeps, void *cuda_stream);

bmg_status_t bmg3_num_levels(bmg3_solver_t h, int *L);
bmg_status_t bmg3_level_shape(bmg3_solver_t h, int level, int *nx, int *ny, int *nz, int *kind);

/* Kernels one bmg3_vcycle cycle launches (the captured graph's kernel nodes). */
bmg_status_t bmg3_cycle_kernel_count(bmg3_solver_t h, int *count);

/*
 * Copy level `level` to HOST arrays (tests): stencil_host = 14 planes (O, then
 * the 13 lower entries in e order; zero where a 7-point level has none), each
 * (nz+2)(ny+2)(nx+2), compact pitch nx+2; ci_host (NULL allowed; ignored on
 * the coarsest level) = 26 weight planes over the coarse index range
 * (ncz+2)(ncy+2)(ncx+2) in the c19 slot order.  Synchronises.
 */
bmg_status_t bmg3_export_level(bmg3_solver_t h, int level, double *stencil_host, double *ci_host);

bmg_status_t bmg3_destroy(bmg3_solver_t h);

#ifdef __cplusplus
}
#endif
#endif
