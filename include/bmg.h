/*
 * include/bmg.h -- C ABI of the B200-native BoxMG V-cycle library (libbmg.so).
 *
 * The problem (Eq. (1)): -div(D grad u) = f discretised by
 * a "standard finite-difference scheme which leads to a stencil-based
 * description of the resulting linear system, Ax = b", where the stencil
 * "may be different at each point" (fig:stencil_operator).  The
 * solver is the BoxMG V-cycle of fig:vcycle_flowchart: Gauss-Seidel
 * relaxation, residual, operator-induced restriction (fig:restrict_kernel,
 * P:165-189) and interpolation, Cholesky coarse solve, driven
 * by a setup that builds operator-induced interpolation and Galerkin coarse
 * operators "through local stencil operations".  The readings of
 * everything the paper leaves to Dendy/Reisner are listed in DESIGN.md §3.
 *
 * Conventions (all entry points):
 *  - Every array is IEEE fp64, row-major, x fastest.  A grid function g of an
 *    nx*ny interior has element (i,j) at g[j*pitch + i], i in [0,nx+1],
 *    j in [0,ny+1]; the interior is [1,nx]x[1,ny]; the ring is the
 *    homogeneous Dirichlet ghost: the ring of an iterate x must hold 0 and
 *    is never written; the ring of a right-hand side is ignored.
 *  - Unless stated otherwise, pointers are DEVICE pointers on the current
 *    CUDA device, must not alias each other, and stay owned by the caller.
 *  - `cuda_stream` is a cudaStream_t (NULL = legacy default stream).  All
 *    work is enqueued on it; calls that return host values synchronise it.
 *  - Errors are returned as bmg_status_t; nothing is thrown across the ABI.
 *    bmg_last_error_detail() gives thread-local text for the last failure.
 *  - A solver handle is used by one host thread at a time.
 */
#ifndef BMG_H
#define BMG_H

#ifdef __cplusplus
extern "C" {
#endif

typedef struct bmg_solver *bmg_solver_t; /* opaque, library-owned */

typedef enum {
    BMG_OK = 0,
    BMG_EINVAL = 1,   /* bad sizes/pointers/kind, a_O <= 0, interpolation denominator <= 0 */
    BMG_ENOMEM = 2,   /* device allocation failed */
    BMG_ECUDA = 3,    /* CUDA runtime error (detail in bmg_last_error_detail) */
    BMG_ENCCL = 4,    /* a NCCL call of the multi-GPU path failed (bmg_setup_dist, dist cycles) */
    BMG_ENOTSPD = 5,  /* coarsest-level Cholesky pivot <= 0, or a line-block pivot <= 0 */
    BMG_ENOTCONV = 6  /* bmg_solve reached maxiter; x and hist stay valid */
} bmg_status_t;

/*
 * The fine-level operator, stored as its symmetric half with matrix-entry
 * signs (D == 1 gives O=4, W=S=-1):
 *   plane[0] = O  (diagonal),        plane[1] = W = A[p, p-(1,0)],
 *   plane[2] = S  = A[p, p-(0,1)],   plane[3] = SW = A[p, p-(1,1)]  (kind 9),
 *   plane[4] = NW = A[p, p+(-1,1)]   (kind 9).
 * The other half follows by symmetry: E(i,j)=W(i+1,j), N(i,j)=S(i,j+1),
 * NE(i,j)=SW(i+1,j+1), SE(i,j)=NW(i+1,j-1).  Each plane is a grid function
 * with `pitch` elements per row; entries on the ghost ring and couplings that
 * point into the ring are dropped (Dirichlet elimination).
 * Plane pointers are DEVICE pointers, read only during bmg_setup (copied).
 */
typedef struct {
    int kind;              /* 5 -> planes {O,W,S}; 9 -> planes {O,W,S,SW,NW} */
    int nx, ny;            /* interior sizes, >= 1 */
    long long pitch;       /* elements per row, >= nx+2; also the pitch of rhs/x */
    const double *plane[5];
} bmg_stencil_t;

typedef struct {
    int nu1, nu2;    /* pre-/post-smoothing sweeps, default 2, 1 (V(2,1)) */
    int coarsest;    /* stop coarsening when min(nx,ny) <= coarsest; default 3 */
    int max_levels;  /* 0 = unlimited */
    int agglom_rows; /* multi-GPU: agglomerate below this many rows per rank (default 128) */
    int cycle_sym;   /* 0 = same colour order on both legs (default); 1 = the post-smoother is
                        the adjoint of the pre-smoother: colours (and, for alternating
                        lines, directions) in reverse order (DESIGN §3 c12), so that
                        V(nu,nu) is a symmetric operator (bmg_pcg's preconditioner).
                        cycle_sym = 1 runs the per-step kernels on the large levels. */
    int fused;       /* 1 = fused streaming kernels on large levels (default), 0 = one kernel per step */
    int relax;       /* relaxation (fig:vcycle_flowchart's "Relaxation" boxes):
                        BMG_RELAX_POINT (default) multicolour point Gauss-Seidel (DESIGN §3 c6);
                        BMG_RELAX_XLINES / _YLINES zebra line Gauss-Seidel along x / y, one
                        sweep = the lines of colour (line index mod 2) 0 then 1, each line's
                        tridiagonal block solved exactly (the "Line" box; c11);
                        BMG_RELAX_ALTLINES one sweep = an x-line then a y-line sweep.
                        Line modes run the per-step kernels (fused ignored) and need
                        nx, ny <= 32768 (EINVAL otherwise). */
    int affine;      /* 0 (default): u += P e (DESIGN §3 c7); 1: BoxMG's affine
                        interpolation-correction u(F) += (P e)(F) + r(F)/a_O(F) at the
                        non-coarse points, r the residual restricted on the down leg
                        (c14).  Runs the per-step kernels on the
                        large levels (the fused down legs do not store r). */
} bmg_params_t;

#define BMG_RELAX_POINT 0
#define BMG_RELAX_XLINES 1
#define BMG_RELAX_YLINES 2
#define BMG_RELAX_ALTLINES 3

/* Fill *p with the defaults above. */
void bmg_params_default(bmg_params_t *p);

/*
 * Setup (fig:vcycle_flowchart's setup phase): copy the stencil
 * (S0), then on every level l < L-1 build the operator-induced interpolation
 * weights (S1, DESIGN §3 c3) and the Galerkin operator A_{l+1} = P^T A_l P
 * (S2, c4); factor the coarsest level densely by Cholesky (S3, c8).
 * Levels: n_{l+1} = floor(n_l/2) until min(nx,ny) <= coarsest (c1).
 * params may be NULL (defaults).  On success *out owns all device memory.
 * Line relaxation modes also check that every line block (the tridiagonal
 * part of A along each relaxed line, on every level but the coarsest) has
 * positive elimination pivots, as the blocks of an SPD operator do.
 * Errors: EINVAL (sizes, kind, pitch, a_O <= 0, den <= 0, relax not a mode),
 * ENOMEM, ENOTSPD (coarsest Cholesky pivot or line pivot <= 0), ECUDA.
 * Synchronises cuda_stream.
 */
bmg_status_t bmg_setup(const bmg_stencil_t *stencil, const bmg_params_t *params, void *cuda_stream,
                       bmg_solver_t *out);

/*
 * ncycles V(nu1,nu2) cycles (fig:vcycle_flowchart) on the fine
 * level: x <- V(x) with right-hand side rhs.  rhs, x: device grid functions
 * with the setup pitch; x is read (initial guess) and overwritten.  Ring of x
 * is not written.  Asynchronous (no host sync).  The cycle is replayed as a
 * CUDA graph cached per (rhs, x) pointer pair.
 */
bmg_status_t bmg_vcycle(bmg_solver_t h, const double *rhs, double *x, int ncycles, void *cuda_stream);

/*
 * Same as bmg_vcycle, but rhs_host / x_host are HOST arrays (pinned or
 * pageable) with the setup pitch: copies rhs and x host->device, runs the
 * cycles, copies x device->host.  Synchronises cuda_stream.
 */
bmg_status_t bmg_vcycle_host(bmg_solver_t h, const double *rhs_host, double *x_host, int ncycles,
                             void *cuda_stream);

/*
 * bmg_vcycle_host for a batch of nprob INDEPENDENT problems on the same
 * operator (fig:vcycle_flowchart P:108-162 applied to each): for each i,
 * x_host[i] <- V^ncycles(x_host[i]) with right-hand side rhs_host[i].
 * rhs_host, x_host: arrays of nprob HOST pointers (pinned for the copies to
 * overlap; pageable works, serialised), each a grid function with the setup
 * pitch; x_host[i] is read and overwritten, rhs_host[i] only read.  The
 * arrays must not alias each other.  Pipelined over two device staging slots:
 * problem i's host->device copies and problem i-1's device->host copy run on
 * the handle's own copy streams while cuda_stream runs the cycles in between,
 * so a batch is bound by the PCIe rate rather than copy + cycle + copy in
 * series.  Results are bitwise those of bmg_vcycle_host per problem.  Returns
 * after every copy completed (synchronises cuda_stream).  BMG_EINVAL: NULL
 * arrays, nprob < 0, ncycles < 0, or a distributed handle.
 */
bmg_status_t bmg_vcycle_host_batch(bmg_solver_t h, int nprob, const double *const *rhs_host,
                                   double *const *x_host, int ncycles, void *cuda_stream);

/*
 * Solve loop: hist[0] = ||rhs - A x0||_2; repeat V-cycles
 * until ||r_k||_2 <= tol*||rhs||_2 or maxiter cycles.  ||rhs|| = 0 sets
 * x = 0 (interior) and returns 0 iterations.  iters_out (host, may be NULL)
 * receives the cycle count; hist_host (host, maxiter+1 doubles, may be NULL)
 * the absolute residual norms.  Returns ENOTCONV if maxiter was reached.
 * Single-GPU handles run the loop on the device (one graph launch: a
 * conditional WHILE node around cycle + norm + stopping test) and synchronise
 * cuda_stream once; distributed handles loop on the host.
 */
bmg_status_t bmg_solve(bmg_solver_t h, const double *rhs, double *x, double tol, int maxiter, int *iters_out,
                       double *hist_host, void *cuda_stream);

/*
 * Conjugate gradients preconditioned by one V(nu,nu) cycle from a zero guess
 * ("V-cycle-preconditioned CG"; Cedar's Krylov use of
 * BoxMG; DESIGN §3 c13): textbook PCG, r updated recursively,
 * hist_host[0] = ||rhs - A x0||_2, hist_host[k] = ||r_k||_2; stops when
 * ||r_k|| <= tol*||rhs|| (||rhs|| = 0: x = 0, 0 iterations).  Needs a
 * symmetric preconditioner: params nu1 == nu2 and cycle_sym = 1 (EINVAL
 * otherwise; single-GPU handles only).  Workspace: four level-0 arrays,
 * allocated on the first call and owned by the handle.  Returns ENOTCONV at
 * maxiter (x, hist valid).  The host waits once per iteration (for ||r_k||);
 * alpha and beta are formed on the device.  On return x and hist are final;
 * the next iteration's preconditioner, enqueued speculatively before the last
 * wait (never after the maxiter-th iteration), may still be running on
 * cuda_stream: it writes the PCG workspace AND the handle's hierarchy arrays,
 * so every later call on this handle (any stream) first waits for it.
 */
bmg_status_t bmg_pcg(bmg_solver_t h, const double *rhs, double *x, double tol, int maxiter, int *iters_out,
                     double *hist_host, void *cuda_stream);

/*
 * Block multi-RHS V-cycles (§5 "solve
 * several initial vectors in block fashion"; DESIGN §3 c15): nrhs systems
 * A x_c = rhs_c on the same hierarchy, every kernel of the cycle applying one
 * read of the operator / interpolation weights to all nrhs columns.
 *   rhs, x: DEVICE arrays of (ny+2) * pitch * nrhs doubles, INTERLEAVED:
 *           column c of point (i, j) at ((size_t)j * pitch + i) * nrhs + c
 *           (16-byte aligned when nrhs is even); ring as in bmg_vcycle.
 *   nrhs:   1 .. BMG_MAX_NRHS.
 * Column c after ncycles block cycles is bmg_vcycle(rhs_c, x_c, ncycles): the
 * same per-point operations in the same order (up to the FMA contraction the
 * compiler picks in the single-RHS kernels: a few ulp).  Point relaxation only
 * (params.relax != POINT: EINVAL); cycle_sym and affine apply.  Single-GPU
 * handles only.  Workspace (per level r, and f, u below level 0, nrhs columns
 * each) is allocated on the first call for a given nrhs and owned by the
 * handle; a call with another nrhs reallocates it.  Asynchronous on cuda_stream.
 */
#define BMG_MAX_NRHS 8
bmg_status_t bmg_vcycle_block(bmg_solver_t h, int nrhs, const double *rhs, double *x, int ncycles,
                              void *cuda_stream);

/* ||rhs_c - A x_c||_2 for every column into norms_host[0..nrhs) (host);
 * synchronises cuda_stream.  Layout and limits as bmg_vcycle_block. */
bmg_status_t bmg_residual_norm_block(bmg_solver_t h, int nrhs, const double *rhs, const double *x,
                                     double *norms_host, void *cuda_stream);

/*
 * Block solve (c15): hist row 0 = the nrhs initial residual norms; each block
 * step is one block V-cycle followed by the nrhs residual norms (row k).  Stops
 * when EVERY column has ||r_c|| <= tol*||rhs_c|| (a column that met its test
 * earlier keeps being cycled) or after maxiter steps.  A column with
 * ||rhs_c|| = 0 is set to x_c = 0 and counts as converged.
 * hist_host: (maxiter+1) * nrhs doubles (row-major, may be NULL); iters_out:
 * block steps taken (may be NULL).  Returns ENOTCONV if maxiter was reached.
 * The loop runs on the device (one graph launch, as bmg_solve).
 */
bmg_status_t bmg_solve_block(bmg_solver_t h, int nrhs, const double *rhs, double *x, double tol, int maxiter,
                             int *iters_out, double *hist_host, void *cuda_stream);

/*
 * Block PCG (c13 on each column of a c15 block): column c runs the recurrences
 * of bmg_pcg on (rhs_c, x_c) -- its own alpha_c and beta_c, the preconditioner
 * one block V(nu,nu) cycle from zero (needs nu1 == nu2 and cycle_sym = 1,
 * EINVAL otherwise) -- and is frozen once ||r_c|| <= tol*||rhs_c|| (so x_c is
 * what bmg_pcg would return for it, up to rounding).  A column with
 * ||rhs_c|| = 0 is set to 0.  hist_host: (maxiter+1) * nrhs doubles, row k =
 * the K recursive residual norms after k steps (a frozen column repeats its
 * last); iters_out: steps taken (the slowest column's count).  Layout, limits
 * and workspace as bmg_vcycle_block (plus four block arrays for r, z, p, q).
 * Synchronises cuda_stream once per step.  Returns ENOTCONV at maxiter.
 */
bmg_status_t bmg_pcg_block(bmg_solver_t h, int nrhs, const double *rhs, double *x, double tol, int maxiter,
                           int *iters_out, double *hist_host, void *cuda_stream);

/* ||rhs - A x||_2 over the fine interior ("l2 norm"), deterministic
 * fixed-tree reduction; optional r_out (device, setup pitch, ring untouched)
 * receives the residual.  *norm_host is a host double.  Synchronises. */
bmg_status_t bmg_residual_norm(bmg_solver_t h, const double *rhs, const double *x, double *r_out,
                               double *norm_host, void *cuda_stream);

/* Hierarchy queries (host outputs). */
bmg_status_t bmg_num_levels(bmg_solver_t h, int *L);
bmg_status_t bmg_level_shape(bmg_solver_t h, int level, int *nx, int *ny, int *kind);
/* Elements per row of level `level`'s grid functions (level 0: the setup pitch). */
bmg_status_t bmg_level_pitch(bmg_solver_t h, int level, long long *pitch);

/*
 * Copy level `level`'s operator and interpolation weights to HOST memory, for
 * tests.  stencil_host: 5 planes (O,W,S,SW,NW), each (ny+2)*(nx+2) with pitch
 * nx+2 (SW,NW are 0 on a 5-point level).  ci_host (may be NULL; ignored on
 * the coarsest level): 8 planes LNE,LA,LNW,LR,LL,LSE,LB,LSW (fig:restrict_kernel
 * names), each (ncy+2)*(ncx+2) with pitch ncx+2, ncx = nx/2, ncy = ny/2.
 * Synchronises the legacy stream.
 */
bmg_status_t bmg_export_level(bmg_solver_t h, int level, double *stencil_host, double *ci_host);

/*
 * Single method steps on one level, for per-kernel parity tests.  All arrays
 * are device grid functions of that level with bmg_level_pitch(level); for
 * restriction/interpolation the coarse array uses bmg_level_pitch(level+1).
 *  bmg_relax:      nsweeps sweeps of the handle's relaxation (params.relax:
 *                  multicolour point GS, c6, or zebra line GS, c11), u in/out.
 *  bmg_residual:   r = f - A u on the interior; r's ring set to 0.
 *  bmg_restrict:   fc = P^T r, the fig:restrict_kernel listing (c5); ring 0.
 *  bmg_interp_add: u += P ec (c7); ec's ring must be 0.
 * Asynchronous.
 */
bmg_status_t bmg_relax(bmg_solver_t h, int level, const double *f, double *u, int nsweeps, void *cuda_stream);
bmg_status_t bmg_residual(bmg_solver_t h, int level, const double *f, const double *u, double *r,
                          void *cuda_stream);
bmg_status_t bmg_restrict(bmg_solver_t h, int level, const double *r, double *fc, void *cuda_stream);
bmg_status_t bmg_interp_add(bmg_solver_t h, int level, const double *ec, double *u, void *cuda_stream);

/*
 * The two legs of one level of the V-cycle, as the cycle runs them (the fused
 * streaming kernel where the level is fused, else the per-step kernels):
 *  bmg_smooth_restrict: u_out = nu1 GS sweeps applied to u_in (rhs f); then
 *                       fc = P^T (f - A u_out) and, if uc != NULL, uc = 0 (the
 *                       coarse correction's zero start).
 *  bmg_correct_smooth:  u_out = nu2 GS sweeps applied to u_in + P ec.
 * u_in and u_out are distinct level-`level` grid functions (bmg_level_pitch);
 * the ring of u_out is not written.  fc, uc, ec use bmg_level_pitch(level+1).
 * Asynchronous.  EINVAL if u_in == u_out or a pointer is NULL.
 */
bmg_status_t bmg_smooth_restrict(bmg_solver_t h, int level, const double *f, const double *u_in, double *u_out,
                                 double *fc, double *uc, void *cuda_stream);
bmg_status_t bmg_correct_smooth(bmg_solver_t h, int level, const double *f, const double *u_in, const double *ec,
                                double *u_out, void *cuda_stream);

/* Number of kernels one bmg_vcycle cycle launches (the captured graph's kernel nodes). */
bmg_status_t bmg_cycle_kernel_count(bmg_solver_t h, int *count);

/* Measurement hook (bench.py's roofline figure).  enable != 0: subsequent
 * bmg_vcycle calls on this single-GPU handle replay a variant of the cycle's
 * graph with two event-record nodes around the level-0 down-leg launch (or, when
 * the single-CTA tail kernel starts at level 0, around that launch), each
 * launch re-pointed at a fresh CUDA event pair (timed on the caller's stream);
 * enable == 0 returns to the plain graph.  Either call clears the records.
 * bmg_timing_read waits for the recorded events and returns the summed
 * duration (ms) and number of those launches since the last clear.
 * EINVAL on a distributed handle. */
bmg_status_t bmg_timing(bmg_solver_t h, int enable);
bmg_status_t bmg_timing_read(bmg_solver_t h, double *ms_total, int *launches);

/* Device time (ms) of the setup kernels of a single-GPU handle: S0 ingest through the
 * S3 Cholesky factor (events around them; excludes allocation, which bmg_setup's wall
 * clock includes).  Blocks until they have run.  EINVAL on a distributed handle. */
bmg_status_t bmg_setup_time(bmg_solver_t h, double *device_ms);

/* Per-leg breakdown of one cycle (SURVEY §5 per-level report, mirroring the
 * paper's per-level kernel timings, fig:kernel_timings P:492-500).  Captures a
 * variant of the cycle's graph with an event-record node between every two
 * legs, replays it ncycles times on cuda_stream (synchronising after each) and
 * returns the mean duration (ms) of every segment in ms_out[0 .. *nseg-1]:
 *   ms_out[l]            l = 0..lt-1   down leg of level l (fused kernel or per-step kernels)
 *   ms_out[lt]                         the tail: levels >= lt, the coarse solve and their up legs
 *   ms_out[lt+1+k]       k = 0..lt-1   up leg of level lt-1-k
 * with lt = (*nseg - 1) / 2.  x is advanced by ncycles cycles (as bmg_vcycle).
 * Blocking.  EINVAL if cap < 2L+1, ncycles < 1 or the handle is distributed. */
bmg_status_t bmg_profile_legs(bmg_solver_t h, const double *rhs, double *x, int ncycles, double *ms_out, int cap,
                              int *nseg, void *cuda_stream);

/* ---------------------------------------------------------------------------
 * Multi-GPU: row-slab domain decomposition.
 *
 * Rows 1..ny are split into nranks contiguous slabs [y_p, y_{p+1}) whose
 * starts are multiples of 2^K, K = number of distributed levels (largest K
 * keeping at least max(agglom_rows, 2*BMG_HALO) rows per rank on level K-1).
 * Level K and below are replicated on every rank (agglomeration by
 * all-gather).  A rank's LOCAL arrays hold global rows
 * [row0, row0+nrows) = [max(y_p - BMG_HALO, 0), min(y_{p+1} + BMG_HALO, ny+2)),
 * pitch as in bmg_stencil_t: the owned rows plus BMG_HALO ghost rows, which
 * the library overwrites (also in rhs) with the neighbours' values.
 * ------------------------------------------------------------------------- */
#define BMG_HALO 6

typedef struct {
    int nranks;           /* number of slabs (>= 1) */
    int rank;             /* this process's slab (NCCL mode) */
    void *nccl_comm;      /* ncclComm_t over the nranks processes (NCCL mode) */
    const char *nccl_lib; /* path of the libnccl.so.2 to dlopen (NULL: "libnccl.so.2") */
    int loopback;         /* 1: all nranks slabs simulated in THIS process on the current
                             GPU, ghost rows copied device-to-device (tests); stencil,
                             rhs and x are then GLOBAL arrays */
    int peer;             /* 1: the ghost rows of the distributed legs move by in-kernel peer
                             stores (SURVEY §8(e) lever 3): each fused leg's store and
                             restriction tasks also write the rows within BMG_HALO of the
                             slab edges into the neighbours' arrays (CUDA-IPC mapped peer
                             memory over NVLink; other ranks' slabs in loopback), and a
                             one-thread signal / wait pair per leg orders the neighbours
                             (system-scope flags in peer memory) -- instead of a grouped
                             NCCL send/recv between legs.  The level-0 u/f ghost rows at the
                             start of a cycle, the level-K all-gather and the norm stay NCCL.
                             NCCL mode needs the ranks on one node (CUDA IPC). */
} bmg_comm_t;

/* Host-only: slab boundaries ybounds[0..nranks] (y_0 = 1, y_nranks = ny+1) and the
 * number of distributed levels *kdist for an nx*ny grid.  EINVAL if the grid is too
 * small for nranks slabs.  params may be NULL. */
bmg_status_t bmg_partition(int nx, int ny, int nranks, const bmg_params_t *params, int *ybounds, int *kdist);

/*
 * Distributed setup.  stencil->nx, ny are the GLOBAL sizes; in NCCL mode its planes
 * are this rank's local arrays (rows [row0, row0+nrows) of bmg_local_rows; only the
 * owned rows are read), in loopback mode the global arrays.  Collective over the
 * communicator.  The returned handle works with bmg_vcycle, bmg_solve,
 * bmg_residual_norm, bmg_num_levels, bmg_local_rows and bmg_destroy; rhs and x are
 * local arrays (NCCL) or global arrays (loopback).  Errors: EINVAL (grid too small,
 * params unsupported: needs fused = 1, relax = BMG_RELAX_POINT, nu1, nu2 in {1,2}),
 * ENCCL, ENOMEM, ECUDA.
 */
bmg_status_t bmg_setup_dist(const bmg_stencil_t *stencil, const bmg_comm_t *comm, const bmg_params_t *params,
                            void *cuda_stream, bmg_solver_t *out);

/* Local layout of this rank's level-0 arrays: stored global rows [row0, row0+nrows),
 * owned rows [ylo, yhi), distributed levels kdist.  Any pointer may be NULL.  For a
 * single-GPU handle: row0 = 0, nrows = ny+2, [1, ny+1), kdist = 0. */
bmg_status_t bmg_local_rows(bmg_solver_t h, int *row0, int *nrows, int *ylo, int *yhi, int *kdist);

/* Free everything owned by the handle (synchronises the device). NULL is OK. */
bmg_status_t bmg_destroy(bmg_solver_t h);

const char *bmg_strerror(bmg_status_t s);
const char *bmg_last_error_detail(void);

#ifdef __cplusplus
}
#endif
#endif /* BMG_H */
