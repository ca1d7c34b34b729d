/*
 * oracle/bmg_oracle.c -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.
 *
 * A plain, slow, single-threaded fp64 CPU implementation of the 2-D BoxMG
 * V-cycle and its setup, written step by step from the paper
 * (/root/reference/PAPER.md, "P:<line>") and, where the paper delegates to
 * Dendy/Reisner (§2), from the readings fixed in SURVEY.md §8(c)
 * ("c0".."c15"), every one of which is listed in DESIGN.md §3.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  It shares no code, header,
 * table or helper with the CUDA path (paper_2502_05279_b200/csrc); neither
 * includes or links the other.  Built with -O2 -ffp-contract=off so that no
 * multiply-add is contracted: every expression is evaluated as written.
 *
 * Storage (c0): 0-based padded grids, i in [0,nx+1] (x fastest), j in
 * [0,ny+1]; interior [1,nx]x[1,ny]; the ring is the homogeneous Dirichlet
 * ghost.  A grid function g is g[j*(nx+2)+i].  A stencil is stored in FULL
 * (all 9 entries, matrix signs) array-of-structures form, entry order as
 * drawn in fig:stencil_operator: SW,S,SE,W,O,E,NW,N,NE.
 * Interpolation weights ("Ci", fig:restrict_kernel P:173-182) are 8 per
 * coarse index over [0,ncx+1]x[0,ncy+1], order LNE,LA,LNW,LR,LL,LSE,LB,LSW
 * (SPEC.md S:397-400 order), zero-initialised (c3).
 *
 * Parity pins: every function below is pinned by a `-m "not gpu"` test in
 * tests/test_oracle_*.py (closed forms, dense scipy definitions, golden
 * fixtures, brute force).  No function is "parity unpinned".
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---- status codes (mirror SURVEY §8(b) meanings; independent values) ---- */
#define ORC_OK 0
#define ORC_EINVAL 1
#define ORC_ENOMEM 2
#define ORC_ENOTSPD 5
#define ORC_ENOTCONV 6

/* ---- relaxation modes (c6 point GS; c11 line GS) ---- */
#define ORC_POINT 0
#define ORC_XLINES 1
#define ORC_YLINES 2
#define ORC_ALTLINES 3

/* ---- stencil entry order (fig:stencil_operator) ---- */
enum { SW = 0, S_ = 1, SE = 2, W_ = 3, O_ = 4, E_ = 5, NW = 6, N_ = 7, NE = 8 };
static const int DX[9] = {-1, 0, 1, -1, 0, 1, -1, 0, 1};
static const int DY[9] = {-1, -1, -1, 0, 0, 0, 1, 1, 1};

/* ---- interpolation weight order (fig:restrict_kernel names) ---- */
enum { LNE = 0, LA = 1, LNW = 2, LR = 3, LL = 4, LSE = 5, LB = 6, LSW = 7 };

static size_t gidx(int nx, int i, int j) { return (size_t)j * (size_t)(nx + 2) + (size_t)i; }
static int interior(int nx, int ny, int i, int j) { return i >= 1 && i <= nx && j >= 1 && j <= ny; }

/* c1: n_{l+1} = floor(n_l / 2) per dimension (fig:loop_indices index map
 * I=(IC-1)*2; i = istart+(ic-1)*2). */
int orc_coarsen(int n) { return n / 2; }

/* c1: number of levels: coarsen until min(nx,ny) <= coarsest (or max_levels). */
int orc_count_levels(int nx, int ny, int coarsest, int max_levels)
{
    int L = 1;
    while ((nx < ny ? nx : ny) > coarsest && (max_levels <= 0 || L < max_levels)) {
        nx = orc_coarsen(nx);
        ny = orc_coarsen(ny);
        L++;
    }
    return L;
}

/*
 * c0 + c2 (Dirichlet elimination): expand the symmetric-half
 * planes {O,W,S[,SW,NW]} (pitched, row-major, element (i,j) at p[j*pitch+i])
 * into the full 9-entry stencil.  Other half by symmetry:
 *   E(i,j)=W(i+1,j), N(i,j)=S(i,j+1), NE(i,j)=SW(i+1,j+1), SE(i,j)=NW(i+1,j-1).
 * Every coupling whose target is a ghost point is set to 0; ghost rows are 0.
 * Returns ORC_EINVAL if some interior a_O <= 0.
 */
int orc_expand_stencil(int nx, int ny, int kind, long pitch, const double *O, const double *W,
                       const double *S, const double *SWp, const double *NWp, double *st)
{
    memset(st, 0, sizeof(double) * 9 * (size_t)(nx + 2) * (size_t)(ny + 2));
    for (int j = 1; j <= ny; j++)
        for (int i = 1; i <= nx; i++) {
            double *a = st + 9 * gidx(nx, i, j);
            size_t p = (size_t)j * pitch + i;
            a[O_] = O[p];
            a[W_] = W[p];
            a[S_] = S[p];
            a[E_] = W[p + 1];
            a[N_] = S[p + pitch];
            if (kind == 9) {
                a[SW] = SWp[p];
                a[NW] = NWp[p];
                a[NE] = SWp[p + pitch + 1];
                a[SE] = NWp[p - pitch + 1];
            }
            for (int d = 0; d < 9; d++)
                if (d != O_ && !interior(nx, ny, i + DX[d], j + DY[d]))
                    a[d] = 0.0;
            if (!(a[O_] > 0.0))
                return ORC_EINVAL;
        }
    return ORC_OK;
}

/*
 * c3: operator-induced interpolation (Dendy collapse with BoxMG's row-sum
 * switch, hard-test reading (i)).  The paper defers the formula to Dendy
 * 1982/83/2010 and Reisner 2018 (§2); the CI naming follows the
 * fig:restrict_kernel listing: the name is the direction from the
 * fine point to the coarse point it interpolates from.
 * Fine point types by parity (c0): C (even,even), X (odd,even),
 * Y (even,odd), Z (odd,odd).  X at (2I-1,2J), Y at (2I,2J-1), Z at
 * (2I-1,2J-1) are all stored at coarse index (I,J).
 * Phase 1: X and Y points.  Phase 2: Z points (they use edge weights).
 * Returns ORC_EINVAL if a denominator is <= 0 (reading (iii)).
 */
int orc_setup_interp(int nx, int ny, const double *st, double *ci)
{
    int ncx = orc_coarsen(nx), ncy = orc_coarsen(ny);
    memset(ci, 0, sizeof(double) * 8 * (size_t)(ncx + 2) * (size_t)(ncy + 2));
    for (int phase = 1; phase <= 2; phase++)
        for (int j = 1; j <= ny; j++)
            for (int i = 1; i <= nx; i++) {
                int iodd = i & 1, jodd = j & 1;
                if (!iodd && !jodd)
                    continue; /* C point: weight 1, implicit */
                int isZ = iodd && jodd;
                if ((phase == 1) == isZ)
                    continue;
                const double *a = st + 9 * gidx(nx, i, j);
                /* collapsed couplings and row sum (c3) */
                double cW = -(a[W_] + a[NW] + a[SW]);
                double cE = -(a[E_] + a[NE] + a[SE]);
                double cS = -(a[S_] + a[SW] + a[SE]);
                double cN = -(a[N_] + a[NW] + a[NE]);
                double sig = -(a[SW] + a[S_] + a[SE] + a[W_] + a[E_] + a[NW] + a[N_] + a[NE]);
                double R = a[O_] - sig;
                if (iodd && !jodd) { /* X point, stored at (I,J) = ((i+1)/2, j/2) */
                    int I = (i + 1) / 2, J = j / 2;
                    double eps = fmin(fabs(cW), fabs(cE)) / a[O_];
                    double den = cW + cE + (R > eps * sig ? R : 0.0);
                    if (!(den > 0.0))
                        return ORC_EINVAL;
                    double *w = ci + 8 * gidx(ncx, I, J);
                    w[LL] = cW / den; /* toward coarse (I-1,J) */
                    w[LR] = cE / den; /* toward coarse (I,J)   */
                } else if (!iodd && jodd) { /* Y point, stored at (i/2, (j+1)/2) */
                    int I = i / 2, J = (j + 1) / 2;
                    double eps = fmin(fabs(cS), fabs(cN)) / a[O_];
                    double den = cS + cN + (R > eps * sig ? R : 0.0);
                    if (!(den > 0.0))
                        return ORC_EINVAL;
                    double *w = ci + 8 * gidx(ncx, I, J);
                    w[LB] = cS / den; /* toward coarse (I,J-1) */
                    w[LA] = cN / den; /* toward coarse (I,J)   */
                } else { /* Z point, stored at ((i+1)/2, (j+1)/2) */
                    int I = (i + 1) / 2, J = (j + 1) / 2;
                    double eps = fmin(fmin(fabs(cW), fabs(cE)), fmin(fabs(cS), fabs(cN))) / a[O_];
                    double den = sig + (R > eps * sig ? R : 0.0);
                    if (!(den > 0.0))
                        return ORC_EINVAL;
                    const double *wIJ = ci + 8 * gidx(ncx, I, J);       /* X(I,J) north, Y(I,J) east */
                    const double *wIm = ci + 8 * gidx(ncx, I - 1, J);   /* Y(I-1,J) west  */
                    const double *wJm = ci + 8 * gidx(ncx, I, J - 1);   /* X(I,J-1) south */
                    double lne = (-a[NE] - a[N_] * wIJ[LR] - a[E_] * wIJ[LA]) / den;
                    double lnw = (-a[NW] - a[N_] * wIJ[LL] - a[W_] * wIm[LA]) / den;
                    double lse = (-a[SE] - a[S_] * wJm[LR] - a[E_] * wIJ[LB]) / den;
                    double lsw = (-a[SW] - a[S_] * wJm[LL] - a[W_] * wIm[LB]) / den;
                    double *w = ci + 8 * gidx(ncx, I, J);
                    w[LNE] = lne; /* toward (I,J)     */
                    w[LNW] = lnw; /* toward (I-1,J)   */
                    w[LSE] = lse; /* toward (I,J-1)   */
                    w[LSW] = lsw; /* toward (I-1,J-1) */
                }
            }
    return ORC_OK;
}

/*
 * c7: the row of P for fine point (i,j): up to 4 (coarse I, coarse J, weight)
 * entries, ghost coarse targets included (callers drop them).
 */
static int prow(int nx, const double *ci, int i, int j, int *CI_, int *CJ_, double *wt)
{
    int ncx = orc_coarsen(nx);
    int iodd = i & 1, jodd = j & 1;
    if (!iodd && !jodd) {
        CI_[0] = i / 2; CJ_[0] = j / 2; wt[0] = 1.0;
        return 1;
    }
    if (iodd && !jodd) {
        int I = (i + 1) / 2, J = j / 2;
        const double *w = ci + 8 * gidx(ncx, I, J);
        CI_[0] = I - 1; CJ_[0] = J; wt[0] = w[LL];
        CI_[1] = I;     CJ_[1] = J; wt[1] = w[LR];
        return 2;
    }
    if (!iodd && jodd) {
        int I = i / 2, J = (j + 1) / 2;
        const double *w = ci + 8 * gidx(ncx, I, J);
        CI_[0] = I; CJ_[0] = J - 1; wt[0] = w[LB];
        CI_[1] = I; CJ_[1] = J;     wt[1] = w[LA];
        return 2;
    }
    {
        int I = (i + 1) / 2, J = (j + 1) / 2;
        const double *w = ci + 8 * gidx(ncx, I, J);
        CI_[0] = I - 1; CJ_[0] = J - 1; wt[0] = w[LSW];
        CI_[1] = I;     CJ_[1] = J - 1; wt[1] = w[LSE];
        CI_[2] = I - 1; CJ_[2] = J;     wt[2] = w[LNW];
        CI_[3] = I;     CJ_[3] = J;     wt[3] = w[LNE];
        return 4;
    }
}

/*
 * c4: Galerkin coarse operator A_c = P^T A P over interior coarse points
 * ("construction of coarse [operators] through local stencil operations",
 * P:100-101; R = P^T, unscaled, as the unit centre weight of
 * fig:restrict_kernel implies).  Computed by SCATTER: for each
 * interior fine f, each stencil neighbour g of f (incl. f), each coarse C
 * with P(f,C) != 0 and each D with P(g,D) != 0, accumulate
 * P(f,C)*A(f,g)*P(g,D) into A_c(C, D-C).  Output: full 9-entry coarse stencil.
 */
int orc_rap(int nx, int ny, const double *st, const double *ci, double *stc)
{
    int ncx = orc_coarsen(nx), ncy = orc_coarsen(ny);
    memset(stc, 0, sizeof(double) * 9 * (size_t)(ncx + 2) * (size_t)(ncy + 2));
    int fC[4], fJ[4], gC[4], gJ[4];
    double fw[4], gw[4];
    for (int j = 1; j <= ny; j++)
        for (int i = 1; i <= nx; i++) {
            const double *a = st + 9 * gidx(nx, i, j);
            int nf = prow(nx, ci, i, j, fC, fJ, fw);
            for (int d = 0; d < 9; d++) {
                int gi = i + DX[d], gj = j + DY[d];
                if (!interior(nx, ny, gi, gj))
                    continue;
                int ng = prow(nx, ci, gi, gj, gC, gJ, gw);
                for (int a1 = 0; a1 < nf; a1++) {
                    if (!interior(ncx, ncy, fC[a1], fJ[a1]))
                        continue;
                    for (int b1 = 0; b1 < ng; b1++) {
                        if (!interior(ncx, ncy, gC[b1], gJ[b1]))
                            continue;
                        int ox = gC[b1] - fC[a1], oy = gJ[b1] - fJ[a1];
                        if (ox < -1 || ox > 1 || oy < -1 || oy > 1)
                            return ORC_EINVAL; /* cannot happen: P has 3x3 support */
                        int e = (oy + 1) * 3 + (ox + 1);
                        stc[9 * gidx(ncx, fC[a1], fJ[a1]) + e] += fw[a1] * a[d] * gw[b1];
                    }
                }
            }
        }
    return ORC_OK;
}

/* colour of point (i,j) (c6): 2 colours on 5-pt levels, 4 on 9-pt levels */
static int colour(int kind, int i, int j) { return kind == 5 ? ((i + j) & 1) : ((i & 1) + 2 * (j & 1)); }

/* A u at interior point (i,j), summed over the 8 off-diagonal entries in
 * fig:stencil_operator order (diagonal excluded). */
static double offdiag_dot(int nx, const double *a, const double *u, int i, int j)
{
    double s = 0.0;
    for (int d = 0; d < 9; d++)
        if (d != O_)
            s += a[d] * u[gidx(nx, i + DX[d], j + DY[d])];
    return s;
}

/*
 * c6: Gauss-Seidel point relaxation (fig:vcycle_flowchart "Gauss Seidel",
 * P:96) in multicolour order: one sweep = for each colour c in
 * ascending order, u_p <- (f_p - sum_{q!=p} A_pq u_q) / A_pp for every p of
 * colour c.  rev = 1 (c12, the adjoint smoother of the symmetric cycle):
 * colours in descending order.
 */
static void relax_point(int nx, int ny, int kind, const double *st, const double *f, double *u, int nsweeps, int rev)
{
    int ncol = kind == 5 ? 2 : 4;
    for (int s = 0; s < nsweeps; s++)
        for (int cc = 0; cc < ncol; cc++) {
            int c = rev ? ncol - 1 - cc : cc;
            for (int j = 1; j <= ny; j++)
                for (int i = 1; i <= nx; i++) {
                    if (colour(kind, i, j) != c)
                        continue;
                    const double *a = st + 9 * gidx(nx, i, j);
                    size_t p = gidx(nx, i, j);
                    u[p] = (f[p] - offdiag_dot(nx, a, u, i, j)) / a[O_];
                }
        }
}

void orc_relax(int nx, int ny, int kind, const double *st, const double *f, double *u, int nsweeps)
{
    relax_point(nx, ny, kind, st, f, u, nsweeps, 0);
}

void orc_relax_adjoint(int nx, int ny, int kind, const double *st, const double *f, double *u, int nsweeps)
{
    relax_point(nx, ny, kind, st, f, u, nsweeps, 1);
}

/*
 * Thomas algorithm (tridiagonal LU without pivoting, the textbook
 * forward-elimination / back-substitution): solve
 *   lo[k] x[k-1] + di[k] x[k] + up[k] x[k+1] = rhs[k],  k = 0..n-1,
 * lo[0] and up[n-1] ignored.  x receives the solution; gam is n doubles of
 * scratch.  Returns ORC_ENOTSPD if an elimination pivot is <= 0 (a line block
 * of an SPD operator is SPD, so its pivots are positive).
 */
static int thomas(int n, const double *lo, const double *di, const double *up, const double *rhs, double *x,
                  double *gam)
{
    double beta = di[0];
    if (!(beta > 0.0))
        return ORC_ENOTSPD;
    x[0] = rhs[0] / beta;
    for (int k = 1; k < n; k++) {
        gam[k] = up[k - 1] / beta;
        beta = di[k] - lo[k] * gam[k];
        if (!(beta > 0.0))
            return ORC_ENOTSPD;
        x[k] = (rhs[k] - lo[k] * x[k - 1]) / beta;
    }
    for (int k = n - 2; k >= 0; k--)
        x[k] -= gam[k + 1] * x[k + 1];
    return ORC_OK;
}

/*
 * c11: zebra line Gauss-Seidel (fig:vcycle_flowchart's "Line" relaxation box,
 * P:144; the paper gives no formula, reading in DESIGN.md §3 c11).
 * dir = ORC_XLINES: the lines are the grid rows; one sweep = rows j with
 * j mod 2 == 0 (the rows through coarse points, as c6's colour 0), then rows
 * with j mod 2 == 1.  Every row of a colour is solved exactly for its nx
 * unknowns, the couplings to the two neighbouring rows (the other colour,
 * current values) moved to the right-hand side:
 *   W u(i-1,j) + O u(i,j) + E u(i+1,j)
 *     = f(i,j) - [SW u(i-1,j-1) + S u(i,j-1) + SE u(i+1,j-1)
 *                 + NW u(i-1,j+1) + N u(i,j+1) + NE u(i+1,j+1)]
 * (off-line terms summed in fig:stencil_operator order).  A 9-point stencil
 * couples row j only to rows j-1, j+1, so the rows of one colour are
 * independent.  dir = ORC_YLINES: the same with the roles of x and y swapped
 * (columns i, colour i mod 2, couplings S, N on the line, SW,W,NW,SE,E,NE
 * off it).  dir = ORC_ALTLINES: one sweep = an x-line sweep then a y-line
 * sweep.  Returns ORC_ENOTSPD if a line pivot is <= 0 (u then partial).
 */
static int relax_lines(int nx, int ny, const double *st, const double *f, double *u, int nsweeps, int dir, int rev);

int orc_relax_lines(int nx, int ny, const double *st, const double *f, double *u, int nsweeps, int dir)
{
    return relax_lines(nx, ny, st, f, u, nsweeps, dir, 0);
}

/* c12: the adjoint line smoother: each sweep runs its (direction, colour)
 * passes in reverse order (y-lines before x-lines, colour 1 before 0). */
int orc_relax_lines_adjoint(int nx, int ny, const double *st, const double *f, double *u, int nsweeps, int dir)
{
    return relax_lines(nx, ny, st, f, u, nsweeps, dir, 1);
}

static int relax_lines(int nx, int ny, const double *st, const double *f, double *u, int nsweeps, int dir, int rev)
{
    int nmax = nx > ny ? nx : ny;
    double *lo = (double *)malloc(sizeof(double) * (size_t)nmax * 6);
    if (!lo)
        return ORC_ENOMEM;
    double *di = lo + nmax, *up = di + nmax, *rhs = up + nmax, *x = rhs + nmax, *gam = x + nmax;
    int rc = ORC_OK;
    for (int s = 0; s < nsweeps && rc == ORC_OK; s++) {
        for (int pp = 0; pp < 2 && rc == ORC_OK; pp++) {
            int pass = rev ? 1 - pp : pp;
            int on = pass == 0 ? (dir == ORC_XLINES || dir == ORC_ALTLINES) : (dir == ORC_YLINES || dir == ORC_ALTLINES);
            if (!on)
                continue;
            int ylines = pass == 1;
            int nl = ylines ? nx : ny;  /* number of lines */
            int n = ylines ? ny : nx;   /* unknowns per line */
            for (int cc = 0; cc < 2 && rc == ORC_OK; cc++)
                for (int line = 1; line <= nl && rc == ORC_OK; line++) {
                    int c = rev ? 1 - cc : cc;
                    if ((line & 1) != c)
                        continue;
                    for (int k = 0; k < n; k++) {
                        int i = ylines ? line : k + 1, j = ylines ? k + 1 : line;
                        const double *a = st + 9 * gidx(nx, i, j);
                        double off = 0.0;
                        for (int d = 0; d < 9; d++) {
                            int online = ylines ? DX[d] == 0 : DY[d] == 0;
                            if (!online)
                                off += a[d] * u[gidx(nx, i + DX[d], j + DY[d])];
                        }
                        rhs[k] = f[gidx(nx, i, j)] - off;
                        di[k] = a[O_];
                        lo[k] = ylines ? a[S_] : a[W_];
                        up[k] = ylines ? a[N_] : a[E_];
                    }
                    rc = thomas(n, lo, di, up, rhs, x, gam);
                    for (int k = 0; k < n && rc == ORC_OK; k++) {
                        int i = ylines ? line : k + 1, j = ylines ? k + 1 : line;
                        u[gidx(nx, i, j)] = x[k];
                    }
                }
        }
    }
    free(lo);
    return rc;
}

/* Relaxation of the cycle: point GS (c6) or line GS (c11) by mode; rev = 1
 * the adjoint ordering (c12). */
static int relax_mode(int mode, int nx, int ny, int kind, const double *st, const double *f, double *u, int nsweeps,
                      int rev)
{
    if (mode == ORC_POINT) {
        relax_point(nx, ny, kind, st, f, u, nsweeps, rev);
        return ORC_OK;
    }
    return relax_lines(nx, ny, st, f, u, nsweeps, mode, rev);
}

/* fig:vcycle_flowchart "Residual": r = f - A u on the interior; ring 0. */
void orc_residual(int nx, int ny, const double *st, const double *f, const double *u, double *r)
{
    memset(r, 0, sizeof(double) * (size_t)(nx + 2) * (size_t)(ny + 2));
    for (int j = 1; j <= ny; j++)
        for (int i = 1; i <= nx; i++) {
            const double *a = st + 9 * gidx(nx, i, j);
            size_t p = gidx(nx, i, j);
            r[p] = f[p] - (a[O_] * u[p] + offdiag_dot(nx, a, u, i, j));
        }
}

/*
 * c5: restriction, the fig:restrict_kernel listing in c0
 * indices (Fortran i = istart+(ic-1)*2 with istart = 1 -> fine 2I):
 *   QC(I,J) = Ci(I,J,LNE)Q(2I-1,2J-1) + Ci(I,J,LA)Q(2I,2J-1)
 *           + Ci(I+1,J,LNW)Q(2I+1,2J-1) + Ci(I,J,LR)Q(2I-1,2J) + Q(2I,2J)
 *           + Ci(I+1,J,LL)Q(2I+1,2J) + Ci(I,J+1,LSE)Q(2I-1,2J+1)
 *           + Ci(I,J+1,LB)Q(2I,2J+1) + Ci(I+1,J+1,LSW)Q(2I+1,2J+1)
 * summed in the listing's order, for interior coarse (I,J); ring 0.
 */
void orc_restrict(int nx, int ny, const double *ci, const double *q, double *qc)
{
    int ncx = orc_coarsen(nx), ncy = orc_coarsen(ny);
    memset(qc, 0, sizeof(double) * (size_t)(ncx + 2) * (size_t)(ncy + 2));
    for (int J = 1; J <= ncy; J++)
        for (int I = 1; I <= ncx; I++) {
            int i = 2 * I, j = 2 * J;
            const double *c00 = ci + 8 * gidx(ncx, I, J);
            const double *c10 = ci + 8 * gidx(ncx, I + 1, J);
            const double *c01 = ci + 8 * gidx(ncx, I, J + 1);
            const double *c11 = ci + 8 * gidx(ncx, I + 1, J + 1);
            double v = c00[LNE] * q[gidx(nx, i - 1, j - 1)];
            v = v + c00[LA] * q[gidx(nx, i, j - 1)];
            v = v + c10[LNW] * q[gidx(nx, i + 1, j - 1)];
            v = v + c00[LR] * q[gidx(nx, i - 1, j)];
            v = v + q[gidx(nx, i, j)];
            v = v + c10[LL] * q[gidx(nx, i + 1, j)];
            v = v + c01[LSE] * q[gidx(nx, i - 1, j + 1)];
            v = v + c01[LB] * q[gidx(nx, i, j + 1)];
            v = v + c11[LSW] * q[gidx(nx, i + 1, j + 1)];
            qc[gidx(ncx, I, J)] = v;
        }
}

void orc_interp_add(int nx, int ny, const double *ci, const double *e, double *u);

/*
 * c14: BoxMG's affine interpolation-correction (the
 * "r_F/a_O term" of BoxMG's interp_add): u += P e as in c7, plus, at every
 * fine point that is not coincident with a coarse point (X, Y, Z), the
 * residual r (the one restricted on the down leg) divided by the diagonal:
 *   u(F) += (P e)(F) + r(F) / a_O(F),     u(C) += e(C).
 * st: the level's full stencil (a_O at entry O_).
 */
void orc_interp_add_affine(int nx, int ny, const double *ci, const double *e, const double *st, const double *r,
                           double *u)
{
    orc_interp_add(nx, ny, ci, e, u);
    for (int j = 1; j <= ny; j++)
        for (int i = 1; i <= nx; i++) {
            if (!(i & 1) && !(j & 1))
                continue; /* C point */
            size_t p = gidx(nx, i, j);
            u[p] += r[p] / st[9 * p + O_];
        }
}

/*
 * c7: interpolation + correction (fig:vcycle_flowchart "Interpolate",
 * P:152; index map of fig:loop_indices P:382-403): u += P e over the fine
 * interior, P's rows as in prow(); ghost coarse values of e are 0.
 */
void orc_interp_add(int nx, int ny, const double *ci, const double *e, double *u)
{
    int ncx = orc_coarsen(nx), ncy = orc_coarsen(ny);
    int CI_[4], CJ_[4];
    double wt[4];
    for (int j = 1; j <= ny; j++)
        for (int i = 1; i <= nx; i++) {
            int n = prow(nx, ci, i, j, CI_, CJ_, wt);
            double s = 0.0;
            for (int k = 0; k < n; k++)
                if (interior(ncx, ncy, CI_[k], CJ_[k]))
                    s += wt[k] * e[gidx(ncx, CI_[k], CJ_[k])];
            u[gidx(nx, i, j)] += s;
        }
}

/*
 * c8: dense Cholesky A = L L^T (fig:vcycle_flowchart "Cholesky", P:158;
 * cuBLAS in the paper's runs).  A is n*n row-major, overwritten by L
 * in its lower triangle (upper triangle zeroed).  Pivot <= 0 -> ORC_ENOTSPD
 * (SPEC S:363).
 */
int orc_chol_factor(int n, double *A)
{
    for (int j = 0; j < n; j++) {
        double d = A[(size_t)j * n + j];
        for (int k = 0; k < j; k++)
            d -= A[(size_t)j * n + k] * A[(size_t)j * n + k];
        if (!(d > 0.0))
            return ORC_ENOTSPD;
        double ljj = sqrt(d);
        A[(size_t)j * n + j] = ljj;
        for (int i = j + 1; i < n; i++) {
            double s = A[(size_t)i * n + j];
            for (int k = 0; k < j; k++)
                s -= A[(size_t)i * n + k] * A[(size_t)j * n + k];
            A[(size_t)i * n + j] = s / ljj;
        }
        for (int k = j + 1; k < n; k++)
            A[(size_t)j * n + k] = 0.0;
    }
    return ORC_OK;
}

/* c8: forward then backward substitution with L (in place on b). */
void orc_chol_solve(int n, const double *L, double *b)
{
    for (int i = 0; i < n; i++) {
        double s = b[i];
        for (int k = 0; k < i; k++)
            s -= L[(size_t)i * n + k] * b[k];
        b[i] = s / L[(size_t)i * n + i];
    }
    for (int i = n - 1; i >= 0; i--) {
        double s = b[i];
        for (int k = i + 1; k < n; k++)
            s -= L[(size_t)k * n + i] * b[k];
        b[i] = s / L[(size_t)i * n + i];
    }
}

/* c8: dense assembly of the level operator in lexicographic order (x fastest). */
void orc_assemble_dense(int nx, int ny, const double *st, double *A)
{
    int n = nx * ny;
    memset(A, 0, sizeof(double) * (size_t)n * (size_t)n);
    for (int j = 1; j <= ny; j++)
        for (int i = 1; i <= nx; i++) {
            const double *a = st + 9 * gidx(nx, i, j);
            int p = (j - 1) * nx + (i - 1);
            for (int d = 0; d < 9; d++) {
                int qi = i + DX[d], qj = j + DY[d];
                if (!interior(nx, ny, qi, qj))
                    continue;
                A[(size_t)p * n + (size_t)((qj - 1) * nx + (qi - 1))] = a[d];
            }
        }
}

/* l2 norm over the interior ("l2 norm"), lexicographic summation. */
double orc_norm2(int nx, int ny, const double *g)
{
    double s = 0.0;
    for (int j = 1; j <= ny; j++)
        for (int i = 1; i <= nx; i++)
            s += g[gidx(nx, i, j)] * g[gidx(nx, i, j)];
    return sqrt(s);
}

/* ------------------------------------------------------------------------
 * Hierarchy + V-cycle + solve (c1, c9; fig:vcycle_flowchart P:108-162)
 * ---------------------------------------------------------------------- */
#define ORC_MAXLEV 32
typedef struct {
    int nx, ny, kind;
    double *st; /* full 9-entry stencil */
    double *ci; /* interpolation from level l+1 to l (NULL on coarsest) */
    double *u, *f, *r;
} orc_level;

typedef struct {
    int L, nu1, nu2, relax, cycle_sym, affine;
    orc_level lv[ORC_MAXLEV];
    double *chol; /* coarsest L factor, n*n */
    int nco;
} orc_hier;

void orc_destroy(orc_hier *h)
{
    if (!h)
        return;
    for (int l = 0; l < h->L; l++) {
        free(h->lv[l].st);
        free(h->lv[l].ci);
        free(h->lv[l].u);
        free(h->lv[l].f);
        free(h->lv[l].r);
    }
    free(h->chol);
    free(h);
}

/*
 * Setup: expand the fine stencil (c0/c2), then per level l < L-1
 * interpolation (c3) and Galerkin operator (c4), then the coarsest dense
 * Cholesky factor (c8).  Coarse levels are 9-point.
 */
int orc_setup(int nx, int ny, int kind, long pitch, const double *O, const double *W, const double *S,
              const double *SWp, const double *NWp, int nu1, int nu2, int coarsest, int max_levels, int relax,
              int cycle_sym, orc_hier **out)
{
    *out = NULL;
    if (nx < 1 || ny < 1 || (kind != 5 && kind != 9) || pitch < nx + 2 || relax < ORC_POINT || relax > ORC_ALTLINES ||
        (cycle_sym != 0 && cycle_sym != 1))
        return ORC_EINVAL;
    orc_hier *h = (orc_hier *)calloc(1, sizeof(orc_hier));
    if (!h)
        return ORC_ENOMEM;
    h->L = orc_count_levels(nx, ny, coarsest, max_levels);
    if (h->L > ORC_MAXLEV) {
        free(h);
        return ORC_EINVAL;
    }
    h->nu1 = nu1;
    h->nu2 = nu2;
    h->relax = relax;
    h->cycle_sym = cycle_sym;
    int cx = nx, cy = ny;
    for (int l = 0; l < h->L; l++) {
        orc_level *v = &h->lv[l];
        v->nx = cx;
        v->ny = cy;
        v->kind = l == 0 ? kind : 9;
        size_t np = (size_t)(cx + 2) * (size_t)(cy + 2);
        v->st = (double *)calloc(9 * np, sizeof(double));
        v->u = (double *)calloc(np, sizeof(double));
        v->f = (double *)calloc(np, sizeof(double));
        v->r = (double *)calloc(np, sizeof(double));
        if (l + 1 < h->L)
            v->ci = (double *)calloc(8 * (size_t)(cx / 2 + 2) * (size_t)(cy / 2 + 2), sizeof(double));
        if (!v->st || !v->u || !v->f || !v->r || (l + 1 < h->L && !v->ci)) {
            orc_destroy(h);
            return ORC_ENOMEM;
        }
        cx = orc_coarsen(cx);
        cy = orc_coarsen(cy);
    }
    int rc = orc_expand_stencil(nx, ny, kind, pitch, O, W, S, SWp, NWp, h->lv[0].st);
    for (int l = 0; rc == ORC_OK && l + 1 < h->L; l++) {
        orc_level *v = &h->lv[l];
        rc = orc_setup_interp(v->nx, v->ny, v->st, v->ci);
        if (rc == ORC_OK)
            rc = orc_rap(v->nx, v->ny, v->st, v->ci, h->lv[l + 1].st);
    }
    /* c11: every line block of every relaxed level must have positive pivots */
    for (int l = 0; rc == ORC_OK && relax != ORC_POINT && l + 1 < h->L; l++) {
        orc_level *v = &h->lv[l];
        size_t np = (size_t)(v->nx + 2) * (size_t)(v->ny + 2);
        double *z = (double *)calloc(np, sizeof(double));
        if (!z)
            rc = ORC_ENOMEM;
        else {
            rc = orc_relax_lines(v->nx, v->ny, v->st, z, z, 1, relax);
            free(z);
        }
    }
    if (rc == ORC_OK) {
        orc_level *c = &h->lv[h->L - 1];
        h->nco = c->nx * c->ny;
        h->chol = (double *)malloc(sizeof(double) * (size_t)h->nco * (size_t)h->nco);
        if (!h->chol)
            rc = ORC_ENOMEM;
        else {
            orc_assemble_dense(c->nx, c->ny, c->st, h->chol);
            rc = orc_chol_factor(h->nco, h->chol);
        }
    }
    if (rc != ORC_OK) {
        orc_destroy(h);
        return rc;
    }
    *out = h;
    return ORC_OK;
}

int orc_num_levels(const orc_hier *h) { return h->L; }

/* c14: switch the cycle's interpolation to the affine BoxMG form (on = 1). */
void orc_set_affine(orc_hier *h, int on) { h->affine = on != 0; }

void orc_level_shape(const orc_hier *h, int l, int *nx, int *ny, int *kind)
{
    *nx = h->lv[l].nx;
    *ny = h->lv[l].ny;
    *kind = h->lv[l].kind;
}

/* copy out level l's full stencil ((nx+2)(ny+2)*9) and CI ((ncx+2)(ncy+2)*8, may be NULL) */
void orc_export_level(const orc_hier *h, int l, double *st, double *ci)
{
    const orc_level *v = &h->lv[l];
    memcpy(st, v->st, sizeof(double) * 9 * (size_t)(v->nx + 2) * (size_t)(v->ny + 2));
    if (ci && v->ci)
        memcpy(ci, v->ci, sizeof(double) * 8 * (size_t)(v->nx / 2 + 2) * (size_t)(v->ny / 2 + 2));
}

/* c8 per cycle: u = A_L^{-1} f on the coarsest level */
static void coarse_solve(orc_hier *h, orc_level *c)
{
    double *b = (double *)malloc(sizeof(double) * (size_t)h->nco);
    for (int j = 1; j <= c->ny; j++)
        for (int i = 1; i <= c->nx; i++)
            b[(j - 1) * c->nx + (i - 1)] = c->f[gidx(c->nx, i, j)];
    orc_chol_solve(h->nco, h->chol, b);
    for (int j = 1; j <= c->ny; j++)
        for (int i = 1; i <= c->nx; i++)
            c->u[gidx(c->nx, i, j)] = b[(j - 1) * c->nx + (i - 1)];
    free(b);
}

/*
 * c9: V(nu1,nu2) cycle at level l (fig:vcycle_flowchart): relax nu1 (c6
 * point or c11 line GS, the hierarchy's mode; line pivots checked at setup;
 * with cycle_sym the post-smoother is the adjoint ordering, c12), r = f -
 * A u, f_{l+1} = P^T r, u_{l+1} = 0, recurse (coarsest: Cholesky solve),
 * u += P u_{l+1}, relax nu2.
 */
static void vcycle_level(orc_hier *h, int l)
{
    orc_level *v = &h->lv[l];
    if (l == h->L - 1) {
        coarse_solve(h, v);
        return;
    }
    orc_level *c = &h->lv[l + 1];
    relax_mode(h->relax, v->nx, v->ny, v->kind, v->st, v->f, v->u, h->nu1, 0);
    orc_residual(v->nx, v->ny, v->st, v->f, v->u, v->r);
    orc_restrict(v->nx, v->ny, v->ci, v->r, c->f);
    memset(c->u, 0, sizeof(double) * (size_t)(c->nx + 2) * (size_t)(c->ny + 2));
    vcycle_level(h, l + 1);
    if (h->affine) /* c14: r still holds the residual restricted above */
        orc_interp_add_affine(v->nx, v->ny, v->ci, c->u, v->st, v->r, v->u);
    else
        orc_interp_add(v->nx, v->ny, v->ci, c->u, v->u);
    relax_mode(h->relax, v->nx, v->ny, v->kind, v->st, v->f, v->u, h->nu2, h->cycle_sym);
}

/* ncycles V-cycles on the fine level; f, u are (nx+2)*(ny+2), u in/out. */
void orc_vcycle(orc_hier *h, const double *f, double *u, int ncycles)
{
    orc_level *v = &h->lv[0];
    size_t np = (size_t)(v->nx + 2) * (size_t)(v->ny + 2);
    memcpy(v->f, f, sizeof(double) * np);
    memcpy(v->u, u, sizeof(double) * np);
    for (int k = 0; k < ncycles; k++)
        vcycle_level(h, 0);
    memcpy(u, v->u, sizeof(double) * np);
}

/* fine-level residual norm ||f - A u||_2 */
double orc_residual_norm(orc_hier *h, const double *f, const double *u)
{
    orc_level *v = &h->lv[0];
    orc_residual(v->nx, v->ny, v->st, f, u, v->r);
    return orc_norm2(v->nx, v->ny, v->r);
}

/*
 * Solve loop (c9): hist[0] = ||f - A x0||; cycle until
 * ||r_k|| <= tol*||f|| or maxiter.  ||f|| = 0 -> x = 0, 0 iterations.
 * hist has room for maxiter+1 entries (may be NULL).
 */
int orc_solve(orc_hier *h, const double *f, double *u, double tol, int maxiter, int *iters, double *hist)
{
    orc_level *v = &h->lv[0];
    size_t np = (size_t)(v->nx + 2) * (size_t)(v->ny + 2);
    double fn = orc_norm2(v->nx, v->ny, f);
    *iters = 0;
    if (fn == 0.0) {
        memset(u, 0, sizeof(double) * np);
        if (hist)
            hist[0] = 0.0;
        return ORC_OK;
    }
    double rn = orc_residual_norm(h, f, u);
    if (hist)
        hist[0] = rn;
    int k = 0;
    while (rn > tol * fn && k < maxiter) {
        orc_vcycle(h, f, u, 1);
        k++;
        rn = orc_residual_norm(h, f, u);
        if (hist)
            hist[k] = rn;
    }
    *iters = k;
    return rn <= tol * fn ? ORC_OK : ORC_ENOTCONV;
}

/* ------------------------------------------------------------------------
 * c15: block multi-RHS solve (§5, "solve
 * several initial vectors in block fashion").  nrhs independent systems
 * A x_c = f_c share the hierarchy; each block step applies one V-cycle (c9)
 * to every column, then measures every column's residual.  The block stops
 * when EVERY column meets its own test ||r_c|| <= tol ||f_c|| (a column that
 * met it earlier keeps being cycled), or after maxiter block steps.  A column
 * with f_c = 0 is set to x_c = 0 and counts as converged.
 * f, u: nrhs grid functions one after another ((ny+2)(nx+2) each);
 * hist: (maxiter+1) rows of nrhs norms, row k after k block steps.
 * ---------------------------------------------------------------------- */
int orc_solve_block(orc_hier *h, int nrhs, const double *f, double *u, double tol, int maxiter, int *iters,
                    double *hist)
{
    orc_level *v = &h->lv[0];
    size_t np = (size_t)(v->nx + 2) * (size_t)(v->ny + 2);
    double *fn = malloc(sizeof(double) * (size_t)nrhs), *rn = malloc(sizeof(double) * (size_t)nrhs);
    if (!fn || !rn) {
        free(fn);
        free(rn);
        return ORC_ENOMEM;
    }
    for (int c = 0; c < nrhs; c++) {
        fn[c] = orc_norm2(v->nx, v->ny, f + c * np);
        if (fn[c] == 0.0)
            memset(u + c * np, 0, sizeof(double) * np);
        rn[c] = orc_residual_norm(h, f + c * np, u + c * np);
        if (hist)
            hist[c] = rn[c];
    }
    int k = 0;
    for (;;) {
        int done = 1;
        for (int c = 0; c < nrhs; c++)
            if (rn[c] > tol * fn[c])
                done = 0;
        if (done || k >= maxiter)
            break;
        for (int c = 0; c < nrhs; c++)
            orc_vcycle(h, f + c * np, u + c * np, 1);
        k++;
        for (int c = 0; c < nrhs; c++) {
            rn[c] = orc_residual_norm(h, f + c * np, u + c * np);
            if (hist)
                hist[(size_t)k * nrhs + c] = rn[c];
        }
    }
    int ok = 1;
    for (int c = 0; c < nrhs; c++)
        if (rn[c] > tol * fn[c])
            ok = 0;
    *iters = k;
    free(fn);
    free(rn);
    return ok ? ORC_OK : ORC_ENOTCONV;
}

/* ------------------------------------------------------------------------
 * c13: V-cycle-preconditioned conjugate gradients (the
 * Krylov acceleration Cedar offers around BoxMG)
 * ---------------------------------------------------------------------- */

/* q = A p on the interior (full stencil, fig:stencil_operator order); ring 0. */
static void apply_A(int nx, int ny, const double *st, const double *p, double *q)
{
    memset(q, 0, sizeof(double) * (size_t)(nx + 2) * (size_t)(ny + 2));
    for (int j = 1; j <= ny; j++)
        for (int i = 1; i <= nx; i++) {
            const double *a = st + 9 * gidx(nx, i, j);
            size_t k = gidx(nx, i, j);
            q[k] = a[O_] * p[k] + offdiag_dot(nx, a, p, i, j);
        }
}

/* <a, b> over the interior, lexicographic summation. */
static double dot_int(int nx, int ny, const double *a, const double *b)
{
    double s = 0.0;
    for (int j = 1; j <= ny; j++)
        for (int i = 1; i <= nx; i++)
            s += a[gidx(nx, i, j)] * b[gidx(nx, i, j)];
    return s;
}

/* z = M^{-1} r: one V-cycle of the hierarchy from a zero guess (c9). */
static void precondition(orc_hier *h, const double *r, double *z)
{
    orc_level *v = &h->lv[0];
    size_t np = (size_t)(v->nx + 2) * (size_t)(v->ny + 2);
    memcpy(v->f, r, sizeof(double) * np);
    memset(v->u, 0, sizeof(double) * np);
    vcycle_level(h, 0);
    memcpy(z, v->u, sizeof(double) * np);
}

/*
 * Textbook PCG (Hestenes-Stiefel) with M^{-1} = one V(nu,nu) cycle from a zero
 * guess; M is SPD when nu1 == nu2 and cycle_sym == 1 (the post-smoother is the
 * adjoint of the pre-smoother, c12; R = P^T, Galerkin coarse operators, exact
 * coarsest solve):
 *   r = f - A x; z = M^{-1} r; p = z; rho = <r, z>
 *   repeat: q = A p; alpha = rho / <p, q>; x += alpha p; r -= alpha q;
 *           stop if ||r|| <= tol ||f||; z = M^{-1} r; rho' = <r, z>;
 *           p = z + (rho'/rho) p; rho = rho'.
 * hist[0] = ||f - A x0||, hist[k] = ||r_k|| of the recursively updated r.
 * ORC_EINVAL unless nu1 == nu2 and cycle_sym == 1; ||f|| = 0 -> x = 0, 0 its;
 * ORC_ENOTCONV at maxiter (x and hist valid).
 */
int orc_pcg(orc_hier *h, const double *f, double *x, double tol, int maxiter, int *iters, double *hist)
{
    orc_level *v = &h->lv[0];
    int nx = v->nx, ny = v->ny;
    size_t np = (size_t)(nx + 2) * (size_t)(ny + 2);
    *iters = 0;
    if (h->nu1 != h->nu2 || h->cycle_sym != 1)
        return ORC_EINVAL;
    double fn = orc_norm2(nx, ny, f);
    if (fn == 0.0) {
        memset(x, 0, sizeof(double) * np);
        if (hist)
            hist[0] = 0.0;
        return ORC_OK;
    }
    double *r = (double *)calloc(4 * np, sizeof(double));
    if (!r)
        return ORC_ENOMEM;
    double *z = r + np, *p = z + np, *q = p + np;
    orc_residual(nx, ny, v->st, f, x, r);
    double rn = orc_norm2(nx, ny, r);
    if (hist)
        hist[0] = rn;
    int k = 0;
    if (rn > tol * fn && maxiter > 0) {
        precondition(h, r, z);
        memcpy(p, z, sizeof(double) * np);
        double rho = dot_int(nx, ny, r, z);
        while (k < maxiter) {
            apply_A(nx, ny, v->st, p, q);
            double alpha = rho / dot_int(nx, ny, p, q);
            for (int j = 1; j <= ny; j++)
                for (int i = 1; i <= nx; i++) {
                    size_t t = gidx(nx, i, j);
                    x[t] += alpha * p[t];
                    r[t] -= alpha * q[t];
                }
            k++;
            rn = orc_norm2(nx, ny, r);
            if (hist)
                hist[k] = rn;
            if (rn <= tol * fn)
                break;
            precondition(h, r, z);
            double rho1 = dot_int(nx, ny, r, z);
            double beta = rho1 / rho;
            for (int j = 1; j <= ny; j++)
                for (int i = 1; i <= nx; i++) {
                    size_t t = gidx(nx, i, j);
                    p[t] = z[t] + beta * p[t];
                }
            rho = rho1;
        }
    }
    free(r);
    *iters = k;
    return rn <= tol * fn ? ORC_OK : ORC_ENOTCONV;
}
