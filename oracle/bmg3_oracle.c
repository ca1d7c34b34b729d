/*
 * oracle/bmg3_oracle.c -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.
 *
 * A plain, slow, single-threaded fp64 CPU implementation of 3-D BoxMG with
 * point and plane relaxation ("3-D BoxMG (7/27-point)
 * with plane relaxation", §2 "performance optimizations for
 * operations such as plane relaxation", P:143 fig:vcycle_flowchart's "Plane"
 * box).  The paper gives none of the 3-D formulas; every step follows the
 * readings c16..c23 listed in DESIGN.md §3, each of which reduces to the 2-D
 * reading (c0..c9, bmg_oracle.c) when the third dimension is trivial.
 *
 * Only tests/ and bench.py's cpu_baseline / --impl reference legs may load
 * this library.  It shares no code, header, table or helper with the CUDA
 * path (paper_2502_05279_b200/csrc).  It is linked with the 2-D oracle
 * (bmg_oracle.c) whose V-cycle is the plane solver of c23 and whose dense
 * Cholesky is the coarsest solve.  Built -O2 -ffp-contract=off.
 *
 * Storage (c16): 0-based padded grids, g[(k*(ny+2)+j)*(nx+2)+i], interior
 * [1,nx]x[1,ny]x[1,nz], the ring is the homogeneous Dirichlet ghost.  A
 * stencil is stored in FULL (27 entries, matrix signs, array of structures),
 * entry e = (dz+1)*9 + (dy+1)*3 + (dx+1) holds A[p, p+(dx,dy,dz)]; e = 13 is
 * the diagonal.  Interpolation weights: 26 per coarse index over
 * [0,ncx+1]x[0,ncy+1]x[0,ncz+1] (c19 slot layout below), zero-initialised.
 *
 * Parity pins: tests/test_oracle3d.py (closed forms of the 7-/27-point
 * generators, trilinear weights and the Kronecker-product Galerkin operator of
 * the 7-point Laplacian, dense P^T A P, dense colour-ordered Gauss-Seidel and
 * V-cycle, exact zebra block Gauss-Seidel on 3x3 planes, the z-decoupled
 * reduction of plane relaxation to the 2-D cycle, a direct sparse solve).
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>

#define O3_OK 0
#define O3_EINVAL 1
#define O3_ENOMEM 2
#define O3_ENOTSPD 5
#define O3_ENOTCONV 6

#define O3_POINT 0
#define O3_PLANES 1 /* zebra xy-plane relaxation (c23) */

/* the 2-D oracle (bmg_oracle.c): plane solves (c23) and the dense Cholesky (c8) */
int orc_setup(int nx, int ny, int kind, long pitch, const double *O, const double *W, const double *S,
              const double *SWp, const double *NWp, int nu1, int nu2, int coarsest, int max_levels, int relax,
              int cycle_sym, void **out);
void orc_destroy(void *h);
void orc_vcycle(void *h, const double *f, double *u, int ncycles);
int orc_chol_factor(int n, double *A);
void orc_chol_solve(int n, const double *L, double *b);

#define CTR 13
static int EDX(int e) { return e % 3 - 1; }
static int EDY(int e) { return (e / 3) % 3 - 1; }
static int EDZ(int e) { return e / 9 - 1; }
static int ENT(int dx, int dy, int dz) { return (dz + 1) * 9 + (dy + 1) * 3 + (dx + 1); }

static size_t gidx3(int nx, int ny, int i, int j, int k)
{
    return ((size_t)k * (size_t)(ny + 2) + (size_t)j) * (size_t)(nx + 2) + (size_t)i;
}
static int inside(int nx, int ny, int nz, int i, int j, int k)
{
    return i >= 1 && i <= nx && j >= 1 && j <= ny && k >= 1 && k <= nz;
}

/* c17: n_{l+1} = floor(n_l/2) per dimension (c1 in every direction) */
int o3_coarsen(int n) { return n / 2; }

/* c17: coarsen until min(nx,ny,nz) <= coarsest (or max_levels) */
int o3_count_levels(int nx, int ny, int nz, int coarsest, int max_levels)
{
    int L = 1;
    for (;;) {
        int m = nx < ny ? nx : ny;
        m = m < nz ? m : nz;
        if (!(m > coarsest) || (max_levels > 0 && L >= max_levels))
            break;
        nx /= 2;
        ny /= 2;
        nz /= 2;
        L++;
    }
    return L;
}

/*
 * c16 + c18 (Dirichlet elimination, in 3-D): expand the
 * symmetric-half planes into the full 27-entry stencil.  `pl` holds the
 * planes one after another, each (nz+2)(ny+2)(nx+2): kind 7 -> O, W, S, B
 * (entries 12, 10, 4); kind 27 -> O then entries e = 0..12 (the 13 offsets
 * that precede the centre).  The other half by symmetry:
 * A[p, p+o] = A[p+o, p] = plane_{26-e}(p+o) for e > 13.  Couplings into the
 * ghost ring are 0.  EINVAL if some interior a_O <= 0.
 */
int o3_expand_stencil(int nx, int ny, int nz, int kind, const double *pl, double *st)
{
    if (kind != 7 && kind != 27)
        return O3_EINVAL;
    size_t np = (size_t)(nx + 2) * (size_t)(ny + 2) * (size_t)(nz + 2);
    memset(st, 0, sizeof(double) * 27 * np);
    const double *O = pl;
    for (int k = 1; k <= nz; k++)
        for (int j = 1; j <= ny; j++)
            for (int i = 1; i <= nx; i++) {
                double *a = st + 27 * gidx3(nx, ny, i, j, k);
                for (int e = 0; e < 27; e++) {
                    if (e == CTR)
                        continue;
                    int qi = i + EDX(e), qj = j + EDY(e), qk = k + EDZ(e);
                    if (!inside(nx, ny, nz, qi, qj, qk))
                        continue;
                    int le = e < CTR ? e : 26 - e;                        /* stored lower entry */
                    size_t at = e < CTR ? gidx3(nx, ny, i, j, k) : gidx3(nx, ny, qi, qj, qk);
                    const double *plane = NULL;
                    if (kind == 27)
                        plane = pl + (size_t)(1 + le) * np;
                    else if (le == 12)
                        plane = pl + 1 * np; /* W */
                    else if (le == 10)
                        plane = pl + 2 * np; /* S */
                    else if (le == 4)
                        plane = pl + 3 * np; /* B */
                    a[e] = plane ? plane[at] : 0.0;
                }
                a[CTR] = O[gidx3(nx, ny, i, j, k)];
                if (!(a[CTR] > 0.0))
                    return O3_EINVAL;
            }
    return O3_OK;
}

/*
 * c19 slot layout.  A fine point's type is its mask of odd coordinates
 * m = (i&1) | (j&1)<<1 | (k&1)<<2; it is stored at coarse index
 * (I,J,K) = ((i+1)/2 | i/2, ...) (odd | even coordinate).  Its weights go to
 * the 2^|m| coarse corners reached by stepping, on each odd axis, to the lower
 * (I-1) or upper (I) coarse coordinate; corner bit b (b-th odd axis in x,y,z
 * order) = 1 means upper.  Slots: X 0-1, Y 2-3, Z 4-5, XY 6-9, XZ 10-13,
 * YZ 14-17, XYZ 18-25.
 */
static const int SLOT[8] = {-1, 0, 2, 6, 4, 10, 14, 18};

static double *cislot(int ncx, int ncy, double *ci, int I, int J, int K)
{
    return ci + 26 * gidx3(ncx, ncy, I, J, K);
}

/*
 * P(q, C): the weight with which fine point q takes coarse point C
 * (c19/c21): 1 if q = 2C, the stored corner weight if C is one of q's
 * corners, else 0.
 */
static double pw(int ncx, int ncy, const double *ci, int qi, int qj, int qk, int CI, int CJ, int CK)
{
    int q[3] = {qi, qj, qk}, C[3] = {CI, CJ, CK}, Q[3];
    int m = (qi & 1) | (qj & 1) << 1 | (qk & 1) << 2;
    int corner = 0, nb = 0;
    for (int d = 0; d < 3; d++) {
        if (q[d] & 1) {
            Q[d] = (q[d] + 1) / 2;
            if (C[d] == Q[d])
                corner |= 1 << nb;
            else if (C[d] != Q[d] - 1)
                return 0.0;
            nb++;
        } else {
            Q[d] = q[d] / 2;
            if (C[d] != Q[d])
                return 0.0;
        }
    }
    if (m == 0)
        return 1.0;
    return ci[26 * gidx3(ncx, ncy, Q[0], Q[1], Q[2]) + SLOT[m] + corner];
}

/*
 * c19: operator-induced interpolation in 3-D (Dendy's collapse, the paper
 * defers to Dendy/Reisner, §2).  For a fine point p of type m
 * (odd axes S, |S| = 1 line, 2 face, 3 cell), in phases |S| = 1, 2, 3:
 *  - collapse the 27-point row onto the axes in S: b(o) = sum of a over the
 *    offsets that agree with o on S (sum over the even axes);
 *  - sig = -(sum of the 26 off-diagonals), R = a_O - sig (row sum);
 *    sides c_{d,s} = -sum_{o: o_d = s} b(o) for d in S, s = -1, +1;
 *    eps = min |c_{d,s}| / a_O; sig_b = -sum_{o != 0} b(o);
 *    den = sig_b + (R > eps*sig ? R : 0)  (the row-sum switch of c3);
 *  - weight to corner C: w = -(sum_{o != 0} b(o) P(p+o, C)) / den, where
 *    p+o (even axes unchanged) is a coarse point or a point of a lower phase.
 * With no z-couplings this is c3 exactly (X/Y: sig_b = cW+cE; Z: sig_b = sig).
 * EINVAL if a denominator is <= 0.
 */
int o3_setup_interp(int nx, int ny, int nz, const double *st, double *ci)
{
    int ncx = o3_coarsen(nx), ncy = o3_coarsen(ny), ncz = o3_coarsen(nz);
    memset(ci, 0, sizeof(double) * 26 * (size_t)(ncx + 2) * (size_t)(ncy + 2) * (size_t)(ncz + 2));
    for (int phase = 1; phase <= 3; phase++)
        for (int k = 1; k <= nz; k++)
            for (int j = 1; j <= ny; j++)
                for (int i = 1; i <= nx; i++) {
                    int odd[3] = {i & 1, j & 1, k & 1};
                    int m = odd[0] | odd[1] << 1 | odd[2] << 2;
                    if (odd[0] + odd[1] + odd[2] != phase)
                        continue;
                    const double *a = st + 27 * gidx3(nx, ny, i, j, k);
                    /* collapse onto the odd axes: b[e'] over the 27 offsets with even-axis components 0 */
                    double b[27];
                    memset(b, 0, sizeof b);
                    double sig = 0.0;
                    for (int e = 0; e < 27; e++) {
                        int o[3] = {EDX(e), EDY(e), EDZ(e)};
                        for (int d = 0; d < 3; d++)
                            if (!odd[d])
                                o[d] = 0;
                        b[ENT(o[0], o[1], o[2])] += a[e];
                        if (e != CTR)
                            sig -= a[e];
                    }
                    double R = a[CTR] - sig;
                    double eps = INFINITY, sigb = 0.0;
                    for (int d = 0; d < 3; d++) {
                        if (!odd[d])
                            continue;
                        for (int s = -1; s <= 1; s += 2) {
                            double c = 0.0;
                            for (int e = 0; e < 27; e++) {
                                int o[3] = {EDX(e), EDY(e), EDZ(e)};
                                if (o[d] == s)
                                    c -= b[e];
                            }
                            eps = fmin(eps, fabs(c));
                        }
                    }
                    eps /= a[CTR];
                    for (int e = 0; e < 27; e++)
                        if (e != CTR)
                            sigb -= b[e];
                    double den = sigb + (R > eps * sig ? R : 0.0);
                    if (!(den > 0.0))
                        return O3_EINVAL;
                    int I = odd[0] ? (i + 1) / 2 : i / 2;
                    int J = odd[1] ? (j + 1) / 2 : j / 2;
                    int K = odd[2] ? (k + 1) / 2 : k / 2;
                    double *w = cislot(ncx, ncy, ci, I, J, K) + SLOT[m];
                    int ncorner = 1 << phase;
                    for (int c = 0; c < ncorner; c++) {
                        int C[3] = {I, J, K}, nb = 0;
                        for (int d = 0; d < 3; d++)
                            if (odd[d]) {
                                if (!((c >> nb) & 1))
                                    C[d] -= 1;
                                nb++;
                            }
                        double s = 0.0;
                        for (int e = 0; e < 27; e++) {
                            if (e == CTR)
                                continue;
                            int qi = i + EDX(e), qj = j + EDY(e), qk = k + EDZ(e);
                            s -= b[e] * pw(ncx, ncy, ci, qi, qj, qk, C[0], C[1], C[2]);
                        }
                        w[c] = s / den;
                    }
                }
    return O3_OK;
}

/*
 * c21: the row of P at fine point (i,j,k): up to 8 (coarse point, weight)
 * entries (ghost targets included; callers drop them).
 */
static int prow3(int nx, int ny, const double *ci, int i, int j, int k, int C[][3], double *wt)
{
    int ncx = o3_coarsen(nx), ncy = o3_coarsen(ny);
    int q[3] = {i, j, k}, lo[3], hi[3];
    for (int d = 0; d < 3; d++) {
        if (q[d] & 1) {
            lo[d] = (q[d] + 1) / 2 - 1;
            hi[d] = (q[d] + 1) / 2;
        } else
            lo[d] = hi[d] = q[d] / 2;
    }
    int n = 0;
    for (int K = lo[2]; K <= hi[2]; K++)
        for (int J = lo[1]; J <= hi[1]; J++)
            for (int I = lo[0]; I <= hi[0]; I++) {
                C[n][0] = I;
                C[n][1] = J;
                C[n][2] = K;
                wt[n] = pw(ncx, ncy, ci, i, j, k, I, J, K);
                n++;
            }
    return n;
}

/*
 * c20: Galerkin coarse operator A_c = P^T A P (R = P^T unscaled, c4) over the
 * interior coarse points, by SCATTER: for each interior fine f, each
 * interior stencil neighbour g of f (incl. f), each interior coarse C with
 * P(f,C) and each interior coarse D with P(g,D), accumulate
 * P(f,C) A(f,g) P(g,D) into A_c(C, D-C).  Output: full 27-entry stencil.
 */
int o3_rap(int nx, int ny, int nz, const double *st, const double *ci, double *stc)
{
    int ncx = o3_coarsen(nx), ncy = o3_coarsen(ny), ncz = o3_coarsen(nz);
    memset(stc, 0, sizeof(double) * 27 * (size_t)(ncx + 2) * (size_t)(ncy + 2) * (size_t)(ncz + 2));
    int fC[8][3], gC[8][3];
    double fw[8], gw[8];
    for (int k = 1; k <= nz; k++)
        for (int j = 1; j <= ny; j++)
            for (int i = 1; i <= nx; i++) {
                const double *a = st + 27 * gidx3(nx, ny, i, j, k);
                int nf = prow3(nx, ny, ci, i, j, k, fC, fw);
                for (int e = 0; e < 27; e++) {
                    int gi = i + EDX(e), gj = j + EDY(e), gk = k + EDZ(e);
                    if (!inside(nx, ny, nz, gi, gj, gk))
                        continue;
                    int ng = prow3(nx, ny, ci, gi, gj, gk, gC, gw);
                    for (int x = 0; x < nf; x++) {
                        if (!inside(ncx, ncy, ncz, fC[x][0], fC[x][1], fC[x][2]))
                            continue;
                        for (int y = 0; y < ng; y++) {
                            if (!inside(ncx, ncy, ncz, gC[y][0], gC[y][1], gC[y][2]))
                                continue;
                            int ox = gC[y][0] - fC[x][0], oy = gC[y][1] - fC[x][1], oz = gC[y][2] - fC[x][2];
                            if (ox < -1 || ox > 1 || oy < -1 || oy > 1 || oz < -1 || oz > 1)
                                return O3_EINVAL; /* cannot happen: P has 3x3x3 support */
                            stc[27 * gidx3(ncx, ncy, fC[x][0], fC[x][1], fC[x][2]) + ENT(ox, oy, oz)] +=
                                fw[x] * a[e] * gw[y];
                        }
                    }
                }
            }
    return O3_OK;
}

/* c22: colour of a point: 2 colours ((i+j+k) mod 2) on 7-point levels, 8 ((i mod 2)+2(j mod 2)+4(k mod 2)) on 27-point */
static int colour3(int kind, int i, int j, int k)
{
    return kind == 7 ? ((i + j + k) & 1) : ((i & 1) + 2 * (j & 1) + 4 * (k & 1));
}

/* c22: nsweeps point Gauss-Seidel sweeps, colours in ascending order; u_p = (f_p - sum_{q != p} a_pq u_q)/a_pp */
void o3_relax(int nx, int ny, int nz, int kind, const double *st, const double *f, double *u, int nsweeps)
{
    int ncol = kind == 7 ? 2 : 8;
    for (int s = 0; s < nsweeps; s++)
        for (int c = 0; c < ncol; c++)
            for (int k = 1; k <= nz; k++)
                for (int j = 1; j <= ny; j++)
                    for (int i = 1; i <= nx; i++) {
                        if (colour3(kind, i, j, k) != c)
                            continue;
                        size_t p = gidx3(nx, ny, i, j, k);
                        const double *a = st + 27 * p;
                        double sum = 0.0;
                        for (int e = 0; e < 27; e++)
                            if (e != CTR)
                                sum += a[e] * u[gidx3(nx, ny, i + EDX(e), j + EDY(e), k + EDZ(e))];
                        u[p] = (f[p] - sum) / a[CTR];
                    }
}

/* r = f - A u on the interior (ring 0) */
void o3_residual(int nx, int ny, int nz, const double *st, const double *f, const double *u, double *r)
{
    memset(r, 0, sizeof(double) * (size_t)(nx + 2) * (size_t)(ny + 2) * (size_t)(nz + 2));
    for (int k = 1; k <= nz; k++)
        for (int j = 1; j <= ny; j++)
            for (int i = 1; i <= nx; i++) {
                size_t p = gidx3(nx, ny, i, j, k);
                const double *a = st + 27 * p;
                double sum = 0.0;
                for (int e = 0; e < 27; e++)
                    sum += a[e] * u[gidx3(nx, ny, i + EDX(e), j + EDY(e), k + EDZ(e))];
                r[p] = f[p] - sum;
            }
}

/*
 * c21: restriction q_c(C) = sum over the 27 fine points f = 2C + o of
 * P(f, C) q(f) (R = P^T; fig:restrict_kernel P:165-189 in 3-D), offsets in
 * e order; ghost fine points contribute nothing.
 */
void o3_restrict(int nx, int ny, int nz, const double *ci, const double *q, double *qc)
{
    int ncx = o3_coarsen(nx), ncy = o3_coarsen(ny), ncz = o3_coarsen(nz);
    memset(qc, 0, sizeof(double) * (size_t)(ncx + 2) * (size_t)(ncy + 2) * (size_t)(ncz + 2));
    for (int K = 1; K <= ncz; K++)
        for (int J = 1; J <= ncy; J++)
            for (int I = 1; I <= ncx; I++) {
                double s = 0.0;
                for (int e = 0; e < 27; e++) {
                    int fi = 2 * I + EDX(e), fj = 2 * J + EDY(e), fk = 2 * K + EDZ(e);
                    if (!inside(nx, ny, nz, fi, fj, fk))
                        continue;
                    s += pw(ncx, ncy, ci, fi, fj, fk, I, J, K) * q[gidx3(nx, ny, fi, fj, fk)];
                }
                qc[gidx3(ncx, ncy, I, J, K)] = s;
            }
}

/* c21: u(f) += sum_C P(f,C) e(C) over f's interior coarse corners, corners in z,y,x order */
void o3_interp_add(int nx, int ny, int nz, const double *ci, const double *e, double *u)
{
    int ncx = o3_coarsen(nx), ncy = o3_coarsen(ny), ncz = o3_coarsen(nz);
    int C[8][3];
    double w[8];
    for (int k = 1; k <= nz; k++)
        for (int j = 1; j <= ny; j++)
            for (int i = 1; i <= nx; i++) {
                int n = prow3(nx, ny, ci, i, j, k, C, w);
                double s = 0.0;
                for (int x = 0; x < n; x++)
                    if (inside(ncx, ncy, ncz, C[x][0], C[x][1], C[x][2]))
                        s += w[x] * e[gidx3(ncx, ncy, C[x][0], C[x][1], C[x][2])];
                u[gidx3(nx, ny, i, j, k)] += s;
            }
}

/* c24: dense assembly of a level operator, lexicographic order (x fastest, then y, then z) */
void o3_assemble_dense(int nx, int ny, int nz, const double *st, double *A)
{
    size_t n = (size_t)nx * ny * nz;
    memset(A, 0, sizeof(double) * n * n);
    for (int k = 1; k <= nz; k++)
        for (int j = 1; j <= ny; j++)
            for (int i = 1; i <= nx; i++) {
                const double *a = st + 27 * gidx3(nx, ny, i, j, k);
                size_t p = ((size_t)(k - 1) * ny + (j - 1)) * nx + (i - 1);
                for (int e = 0; e < 27; e++) {
                    int qi = i + EDX(e), qj = j + EDY(e), qk = k + EDZ(e);
                    if (!inside(nx, ny, nz, qi, qj, qk))
                        continue;
                    A[p * n + ((size_t)(qk - 1) * ny + (qj - 1)) * nx + (qi - 1)] = a[e];
                }
            }
}

/* l2 norm over the interior, lexicographic summation */
double o3_norm2(int nx, int ny, int nz, const double *g)
{
    double s = 0.0;
    for (int k = 1; k <= nz; k++)
        for (int j = 1; j <= ny; j++)
            for (int i = 1; i <= nx; i++) {
                double v = g[gidx3(nx, ny, i, j, k)];
                s += v * v;
            }
    return sqrt(s);
}

/* ------------------------------------------------------------------------
 * Hierarchy, plane relaxation (c23), V-cycle (c9 in 3-D), solve
 * ---------------------------------------------------------------------- */
#define O3_MAXLEV 24
typedef struct {
    int nx, ny, nz, kind;
    double *st, *ci, *u, *f, *r;
    void **plane; /* c23: nz 2-D hierarchies (plane k at index k-1), NULL for point relaxation / coarsest */
} o3_level;

typedef struct {
    int L, nu1, nu2, relax;
    o3_level lv[O3_MAXLEV];
    double *chol;
    int nco;
} o3_hier;

void o3_destroy(o3_hier *h)
{
    if (!h)
        return;
    for (int l = 0; l < h->L; l++) {
        o3_level *v = &h->lv[l];
        free(v->st);
        free(v->ci);
        free(v->u);
        free(v->f);
        free(v->r);
        if (v->plane) {
            for (int k = 0; k < v->nz; k++)
                orc_destroy(v->plane[k]);
            free(v->plane);
        }
    }
    free(h->chol);
    free(h);
}

/*
 * c23: the 2-D hierarchy of plane k: the in-plane part (dz = 0 entries) of
 * the level's 27-point row as the 2-D ABI's symmetric-half planes O, W, S, SW,
 * NW (NW = A[p, p+(-1,+1,0)], entry 15), kind 5 on 7-point levels (no in-plane
 * corners) else 9; its cycle is V(1,1) point GS (c6), coarsest 3 (c1).
 */
static int plane_setup(o3_level *v, int k, void **out)
{
    int nx = v->nx, ny = v->ny;
    size_t n2 = (size_t)(nx + 2) * (size_t)(ny + 2);
    double *pl = (double *)calloc(5 * n2, sizeof(double));
    if (!pl)
        return O3_ENOMEM;
    static const int ent[5] = {13, 12, 10, 9, 15}; /* O, W, S, SW, NW in the dz = 0 plane */
    for (int j = 1; j <= ny; j++)
        for (int i = 1; i <= nx; i++) {
            const double *a = v->st + 27 * gidx3(nx, ny, i, j, k);
            for (int q = 0; q < 5; q++)
                pl[q * n2 + (size_t)j * (nx + 2) + i] = a[ent[q]];
        }
    int rc = orc_setup(nx, ny, v->kind == 7 ? 5 : 9, nx + 2, pl, pl + n2, pl + 2 * n2, pl + 3 * n2, pl + 4 * n2,
                       1, 1, 3, 0, 0, 0, out);
    free(pl);
    return rc == 0 ? O3_OK : (rc == O3_ENOTSPD ? O3_ENOTSPD : O3_EINVAL);
}

/*
 * c23: zebra xy-plane Gauss-Seidel, nsweeps sweeps; a sweep visits the planes
 * with k mod 2 = 0, then those with k mod 2 = 1 (colour 0 holds the coarse
 * planes, as c11's lines).  Plane k: g = f_k - sum_{dz = +-1} A u (current
 * values of planes k-1, k+1), then ONE 2-D V(1,1) cycle of the plane's
 * hierarchy on A_kk u_k = g from the current u_k.
 */
static int relax_planes(o3_level *v, int nsweeps)
{
    int nx = v->nx, ny = v->ny, nz = v->nz;
    size_t n2 = (size_t)(nx + 2) * (size_t)(ny + 2);
    double *g = (double *)calloc(n2, sizeof(double));
    double *w = (double *)calloc(n2, sizeof(double));
    if (!g || !w) {
        free(g);
        free(w);
        return O3_ENOMEM;
    }
    for (int s = 0; s < nsweeps; s++)
        for (int c = 0; c < 2; c++)
            for (int k = 1; k <= nz; k++) {
                if ((k & 1) != c)
                    continue;
                for (int j = 1; j <= ny; j++)
                    for (int i = 1; i <= nx; i++) {
                        size_t p = gidx3(nx, ny, i, j, k);
                        const double *a = v->st + 27 * p;
                        double sum = 0.0;
                        for (int e = 0; e < 27; e++)
                            if (EDZ(e) != 0)
                                sum += a[e] * v->u[gidx3(nx, ny, i + EDX(e), j + EDY(e), k + EDZ(e))];
                        g[(size_t)j * (nx + 2) + i] = v->f[p] - sum;
                        w[(size_t)j * (nx + 2) + i] = v->u[p];
                    }
                orc_vcycle(v->plane[k - 1], g, w, 1);
                for (int j = 1; j <= ny; j++)
                    for (int i = 1; i <= nx; i++)
                        v->u[gidx3(nx, ny, i, j, k)] = w[(size_t)j * (nx + 2) + i];
            }
    free(g);
    free(w);
    return O3_OK;
}

/*
 * Setup (c16-c24): expand the fine stencil, then per level l < L-1 the
 * interpolation (c19) and the Galerkin operator (c20); plane hierarchies
 * (c23) on every non-coarsest level when relax = O3_PLANES; the coarsest
 * dense Cholesky factor (c24).  Coarse levels are 27-point.
 */
int o3_setup(int nx, int ny, int nz, int kind, const double *pl, int nu1, int nu2, int coarsest, int max_levels,
             int relax, o3_hier **out)
{
    *out = NULL;
    if (nx < 1 || ny < 1 || nz < 1 || (kind != 7 && kind != 27) || (relax != O3_POINT && relax != O3_PLANES) ||
        nu1 < 0 || nu2 < 0)
        return O3_EINVAL;
    o3_hier *h = (o3_hier *)calloc(1, sizeof(o3_hier));
    if (!h)
        return O3_ENOMEM;
    h->L = o3_count_levels(nx, ny, nz, coarsest, max_levels);
    if (h->L > O3_MAXLEV) {
        free(h);
        return O3_EINVAL;
    }
    h->nu1 = nu1;
    h->nu2 = nu2;
    h->relax = relax;
    int cx = nx, cy = ny, cz = nz;
    for (int l = 0; l < h->L; l++) {
        o3_level *v = &h->lv[l];
        v->nx = cx;
        v->ny = cy;
        v->nz = cz;
        v->kind = l == 0 ? kind : 27;
        size_t np = (size_t)(cx + 2) * (size_t)(cy + 2) * (size_t)(cz + 2);
        v->st = (double *)calloc(27 * np, sizeof(double));
        v->u = (double *)calloc(np, sizeof(double));
        v->f = (double *)calloc(np, sizeof(double));
        v->r = (double *)calloc(np, sizeof(double));
        if (l + 1 < h->L)
            v->ci = (double *)calloc(26 * (size_t)(cx / 2 + 2) * (size_t)(cy / 2 + 2) * (size_t)(cz / 2 + 2),
                                     sizeof(double));
        if (!v->st || !v->u || !v->f || !v->r || (l + 1 < h->L && !v->ci)) {
            o3_destroy(h);
            return O3_ENOMEM;
        }
        cx /= 2;
        cy /= 2;
        cz /= 2;
    }
    int rc = o3_expand_stencil(nx, ny, nz, kind, pl, h->lv[0].st);
    for (int l = 0; rc == O3_OK && l + 1 < h->L; l++) {
        o3_level *v = &h->lv[l];
        rc = o3_setup_interp(v->nx, v->ny, v->nz, v->st, v->ci);
        if (rc == O3_OK)
            rc = o3_rap(v->nx, v->ny, v->nz, v->st, v->ci, h->lv[l + 1].st);
    }
    for (int l = 0; rc == O3_OK && relax == O3_PLANES && l + 1 < h->L; l++) {
        o3_level *v = &h->lv[l];
        v->plane = (void **)calloc((size_t)v->nz, sizeof(void *));
        if (!v->plane)
            rc = O3_ENOMEM;
        for (int k = 1; rc == O3_OK && k <= v->nz; k++)
            rc = plane_setup(v, k, &v->plane[k - 1]);
    }
    if (rc == O3_OK) {
        o3_level *c = &h->lv[h->L - 1];
        h->nco = c->nx * c->ny * c->nz;
        h->chol = (double *)malloc(sizeof(double) * (size_t)h->nco * (size_t)h->nco);
        if (!h->chol)
            rc = O3_ENOMEM;
        else {
            o3_assemble_dense(c->nx, c->ny, c->nz, c->st, h->chol);
            rc = orc_chol_factor(h->nco, h->chol) == 0 ? O3_OK : O3_ENOTSPD;
        }
    }
    if (rc != O3_OK) {
        o3_destroy(h);
        return rc;
    }
    *out = h;
    return O3_OK;
}

int o3_num_levels(const o3_hier *h) { return h->L; }

void o3_level_shape(const o3_hier *h, int l, int *nx, int *ny, int *nz, int *kind)
{
    *nx = h->lv[l].nx;
    *ny = h->lv[l].ny;
    *nz = h->lv[l].nz;
    *kind = h->lv[l].kind;
}

/* copy out level l's full stencil (27 per point) and CI (26 per coarse index; may be NULL) */
void o3_export_level(const o3_hier *h, int l, double *st, double *ci)
{
    const o3_level *v = &h->lv[l];
    memcpy(st, v->st, sizeof(double) * 27 * (size_t)(v->nx + 2) * (size_t)(v->ny + 2) * (size_t)(v->nz + 2));
    if (ci && v->ci)
        memcpy(ci, v->ci,
               sizeof(double) * 26 * (size_t)(v->nx / 2 + 2) * (size_t)(v->ny / 2 + 2) * (size_t)(v->nz / 2 + 2));
}

/* relax one level with the hierarchy's mode */
static void relax_level(o3_hier *h, o3_level *v, int nsweeps)
{
    if (h->relax == O3_PLANES)
        relax_planes(v, nsweeps);
    else
        o3_relax(v->nx, v->ny, v->nz, v->kind, v->st, v->f, v->u, nsweeps);
}

/* c24 per cycle: u = A_L^{-1} f on the coarsest level */
static void coarse_solve3(o3_hier *h, o3_level *c)
{
    double *b = (double *)malloc(sizeof(double) * (size_t)h->nco);
    for (int k = 1; k <= c->nz; k++)
        for (int j = 1; j <= c->ny; j++)
            for (int i = 1; i <= c->nx; i++)
                b[((size_t)(k - 1) * c->ny + (j - 1)) * c->nx + (i - 1)] = c->f[gidx3(c->nx, c->ny, i, j, k)];
    orc_chol_solve(h->nco, h->chol, b);
    for (int k = 1; k <= c->nz; k++)
        for (int j = 1; j <= c->ny; j++)
            for (int i = 1; i <= c->nx; i++)
                c->u[gidx3(c->nx, c->ny, i, j, k)] = b[((size_t)(k - 1) * c->ny + (j - 1)) * c->nx + (i - 1)];
    free(b);
}

/* c9 in 3-D: relax nu1, r = f - A u, f_{l+1} = P^T r, u_{l+1} = 0, recurse, u += P u_{l+1}, relax nu2 */
static void vcycle3_level(o3_hier *h, int l)
{
    o3_level *v = &h->lv[l];
    if (l == h->L - 1) {
        coarse_solve3(h, v);
        return;
    }
    o3_level *c = &h->lv[l + 1];
    relax_level(h, v, h->nu1);
    o3_residual(v->nx, v->ny, v->nz, v->st, v->f, v->u, v->r);
    o3_restrict(v->nx, v->ny, v->nz, v->ci, v->r, c->f);
    memset(c->u, 0, sizeof(double) * (size_t)(c->nx + 2) * (size_t)(c->ny + 2) * (size_t)(c->nz + 2));
    vcycle3_level(h, l + 1);
    o3_interp_add(v->nx, v->ny, v->nz, v->ci, c->u, v->u);
    relax_level(h, v, h->nu2);
}

void o3_vcycle(o3_hier *h, const double *f, double *u, int ncycles)
{
    o3_level *v = &h->lv[0];
    size_t np = (size_t)(v->nx + 2) * (size_t)(v->ny + 2) * (size_t)(v->nz + 2);
    memcpy(v->f, f, sizeof(double) * np);
    memcpy(v->u, u, sizeof(double) * np);
    for (int c = 0; c < ncycles; c++)
        vcycle3_level(h, 0);
    memcpy(u, v->u, sizeof(double) * np);
}

/* the hierarchy's relaxation on the fine level alone (tests) */
void o3_relax_level(o3_hier *h, const double *f, double *u, int nsweeps)
{
    o3_level *v = &h->lv[0];
    size_t np = (size_t)(v->nx + 2) * (size_t)(v->ny + 2) * (size_t)(v->nz + 2);
    memcpy(v->f, f, sizeof(double) * np);
    memcpy(v->u, u, sizeof(double) * np);
    relax_level(h, v, nsweeps);
    memcpy(u, v->u, sizeof(double) * np);
}

double o3_residual_norm(o3_hier *h, const double *f, const double *u)
{
    o3_level *v = &h->lv[0];
    o3_residual(v->nx, v->ny, v->nz, v->st, f, u, v->r);
    return o3_norm2(v->nx, v->ny, v->nz, v->r);
}

/* solve loop (SPEC S:438-446 in 3-D): hist[0] = ||f - A x0||; cycle until ||r|| <= tol ||f|| or maxiter */
int o3_solve(o3_hier *h, const double *f, double *u, double tol, int maxiter, int *iters, double *hist)
{
    o3_level *v = &h->lv[0];
    size_t np = (size_t)(v->nx + 2) * (size_t)(v->ny + 2) * (size_t)(v->nz + 2);
    double fn = o3_norm2(v->nx, v->ny, v->nz, f);
    *iters = 0;
    if (fn == 0.0) {
        memset(u, 0, sizeof(double) * np);
        if (hist)
            hist[0] = 0.0;
        return O3_OK;
    }
    double rn = o3_residual_norm(h, f, u);
    if (hist)
        hist[0] = rn;
    int k = 0;
    while (rn > tol * fn && k < maxiter) {
        o3_vcycle(h, f, u, 1);
        k++;
        rn = o3_residual_norm(h, f, u);
        if (hist)
            hist[k] = rn;
    }
    *iters = k;
    return rn <= tol * fn ? O3_OK : O3_ENOTCONV;
}
