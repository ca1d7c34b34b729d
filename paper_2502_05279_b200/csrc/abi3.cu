// abi3.cu -- the bmg3_* entry points (include/bmg3.h): 3-D hierarchy setup,
// the V-cycle with point or zebra-plane relaxation (captured once per (rhs, x)
// as a CUDA graph), the solve loop and the test helpers.  DESIGN.md §5.8.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <map>
#include <string>
#include <utility>
#include <vector>

#include "bmg3.h"
#include "bmg3.cuh"
#include "solver.cuh"

using namespace bmg3;

namespace {

constexpr int MAX_DENSE = 4096;  // coarsest 3-D level / coarsest plane level: dense Cholesky limit

// one 2-D level of the batched plane hierarchies of a 3-D level (c23)
struct PLevel {
    Grid3 g;
    int kind = 9;
    double *pl[5] = {};  // O W S SW SE (m >= 1; level 0 views the 3-D stencil)
    double *u = nullptr, *f = nullptr, *r = nullptr;
    double *ci[8] = {};  // weights to the next plane level (its grid)
    double *chol = nullptr;  // coarsest plane level: nz dense factors
    OpP op() const
    {
        OpP A;
        A.g = g;
        A.kind = kind;
        A.O = pl[0];
        A.W = pl[1];
        A.S = pl[2];
        A.SW = pl[3];
        A.SE = pl[4];
        return A;
    }
    CIP cip(const Grid3 &cg) const
    {
        CIP c;
        c.c = cg;
        for (int q = 0; q < 8; q++)
            c.w[q] = ci[q];
        return c;
    }
};

struct Level3 {
    Grid3 g;
    int kind = 27;
    double *pl[14] = {};  // O, then the 13 lower entries (nullptr where a 7-point level has none)
    double *u = nullptr, *f = nullptr, *r = nullptr;
    double *ci[26] = {};  // weights from level l+1 (its grid)
    std::vector<PLevel> pv;  // plane hierarchy (relax = planes, non-coarsest levels)
    double *pr = nullptr;    // plane level-0 residual scratch (3-D sized)
    double *pt = nullptr;    // 5-point plane level 0: the one-pass sweep's second buffer (3-D sized)
    int ptail = 1 << 30;     // first plane level run by the plane tail (kernels_plane.cu)
    double *rc27 = nullptr;  // 27-point point relaxation: colour-major full rows (kernels3.cu)
    double *tmp = nullptr;   // 7-point point relaxation: the second buffer of the one-pass sweep (k3_rb7)
    double *ro = nullptr;    // and its reciprocal plane rcp_pos(a_O)
    Op3 op() const
    {
        Op3 A;
        A.g = g;
        A.kind = kind;
        A.O = pl[0];
        for (int e = 0; e < 13; e++)
            A.a[e] = pl[1 + e];
        return A;
    }
};

Grid3 mkgrid(int nx, int ny, int nz)
{
    Grid3 g;
    g.nx = nx;
    g.ny = ny;
    g.nz = nz;
    g.px = ((long long)nx + 2 + 7) / 8 * 8;
    g.ps = g.px * (ny + 2);
    return g;
}

size_t gsize(const Grid3 &g) { return (size_t)g.ps * (size_t)(g.nz + 2) + 8; }

}  // namespace

struct bmg3_solver {
    bmg3_params_t prm;
    int L = 0;
    std::vector<Level3> lv;
    std::vector<void *> allocs;
    char *chunk = nullptr;  // bump allocator (alloc): current chunk, the bytes left in it,
    size_t chunk_left = 0;  // the size of the next chunk (64 MB, doubling up to 1 GB)
    size_t chunk_next = (size_t)64 << 20;
    double *chol = nullptr;
    int nco = 0;
    int *d_err = nullptr;
    double *partials = nullptr, *d_norm = nullptr, *h_norm = nullptr;
    cudaStream_t cap = nullptr;
    std::map<std::pair<const void *, const void *>, cudaGraphExec_t> graphs;
    int kernels_per_cycle = 0;
};

namespace {

// Level arrays come from a bump allocator over large chunks (64 MB doubling up to 1 GB, or
// one per larger array; 256-byte aligned pieces): the plane hierarchies alone ask for ~16
// arrays per plane level and 3-D level, and a cudaMalloc each cost ~0.5 s of a 255^3
// setup.  Every piece is zeroed, as before.
bmg_status_t alloc(bmg3_solver *h, size_t ndouble, double **p, cudaStream_t s)
{
    const size_t bytes = (ndouble * sizeof(double) + 255) / 256 * 256;
    if (bytes > h->chunk_left) {
        const size_t cb = bytes > h->chunk_next ? bytes : h->chunk_next;
        if (h->chunk_next < ((size_t)1 << 30))
            h->chunk_next *= 2;
        void *q = nullptr;
        CK(cudaMalloc(&q, cb));
        h->allocs.push_back(q);
        h->chunk = (char *)q;
        h->chunk_left = cb;
    }
    void *q = h->chunk;
    h->chunk += bytes;
    h->chunk_left -= bytes;
    CK(cudaMemsetAsync(q, 0, ndouble * sizeof(double), s));
    *p = (double *)q;
    return BMG_OK;
}

bmg_status_t check_err(bmg3_solver *h, cudaStream_t s, const char *where)
{
    int e = 0;
    CK(cudaMemcpyAsync(&e, h->d_err, sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (e & bmg::ERR_PIVOT)
        return bmg::fail(BMG_ENOTSPD, std::string(where) + ": Cholesky pivot <= 0");
    if (e & bmg::ERR_DIAG)
        return bmg::fail(BMG_EINVAL, std::string(where) + ": a_O <= 0 at an interior point");
    if (e & bmg::ERR_DEN)
        return bmg::fail(BMG_EINVAL, std::string(where) + ": interpolation denominator <= 0");
    return BMG_OK;
}

CI3 ci_view(const Level3 &f, const Level3 &c)
{
    CI3 v;
    v.c = c.g;
    for (int q = 0; q < 26; q++)
        v.w[q] = f.ci[q];
    return v;
}

// c23: the batched 2-D hierarchies of level v's planes
bmg_status_t plane_setup(bmg3_solver *h, Level3 &v, cudaStream_t s)
{
    v.pv.clear();
    int nx = v.g.nx, ny = v.g.ny;
    {
        PLevel p0;
        p0.g = v.g;
        p0.kind = v.kind == 7 ? 5 : 9;
        p0.pl[0] = v.pl[0];
        p0.pl[1] = v.pl[1 + 12];
        p0.pl[2] = v.pl[1 + 10];
        p0.pl[3] = v.pl[1 + 9];
        p0.pl[4] = v.pl[1 + 11];
        v.pv.push_back(p0);
    }
    while ((nx < ny ? nx : ny) > 3) {
        nx /= 2;
        ny /= 2;
        PLevel q;
        q.g = mkgrid(nx, ny, v.g.nz);
        q.kind = 9;
        for (int t = 0; t < 5; t++)
            TRY(alloc(h, gsize(q.g), &q.pl[t], s));
        TRY(alloc(h, gsize(q.g), &q.u, s));
        TRY(alloc(h, gsize(q.g), &q.f, s));
        TRY(alloc(h, gsize(q.g), &q.r, s));
        v.pv.push_back(q);
    }
    const int M = (int)v.pv.size();
    if (M > 1)
        TRY(alloc(h, gsize(v.g), &v.pr, s));
    if (M > 1 && v.pv[0].kind == 5)
        TRY(alloc(h, gsize(v.g), &v.pt, s));
    for (int m = 0; m + 1 < M; m++) {
        PLevel &a = v.pv[m], &c = v.pv[m + 1];
        for (int q = 0; q < 8; q++)
            TRY(alloc(h, gsize(c.g), &a.ci[q], s));
        launchP_interp(a.op(), a.ci, c.g, h->d_err, s);
        TRY(check_err(h, s, "bmg3_setup (plane interpolation)"));
        launchP_rap(a.op(), a.cip(c.g), c.pl, s);
    }
    long long ptmax = PTAIL_MAX;  // tuning knob BMG3_PTAIL_MAX (default measured)
    if (const char *e = getenv("BMG3_PTAIL_MAX"))
        ptmax = atoll(e);
    for (int m = 0; m < M; m++)
        if ((long long)v.pv[m].g.nx * v.pv[m].g.ny <= ptmax && getenv("BMG3_NO_PTAIL") == nullptr) {
            v.ptail = m;
            break;
        }
    PLevel &cl = v.pv[M - 1];
    const long long n = (long long)cl.g.nx * cl.g.ny;
    if (n > MAX_DENSE)
        return bmg::fail(BMG_EINVAL, "bmg3_setup: coarsest plane level has " + std::to_string(n) +
                                         " unknowns (> 4096; planes must coarsen to min(nx,ny) <= 3 within the limit)");
    TRY(alloc(h, (size_t)n * n * v.g.nz, &cl.chol, s));
    launchP_assemble_chol(cl.op(), cl.chol, h->d_err, s);
    TRY(check_err(h, s, "bmg3_setup (plane Cholesky)"));
    return BMG_OK;
}

// the plane tail from plane level m (u, f: that level's iterate and right-hand side)
void plane_tail(Level3 &v, int m, double *u, const double *f, Batch b, cudaStream_t s)
{
    PTail T;
    T.nlev = (int)v.pv.size() - m;
    for (int t = 0; t < T.nlev; t++) {
        PLevel &a = v.pv[m + t];
        T.lv[t].op = a.op();
        if (m + t + 1 < (int)v.pv.size())
            T.lv[t].ci = a.cip(v.pv[m + t + 1].g);
        T.lv[t].u = t == 0 ? u : a.u;
        T.lv[t].f = t == 0 ? const_cast<double *>(f) : a.f;
        T.lv[t].r = (m + t == 0) ? v.pr : a.r;
    }
    T.chol = v.pv.back().chol;
    launchP_tail(T, b, s);
}

// one 2-D V(1,1) cycle (c23, c9 on the plane hierarchy) on the planes of batch b
void plane_vcycle(Level3 &v, int m, double *u, const double *f, Batch b, cudaStream_t s)
{
    PLevel &a = v.pv[m];
    const OpP A = a.op();
    if (m >= v.ptail && (int)v.pv.size() - m <= PTAIL_LEVELS) {
        plane_tail(v, m, u, f, b, s);
        return;
    }
    if (m + 1 == (int)v.pv.size()) {
        launchP_coarse_solve(A, a.chol, f, u, b, s);
        return;
    }
    PLevel &c = v.pv[m + 1];
    double *r = m == 0 ? v.pr : a.r;
    if (m == 0 && v.pt) {  // 5-point plane level: one-pass sweeps u -> pt, (correct pt,) pt -> u
        launchP_rb5(A, f, u, v.pt, b, s);
        launchP_residual(A, f, v.pt, r, b, s);
        launchP_restrict(A, a.cip(c.g), r, c.f, c.u, b, s);
        plane_vcycle(v, m + 1, c.u, c.f, b, s);
        launchP_interp_add(a.g, a.cip(c.g), c.u, v.pt, b, s);
        launchP_rb5(A, f, v.pt, u, b, s);
        return;
    }
    launchP_relax(A, f, u, b, s);
    launchP_residual(A, f, u, r, b, s);
    launchP_restrict(A, a.cip(c.g), r, c.f, c.u, b, s);
    plane_vcycle(v, m + 1, c.u, c.f, b, s);
    launchP_interp_add(a.g, a.cip(c.g), c.u, u, b, s);
    launchP_relax(A, f, u, b, s);
}

// c23: nsweeps zebra xy-plane sweeps (planes k mod 2 = 0, then 1); the level's r is the plane rhs g
void relax_planes(Level3 &v, const double *f, double *u, int nsweeps, cudaStream_t s)
{
    const Op3 A = v.op();
    for (int sw = 0; sw < nsweeps; sw++)
        for (int c = 0; c < 2; c++) {
            Batch b;
            b.k0 = c == 0 ? 2 : 1;
            b.nb = c == 0 ? v.g.nz / 2 : (v.g.nz + 1) / 2;
            if (b.nb == 0)
                continue;
            launch3_plane_rhs(A, f, u, v.r, b, s);
            plane_vcycle(v, 0, u, v.r, b, s);
        }
}

// 7-point point relaxation, nsweeps one-pass sweeps alternating between u and v.tmp,
// starting from the iterate in `from`; returns where the result is
double *rb7_sweeps(Level3 &v, const double *f, double *from, double *u, int nsweeps, cudaStream_t s)
{
    double *a = from, *b = from == u ? v.tmp : u;
    for (int sw = 0; sw < nsweeps; sw++) {
        launch3_rb7(v.op(), f, a, b, s, v.ro);
        std::swap(a, b);
    }
    return a;
}

void relax_level(bmg3_solver *h, Level3 &v, const double *f, double *u, int nsweeps, cudaStream_t s)
{
    if (v.tmp) {
        double *end = rb7_sweeps(v, f, u, u, nsweeps, s);
        if (end != u)
            cudaMemcpyAsync(u, end, gsize(v.g) * sizeof(double), cudaMemcpyDeviceToDevice, s);
        return;
    }
    if (h->prm.relax == BMG3_RELAX_PLANES)
        relax_planes(v, f, u, nsweeps, s);
    else if (v.rc27)
        launch3_relax27c(v.g, v.rc27, f, u, nsweeps, s);
    else
        launch3_relax_point(v.op(), f, u, nsweeps, s, nullptr);
}

// c9 in 3-D
void enqueue_cycle(bmg3_solver *h, const double *rhs, double *x, cudaStream_t s)
{
    const int L = h->L;
    auto F = [&](int l) -> const double * { return l == 0 ? rhs : h->lv[l].f; };
    auto U = [&](int l) -> double * { return l == 0 ? x : h->lv[l].u; };
    // 7-point levels with the one-pass sweep keep the iterate in u or tmp (cur[l]);
    // the up leg's interpolation writes where its nu2 sweeps then end in u
    std::vector<double *> cur(L);
    const int ld = L - 1;
    for (int l = 0; l < ld; l++) {
        Level3 &v = h->lv[l];
        if (v.tmp)
            cur[l] = rb7_sweeps(v, F(l), U(l), U(l), h->prm.nu1, s);
        else {
            relax_level(h, v, F(l), U(l), h->prm.nu1, s);
            cur[l] = U(l);
        }
        launch3_residual(v.op(), F(l), cur[l], v.r, s);
        launch3_restrict(v.op(), ci_view(v, h->lv[l + 1]), v.r, h->lv[l + 1].f, h->lv[l + 1].u, s);
    }
    launch3_coarse_solve(h->lv[L - 1].op(), h->chol, F(L - 1), U(L - 1), s);
    for (int l = ld - 1; l >= 0; l--) {
        Level3 &v = h->lv[l];
        if (v.tmp) {
            double *start = (h->prm.nu2 % 2 == 0) ? U(l) : v.tmp;
            launch3_interp_add(v.g, ci_view(v, h->lv[l + 1]), h->lv[l + 1].u, cur[l], start, s);
            rb7_sweeps(v, F(l), start, U(l), h->prm.nu2, s);
        } else {
            launch3_interp_add(v.g, ci_view(v, h->lv[l + 1]), h->lv[l + 1].u, U(l), U(l), s);
            relax_level(h, v, F(l), U(l), h->prm.nu2, s);
        }
    }
}

bmg_status_t get_graph(bmg3_solver *h, const double *rhs, double *x, cudaGraphExec_t *out)
{
    auto key = std::make_pair((const void *)rhs, (const void *)x);
    auto it = h->graphs.find(key);
    if (it != h->graphs.end()) {
        *out = it->second;
        return BMG_OK;
    }
    cudaGraph_t g = nullptr;
    CK(cudaStreamBeginCapture(h->cap, cudaStreamCaptureModeThreadLocal));
    enqueue_cycle(h, rhs, x, h->cap);
    CK(cudaStreamEndCapture(h->cap, &g));
    cudaGraphExec_t ex = nullptr;
    cudaError_t e = cudaGraphInstantiate(&ex, g, 0);
    size_t nn = 0;
    cudaGraphGetNodes(g, nullptr, &nn);
    std::vector<cudaGraphNode_t> nodes(nn);
    cudaGraphGetNodes(g, nodes.data(), &nn);
    int nk = 0;
    for (auto n : nodes) {
        cudaGraphNodeType t;
        cudaGraphNodeGetType(n, &t);
        nk += t == cudaGraphNodeTypeKernel;
    }
    h->kernels_per_cycle = nk;
    cudaGraphDestroy(g);
    CK(e);
    h->graphs[key] = ex;
    *out = ex;
    return BMG_OK;
}

bmg_status_t resid_norm(bmg3_solver *h, const double *rhs, const double *x, double *out, cudaStream_t s)
{
    const Level3 &v = h->lv[0];
    const Op3 A = v.op();
    launch3_resid_norm(x ? &A : nullptr, v.g, rhs, x, h->partials, h->d_norm, s);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(h->h_norm, h->d_norm, sizeof(double), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    *out = *h->h_norm;
    return BMG_OK;
}

void destroy(bmg3_solver *h)
{
    if (!h)
        return;
    for (auto &kv : h->graphs)
        cudaGraphExecDestroy(kv.second);
    for (void *p : h->allocs)
        cudaFree(p);
    if (h->d_err)
        cudaFree(h->d_err);
    if (h->partials)
        cudaFree(h->partials);
    if (h->d_norm)
        cudaFree(h->d_norm);
    if (h->h_norm)
        cudaFreeHost(h->h_norm);
    if (h->cap)
        cudaStreamDestroy(h->cap);
    delete h;
}

}  // namespace

extern "C" {

void bmg3_params_default(bmg3_params_t *p)
{
    if (!p)
        return;
    p->nu1 = 2;
    p->nu2 = 1;
    p->coarsest = 3;
    p->max_levels = 0;
    p->relax = BMG3_RELAX_POINT;
}

bmg_status_t bmg3_setup(const bmg3_stencil_t *st, const bmg3_params_t *params, void *cuda_stream, bmg3_solver_t *out)
{
    if (!out)
        return bmg::fail(BMG_EINVAL, "bmg3_setup: out is NULL");
    *out = nullptr;
    if (!st)
        return bmg::fail(BMG_EINVAL, "bmg3_setup: stencil is NULL");
    bmg3_params_t prm;
    bmg3_params_default(&prm);
    if (params)
        prm = *params;
    if (st->nx < 1 || st->ny < 1 || st->nz < 1 || (st->kind != 7 && st->kind != 27) || st->pitch < st->nx + 2 ||
        st->plane_stride < st->pitch * (st->ny + 2))
        return bmg::fail(BMG_EINVAL, "bmg3_setup: bad sizes, kind, pitch or plane_stride");
    if (prm.nu1 < 0 || prm.nu2 < 0 || prm.coarsest < 1 ||
        (prm.relax != BMG3_RELAX_POINT && prm.relax != BMG3_RELAX_PLANES))
        return bmg::fail(BMG_EINVAL, "bmg3_setup: bad params");
    const int np = st->kind == 7 ? 4 : 14;
    for (int q = 0; q < np; q++)
        if (!st->plane[q])
            return bmg::fail(BMG_EINVAL, "bmg3_setup: NULL stencil plane");
    cudaStream_t s = (cudaStream_t)cuda_stream;
    bmg3_solver *h = new bmg3_solver();
    h->prm = prm;
    auto bail = [&](bmg_status_t rc) {
        cudaStreamSynchronize(s);
        destroy(h);
        return rc;
    };
#define TRYH(x)                   \
    do {                          \
        bmg_status_t r_ = (x);    \
        if (r_ != BMG_OK)         \
            return bail(r_);      \
    } while (0)
#define CKH(call)                                                                                       \
    do {                                                                                                \
        cudaError_t e_ = (call);                                                                        \
        if (e_ != cudaSuccess)                                                                          \
            return bail(bmg::fail(e_ == cudaErrorMemoryAllocation ? BMG_ENOMEM : BMG_ECUDA,             \
                                  std::string(#call) + ": " + cudaGetErrorString(e_)));                 \
    } while (0)
    CKH(cudaStreamCreateWithFlags(&h->cap, cudaStreamNonBlocking));
    CKH(cudaMalloc(&h->d_err, sizeof(int)));
    CKH(cudaMemsetAsync(h->d_err, 0, sizeof(int), s));
    // c17 ladder
    int nx = st->nx, ny = st->ny, nz = st->nz;
    for (int l = 0;; l++) {
        Level3 v;
        v.g = l == 0 ? Grid3{nx, ny, nz, st->pitch, st->plane_stride} : mkgrid(nx, ny, nz);
        v.kind = l == 0 ? st->kind : 27;
        h->lv.push_back(v);
        const int m = std::min(nx, std::min(ny, nz));
        if (!(m > prm.coarsest) || (prm.max_levels > 0 && (int)h->lv.size() >= prm.max_levels) || h->lv.size() >= 24)
            break;
        nx /= 2;
        ny /= 2;
        nz /= 2;
    }
    h->L = (int)h->lv.size();
    for (int l = 0; l < h->L; l++) {
        Level3 &v = h->lv[l];
        const size_t n = gsize(v.g);
        for (int q = 0; q < 14; q++) {
            const bool need = v.kind == 27 || q == 0 || q == 1 + 12 || q == 1 + 10 || q == 1 + 4;
            if (need)
                TRYH(alloc(h, n, &v.pl[q], s));
        }
        if (l > 0) {
            TRYH(alloc(h, n, &v.u, s));
            TRYH(alloc(h, n, &v.f, s));
        }
        if (l + 1 < h->L) {
            TRYH(alloc(h, n, &v.r, s));
        }
    }
    for (int l = 0; l + 1 < h->L; l++)
        for (int q = 0; q < 26; q++)
            TRYH(alloc(h, gsize(h->lv[l + 1].g), &h->lv[l].ci[q], s));
    // S0 ingest
    {
        const double *src[14] = {};
        src[0] = st->plane[0];
        if (st->kind == 7) {
            src[1 + 12] = st->plane[1];
            src[1 + 10] = st->plane[2];
            src[1 + 4] = st->plane[3];
        } else {
            for (int e = 0; e < 13; e++)
                src[1 + e] = st->plane[1 + e];
        }
        launch3_ingest(st->kind, h->lv[0].g, src, h->lv[0].pl, h->d_err, s);
        CKH(cudaGetLastError());
        TRYH(check_err(h, s, "bmg3_setup (ingest)"));
    }
    // S1 + S2 per level
    for (int l = 0; l + 1 < h->L; l++) {
        Level3 &v = h->lv[l], &c = h->lv[l + 1];
        launch3_interp(v.op(), v.ci, c.g, h->d_err, s);
        CKH(cudaGetLastError());
        TRYH(check_err(h, s, "bmg3_setup (interpolation)"));
        launch3_rap(v.op(), ci_view(v, c), c.pl, h->d_err, s);
        CKH(cudaGetLastError());
    }
    // the one-pass 7-point sweep's second buffer (relaxed 7-point levels)
    if (prm.relax == BMG3_RELAX_POINT)
        for (int l = 0; l + 1 < h->L; l++)
            if (h->lv[l].kind == 7) {
                TRYH(alloc(h, gsize(h->lv[l].g), &h->lv[l].tmp, s));
                TRYH(alloc(h, gsize(h->lv[l].g), &h->lv[l].ro, s));
                launch3_recip(h->lv[l].op(), h->lv[l].ro, s);
            }
    // colour-major rows for the 27-point point smoother (relaxed levels only)
    if (prm.relax == BMG3_RELAX_POINT)
        for (int l = 0; l + 1 < h->L; l++) {
            Level3 &v = h->lv[l];
            if (v.kind != 27)
                continue;
            TRYH(alloc(h, (size_t)relax27_doubles(v.g), &v.rc27, s));
            launch3_build_relax27(v.op(), v.rc27, s);
            CKH(cudaGetLastError());
        }
    // plane hierarchies
    if (prm.relax == BMG3_RELAX_PLANES)
        for (int l = 0; l + 1 < h->L; l++) {
            TRYH(plane_setup(h, h->lv[l], s));
            CKH(cudaGetLastError());
        }
    // S3 coarsest factor
    {
        Level3 &c = h->lv[h->L - 1];
        const long long n = (long long)c.g.nx * c.g.ny * c.g.nz;
        if (n > MAX_DENSE)
            return bail(bmg::fail(BMG_EINVAL, "bmg3_setup: coarsest level has " + std::to_string(n) +
                                                  " unknowns (> 4096)"));
        h->nco = (int)n;
        TRYH(alloc(h, (size_t)n * n, &h->chol, s));
        launch3_assemble_dense(c.op(), h->chol, s);
        bmg::launch_chol_factor((int)n, h->chol, h->d_err, s);
        CKH(cudaGetLastError());
        TRYH(check_err(h, s, "bmg3_setup (coarsest Cholesky)"));
    }
    const int nbp = norm3_partials(h->lv[0].g);
    CKH(cudaMalloc(&h->partials, sizeof(double) * nbp));
    CKH(cudaMalloc(&h->d_norm, sizeof(double)));
    CKH(cudaMallocHost(&h->h_norm, sizeof(double)));
    CKH(cudaStreamSynchronize(s));
#undef TRYH
#undef CKH
    *out = h;
    return BMG_OK;
}

bmg_status_t bmg3_vcycle(bmg3_solver_t h, const double *rhs, double *x, int ncycles, void *cuda_stream)
{
    if (!h || !rhs || !x || ncycles < 0 || (const void *)rhs == (const void *)x)
        return bmg::fail(BMG_EINVAL, "bmg3_vcycle: bad arguments");
    if (ncycles == 0)
        return BMG_OK;
    cudaGraphExec_t ex;
    TRY(get_graph(h, rhs, x, &ex));
    for (int c = 0; c < ncycles; c++)
        CK(cudaGraphLaunch(ex, (cudaStream_t)cuda_stream));
    return BMG_OK;
}

bmg_status_t bmg3_residual_norm(bmg3_solver_t h, const double *rhs, const double *x, double *norm_host,
                                void *cuda_stream)
{
    if (!h || !rhs || !x || !norm_host)
        return bmg::fail(BMG_EINVAL, "bmg3_residual_norm: bad arguments");
    return resid_norm(h, rhs, x, norm_host, (cudaStream_t)cuda_stream);
}

bmg_status_t bmg3_solve(bmg3_solver_t h, const double *rhs, double *x, double tol, int maxiter, int *iters_out,
                        double *hist_host, void *cuda_stream)
{
    if (!h || !rhs || !x || maxiter < 0 || !(tol >= 0.0))
        return bmg::fail(BMG_EINVAL, "bmg3_solve: bad arguments");
    cudaStream_t s = (cudaStream_t)cuda_stream;
    double fn = 0.0, rn = 0.0;
    TRY(resid_norm(h, rhs, nullptr, &fn, s));
    if (iters_out)
        *iters_out = 0;
    if (fn == 0.0) {
        launch3_zero_interior(h->lv[0].g, x, s);
        CK(cudaGetLastError());
        CK(cudaStreamSynchronize(s));
        if (hist_host)
            hist_host[0] = 0.0;
        return BMG_OK;
    }
    TRY(resid_norm(h, rhs, x, &rn, s));
    if (hist_host)
        hist_host[0] = rn;
    int k = 0;
    while (rn > tol * fn && k < maxiter) {
        TRY(bmg3_vcycle(h, rhs, x, 1, cuda_stream));
        k++;
        TRY(resid_norm(h, rhs, x, &rn, s));
        if (hist_host)
            hist_host[k] = rn;
    }
    if (iters_out)
        *iters_out = k;
    return rn <= tol * fn ? BMG_OK : bmg::fail(BMG_ENOTCONV, "bmg3_solve: maxiter reached");
}

bmg_status_t bmg3_relax(bmg3_solver_t h, const double *rhs, double *x, int nsweeps, void *cuda_stream)
{
    if (!h || !rhs || !x || nsweeps < 0)
        return bmg::fail(BMG_EINVAL, "bmg3_relax: bad arguments");
    if (h->prm.relax == BMG3_RELAX_PLANES && h->lv[0].pv.empty())
        return bmg::fail(BMG_EINVAL, "bmg3_relax: the fine level is the coarsest (no plane hierarchy)");
    relax_level(h, h->lv[0], rhs, x, nsweeps, (cudaStream_t)cuda_stream);
    CK(cudaGetLastError());
    return BMG_OK;
}

bmg_status_t bmg3_num_levels(bmg3_solver_t h, int *L)
{
    if (!h || !L)
        return bmg::fail(BMG_EINVAL, "bmg3_num_levels: bad arguments");
    *L = h->L;
    return BMG_OK;
}

bmg_status_t bmg3_level_shape(bmg3_solver_t h, int level, int *nx, int *ny, int *nz, int *kind)
{
    if (!h || level < 0 || level >= h->L)
        return bmg::fail(BMG_EINVAL, "bmg3_level_shape: bad arguments");
    const Level3 &v = h->lv[level];
    if (nx)
        *nx = v.g.nx;
    if (ny)
        *ny = v.g.ny;
    if (nz)
        *nz = v.g.nz;
    if (kind)
        *kind = v.kind;
    return BMG_OK;
}

bmg_status_t bmg3_cycle_kernel_count(bmg3_solver_t h, int *count)
{
    if (!h || !count)
        return bmg::fail(BMG_EINVAL, "bmg3_cycle_kernel_count: bad arguments");
    if (h->kernels_per_cycle == 0) {
        // dry capture on two scratch arrays of the fine level's size
        const Level3 &v = h->lv[0];
        double *a = nullptr, *b = nullptr;
        CK(cudaMalloc(&a, gsize(v.g) * sizeof(double)));
        cudaError_t e = cudaMalloc(&b, gsize(v.g) * sizeof(double));
        if (e != cudaSuccess) {
            cudaFree(a);
            CK(e);
        }
        cudaGraphExec_t ex;
        bmg_status_t rc = get_graph(h, a, b, &ex);
        h->graphs.erase(std::make_pair((const void *)a, (const void *)b));
        if (rc == BMG_OK)
            cudaGraphExecDestroy(ex);
        cudaFree(a);
        cudaFree(b);
        TRY(rc);
    }
    *count = h->kernels_per_cycle;
    return BMG_OK;
}

bmg_status_t bmg3_export_level(bmg3_solver_t h, int level, double *stencil_host, double *ci_host)
{
    if (!h || level < 0 || level >= h->L || !stencil_host)
        return bmg::fail(BMG_EINVAL, "bmg3_export_level: bad arguments");
    const Level3 &v = h->lv[level];
    const Grid3 &g = v.g;
    const size_t nc = (size_t)(g.nx + 2) * (g.ny + 2) * (g.nz + 2);
    std::vector<double> tmp(gsize(g));
    auto repack = [&](const Grid3 &gg, const double *src, double *dst) -> bmg_status_t {
        std::vector<double> t(gsize(gg));
        CK(cudaMemcpy(t.data(), src, t.size() * sizeof(double), cudaMemcpyDeviceToHost));
        for (int k = 0; k < gg.nz + 2; k++)
            for (int j = 0; j < gg.ny + 2; j++)
                for (int i = 0; i < gg.nx + 2; i++)
                    dst[((size_t)k * (gg.ny + 2) + j) * (gg.nx + 2) + i] = t[(size_t)at3(gg, i, j, k)];
        return BMG_OK;
    };
    CK(cudaDeviceSynchronize());
    for (int q = 0; q < 14; q++) {
        if (v.pl[q])
            TRY(repack(g, v.pl[q], stencil_host + q * nc));
        else
            std::fill(stencil_host + q * nc, stencil_host + (q + 1) * nc, 0.0);
    }
    if (ci_host && level + 1 < h->L) {
        const Grid3 &cg = h->lv[level + 1].g;
        const size_t ncc = (size_t)(cg.nx + 2) * (cg.ny + 2) * (cg.nz + 2);
        for (int q = 0; q < 26; q++)
            TRY(repack(cg, v.ci[q], ci_host + q * ncc));
    }
    return BMG_OK;
}

bmg_status_t bmg3_destroy(bmg3_solver_t h)
{
    destroy(h);
    return BMG_OK;
}

}  // extern "C"
