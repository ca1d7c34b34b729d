// abi.cu -- the extern "C" boundary of libbmg.so (include/bmg.h): hierarchy
// construction (setup), CUDA-graph-captured V-cycles, the solve loop, PCG and
// the single-step entry points used by the parity tests (the c15 block
// multi-RHS entry points are in abi_block.cu; the handle is in solver.cuh).
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <chrono>
#include <mutex>
#include <map>
#include <string>
#include <utility>
#include <vector>

#include "solver.cuh"

namespace {

long long round_pitch(int nx) { return ((long long)nx + 2 + 31) / 32 * 32; }

// Levels with at most this many unknowns (and all coarser ones) run in the
// single-CTA tail kernel in fused mode.
// 1024: swept 256 .. 65536 with the 512-thread tail (8191^2 2.986 -> 2.970 ms,
// 1023^2 0.233 -> 0.219 ms, 63^2 cycle 0.060 -> 0.056 ms against 4096)
constexpr long long TAIL_POINTS = 1024;
// levels above the tail with at most this many unknowns run the tile legs (kernels_tile.cu);
// BMG_TILE_POINTS overrides (0: none)
constexpr long long TILE_POINTS = 70000;  // swept 0 .. 1.1e6 (tools/tile_sweep.py): 255^2 and below

}  // namespace

std::string &bmg::abi_detail()
{
    thread_local std::string d;
    return d;
}

// Pinned host slots (8 doubles) for the norms read back by the host: one
// cudaMallocHost per 512 handles instead of one per handle (each costs ~ms).
static std::mutex g_pin_mu;
static std::vector<double *> g_pin_free;
double *pinned_slot()
{
    std::lock_guard<std::mutex> lk(g_pin_mu);
    if (g_pin_free.empty()) {
        double *blk = nullptr;
        if (cudaMallocHost(&blk, 512 * 8 * sizeof(double)) != cudaSuccess)
            return nullptr;  // the block lives for the process
        for (int i = 511; i >= 0; i--)
            g_pin_free.push_back(blk + 8 * i);
    }
    double *p = g_pin_free.back();
    g_pin_free.pop_back();
    return p;
}
void pinned_release(double *p)
{
    std::lock_guard<std::mutex> lk(g_pin_mu);
    g_pin_free.push_back(p);
}

extern "C" {

void bmg_params_default(bmg_params_t *p)
{
    p->nu1 = 2;
    p->nu2 = 1;
    p->coarsest = 3;
    p->max_levels = 0;
    p->agglom_rows = 128;
    p->cycle_sym = 0;
    p->fused = 1;
    p->relax = BMG_RELAX_POINT;
    p->affine = 0;
}

const char *bmg_strerror(bmg_status_t s)
{
    switch (s) {
    case BMG_OK: return "ok";
    case BMG_EINVAL: return "invalid argument or operator";
    case BMG_ENOMEM: return "out of device memory";
    case BMG_ECUDA: return "CUDA error";
    case BMG_ENCCL: return "NCCL error";
    case BMG_ENOTSPD: return "coarsest operator not SPD (Cholesky pivot <= 0)";
    case BMG_ENOTCONV: return "not converged within maxiter";
    }
    return "unknown status";
}

const char *bmg_last_error_detail(void) { return abi_detail().c_str(); }

bmg_status_t bmg_destroy(bmg_solver_t h)
{
    if (!h)
        return BMG_OK;
    if (h->dist) {
        dist_destroy(h->dist);
        for (void *p : h->allocs)
            cudaFree(p);
        delete h;
        return BMG_OK;
    }
    cudaDeviceSynchronize();
    for (auto &kv : h->graphs)
        kv.second.destroy();
    for (auto &kv : h->tgraphs)
        kv.second.destroy();
    for (cudaEvent_t e : h->tev)
        cudaEventDestroy(e);
    for (cudaEvent_t e : h->cev)
        if (e)
            cudaEventDestroy(e);
    if (h->pcg_ev)
        cudaEventDestroy(h->pcg_ev);
    if (h->pcg_tail)
        cudaEventDestroy(h->pcg_tail);
    for (auto &kv : h->sgraphs)
        cudaGraphExecDestroy(kv.second);
    if (h->solve_hist)
        cudaFree(h->solve_hist);
    if (h->solve_st_h)
        cudaFreeHost(h->solve_st_h);
    for (void *p : h->allocs)
        cudaFree(p);
    for (auto &kv : h->bgraphs)
        cudaGraphExecDestroy(kv.second);
    if (h->blk_arena)
        cudaFree(h->blk_arena);
    if (h->pcgb_ws)
        cudaFree(h->pcgb_ws);
    for (auto &kv : h->sbgraphs)
        cudaGraphExecDestroy(kv.second);
    if (h->sb_hist)
        cudaFree(h->sb_hist);
    if (h->sb_st_h)
        cudaFreeHost(h->sb_st_h);
    if (h->h_norm)
        pinned_release(h->h_norm);
    for (cudaEvent_t e : h->setup_ev)
        if (e)
            cudaEventDestroy(e);
    if (h->cap)
        cudaStreamDestroy(h->cap);
    for (cudaEvent_t e : h->hb_ev)
        if (e)
            cudaEventDestroy(e);
    if (h->hb_in)
        cudaStreamDestroy(h->hb_in);
    if (h->hb_out)
        cudaStreamDestroy(h->hb_out);
    delete h;
    return BMG_OK;
}

// BMG_SETUP_TRACE=1: host wall-clock of the setup phases on stderr (tuning aid)
static void setup_trace(const char *what, cudaStream_t s)
{
    static const bool on = getenv("BMG_SETUP_TRACE") != nullptr;
    if (!on)
        return;
    static std::chrono::steady_clock::time_point t0;
    cudaStreamSynchronize(s);
    auto now = std::chrono::steady_clock::now();
    if (strcmp(what, "start") != 0)
        fprintf(stderr, "bmg_setup %-16s %8.3f ms\n", what,
                std::chrono::duration<double, std::milli>(now - t0).count());
    t0 = now;
}

static bmg_status_t setup_impl(bmg_solver *h, const bmg_stencil_t *st, cudaStream_t s)
{
    const bmg_params_t &pr = h->prm;
    setup_trace("start", s);
    // level ladder (c1): n_{l+1} = floor(n_l/2) until min(nx,ny) <= coarsest
    {
        int nx = st->nx, ny = st->ny;
        h->L = 1;
        while ((nx < ny ? nx : ny) > pr.coarsest && (pr.max_levels <= 0 || h->L < pr.max_levels)) {
            nx /= 2;
            ny /= 2;
            h->L++;
        }
    }
    h->lv.resize(h->L);
    for (int l = 0; l < h->L; l++) {
        Level &v = h->lv[l];
        v.nx = l == 0 ? st->nx : h->lv[l - 1].nx / 2;
        v.ny = l == 0 ? st->ny : h->lv[l - 1].ny / 2;
        v.kind = l == 0 ? st->kind : 9;
        v.pitch = l == 0 ? st->pitch : round_pitch(v.nx);
    }
    // Every level array lives in ONE zeroed device block (one cudaMalloc: a few
    // large allocations cost ~1 ms, a dozen separate ones ~7-10 ms).  Pass 0 sizes
    // the arena, pass 1 carves it (256-B aligned pieces).
    double *arena = nullptr;
    size_t used = 0;
    auto take = [&](size_t n) {
        double *p = arena ? arena + used : nullptr;
        used += (n + 31) / 32 * 32;
        return p;
    };
    for (int pass = 0; pass < 2; pass++) {
        if (pass == 1) {
            TRY(dalloc(h, &arena, used));
            setup_trace("cudaMalloc", s);
            // zero everything but the level-0 planes (the arena's first block: S0 ingest
            // writes every element of it, ring and padding included)
            const Level &v0 = h->lv[0];
            const size_t np0 = (size_t)(v0.ny + 2) * (size_t)v0.pitch * (v0.kind == 9 ? 5 : 3);
            const size_t skip = (np0 + 31) / 32 * 32;
            CK(cudaMemsetAsync(arena + skip, 0, (used - skip) * sizeof(double), s));
            setup_trace("memset", s);
            used = 0;
        }
        for (int l = 0; l < h->L; l++) {
            Level &v = h->lv[l];
            size_t np = (size_t)(v.ny + 2) * (size_t)v.pitch;
            int npl = v.kind == 9 ? 5 : 3;
            double *blk = take(np * npl);  // the planes of a level form one block (plane
            for (int k = 0; k < npl; k++)  // stride np): one 3-D TMA box per row
                v.pl[k] = blk ? blk + k * np : nullptr;
            v.r = take(np);
            if (l > 0) {
                v.u = take(np);
                v.f = take(np);
            }
        }
        for (int l = 0; l + 1 < h->L; l++) {
            Level &c = h->lv[l + 1];
            size_t np = (size_t)(c.ny + 2) * (size_t)c.pitch;
            double *blk = take(np * 8);  // the 8 weight planes form one block (plane stride np)
            for (int k = 0; k < 8; k++)
                h->lv[l].ci[k] = blk ? blk + k * np : nullptr;
        }
        // the error word (zeroed with the arena), the norm partials and result
        h->d_err = (int *)take(64);
        h->partials = take(NORM_BLOCKS + 8);
        h->d_norm = take(8);
    }
    h->h_norm = pinned_slot();
    if (!h->h_norm)
        return fail(BMG_ENOMEM, "pinned host slot");

    setup_trace("allocate", s);
    CK(cudaEventCreate(&h->setup_ev[0]));
    CK(cudaEventCreate(&h->setup_ev[1]));
    CK(cudaEventRecord(h->setup_ev[0], s));
    // S0 ingest
    {
        Level &v = h->lv[0];
        const double *src[5] = {st->plane[0], st->plane[1], st->plane[2], st->plane[3], st->plane[4]};
        launch_ingest(v.nx, v.ny, v.kind, v.pitch, src, v.pl, h->d_err, s, 0, v.ny + 2);
        CK(cudaGetLastError());
    }
    setup_trace("ingest", s);
    // S1 + S2 per level
    for (int l = 0; l + 1 < h->L; l++) {
        Level &v = h->lv[l], &c = h->lv[l + 1];
        launch_setup_interp(v.op(), v.ci, c.pitch, h->d_err, s, 1, c.ny + 1);
        CK(cudaGetLastError());
        launch_setup_rap(v.op(), h->civ(l), c.nx, c.ny, c.pitch, c.pl, s, 1, c.ny);
        CK(cudaGetLastError());
    }
    setup_trace("interp+rap", s);
    // S3 coarsest dense Cholesky
    {
        Level &c = h->lv[h->L - 1];
        h->nco = c.nx * c.ny;
        if (h->nco > 6144)
            return fail(BMG_EINVAL, "coarsest level has more than 6144 unknowns; raise max_levels or lower coarsest");
        TRY(dalloc(h, &h->chol, (size_t)h->nco * h->nco));
        launch_assemble_dense(c.op(), h->chol, s);
        launch_chol_factor(h->nco, h->chol, h->d_err, s);
        CK(cudaGetLastError());
    }
    CK(cudaEventRecord(h->setup_ev[1], s));
    int herr = 0;
    CK(cudaMemcpyAsync(&herr, h->d_err, sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (herr & ERR_DIAG)
        return fail(BMG_EINVAL, "stencil diagonal a_O <= 0 at an interior point");
    if (herr & ERR_DEN)
        return fail(BMG_EINVAL, "interpolation denominator <= 0 (operator not suited to BoxMG collapse)");
    if (herr & ERR_PIVOT)
        return fail(BMG_ENOTSPD, "coarsest-level Cholesky pivot <= 0");
    setup_trace("cholesky+check", s);
    // c11 line relaxation: scratch sized for level 0, line pivots of every relaxed level
    if (pr.relax != BMG_RELAX_POINT) {
        if (h->lv[0].nx > LINE_NMAX || h->lv[0].ny > LINE_NMAX)
            return fail(BMG_EINVAL, "line relaxation: lines of at most 32768 unknowns");
        TRY(dalloc(h, &h->line_scr, line_scratch_doubles(h->lv[0].nx, h->lv[0].ny)));
        for (int l = 0; l + 1 < h->L; l++)
            launch_line_pivots(h->lv[l].op(), pr.relax, h->d_err, s);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(&herr, h->d_err, sizeof(int), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        if (herr & ERR_LINE)
            return fail(BMG_ENOTSPD, "line relaxation: a line block has an elimination pivot <= 0");
    }
    CK(cudaStreamCreateWithFlags(&h->cap, cudaStreamNonBlocking));
    // tail kernel: levels from the first with <= TAIL_POINTS unknowns down to the coarsest
    if (h->prm.fused && h->prm.relax == BMG_RELAX_POINT && h->L >= 2 && h->L <= 32) {
        long long lim = TAIL_POINTS;
        if (const char *e = getenv("BMG_TAIL_POINTS"))  // tuning knob (bench sweeps)
            lim = atoll(e);
        int l0 = h->L - 1;
        while (l0 > 0 && (long long)h->lv[l0 - 1].nx * h->lv[l0 - 1].ny <= lim)
            l0--;
        if (l0 <= h->L - 2) {
            TailPlan tp;
            memset(&tp, 0, sizeof(tp));
            tp.l0 = l0;
            tp.L = h->L;
            tp.nu1 = h->prm.nu1;
            tp.nu2 = h->prm.nu2;
            tp.cycle_sym = h->prm.cycle_sym;
            tp.affine = h->prm.affine;
            tp.chol = h->chol;
            for (int l = l0; l < h->L; l++) {
                tp.lv[l].A = h->lv[l].op();
                if (l + 1 < h->L)
                    tp.lv[l].ci = h->civ(l);
                tp.lv[l].f = h->lv[l].f;
                tp.lv[l].u = h->lv[l].u;
                tp.lv[l].r = h->lv[l].r;
            }
            // every tail level in shared memory when it fits (k_tail_sm); BMG_TAIL_SM=0: k_tail
            const char *tsm = getenv("BMG_TAIL_SM");
            if (!(tsm && atoi(tsm) == 0))
                tail_plan_smem(tp, h->nco, 200 * 1024 / 8);
            h->tail_sm = tp.sm_doubles;
            double *d = nullptr;
            TRY(dalloc(h, &d, sizeof(TailPlan) / sizeof(double) + 1));
            CK(cudaMemcpyAsync(d, &tp, sizeof(TailPlan), cudaMemcpyHostToDevice, s));
            h->tail = (TailPlan *)d;
            h->tail_l0 = l0;
        }
    }
    // small levels above the tail: the shared-memory tile legs
    if (h->prm.fused && h->prm.relax == BMG_RELAX_POINT && !h->prm.affine) {
        long long lim = TILE_POINTS;
        if (const char *e = getenv("BMG_TILE_POINTS"))  // tuning knob (bench sweeps)
            lim = atoll(e);
        for (int l = 0; l + 1 < h->L && l < 32 && l < h->tail_l0; l++) {
            Level &v = h->lv[l];
            if ((long long)v.nx * v.ny <= lim && tile_supported(v.kind, h->prm.nu1, h->prm.nu2)) {
                h->tile[l] = true;
                h->fplan.tmp[l] = v.r;  // ping-pong partner, as for a fused level (ring zero)
            }
        }
    }
    // fused streaming plan + ping-pong partner of u for every fused level above the tail
    for (int l = 0; l + 1 < h->L && l < 32 && l < h->tail_l0; l++) {
        Level &v = h->lv[l];
        if (!h->prm.fused || h->prm.relax != BMG_RELAX_POINT || h->prm.affine)
            break;
        if (h->tile[l])
            continue;
        TRY(fused_plan_level(h->fplan, l, v.nx, v.ny, v.pitch, v.kind, h->prm.nu1, h->prm.nu2, (v.pitch & 1) == 0,
                             h->prm.cycle_sym == 1));
        LevelPlan &lp = h->fplan.lv[l];
        if (!(lp.down && lp.up)) {
            lp.down = lp.up = false;
            continue;
        }
        // the ping-pong partner T is the level's residual array: a fused level never
        // stores r (its down leg restricts from shared memory), and T lives only
        // within one cycle; its ring must be 0 (the arena is zeroed, nothing wrote r yet)
        h->fplan.tmp[l] = v.r;
    }
    CK(cudaStreamSynchronize(s));
    setup_trace("lines/tail/fused", s);
    return BMG_OK;
}

bmg_status_t bmg_setup(const bmg_stencil_t *st, const bmg_params_t *params, void *cuda_stream, bmg_solver_t *out)
{
    if (!st || !out)
        return fail(BMG_EINVAL, "null stencil or out pointer");
    *out = nullptr;
    if (st->nx < 1 || st->ny < 1 || (st->kind != 5 && st->kind != 9) || st->pitch < (long long)st->nx + 2)
        return fail(BMG_EINVAL, "bad sizes: need nx,ny >= 1, kind in {5,9}, pitch >= nx+2");
    int npl = st->kind == 9 ? 5 : 3;
    for (int k = 0; k < npl; k++)
        if (!st->plane[k])
            return fail(BMG_EINVAL, "null stencil plane");
    bmg_solver *h = new bmg_solver();
    if (params)
        h->prm = *params;
    else
        bmg_params_default(&h->prm);
    if (h->prm.nu1 < 0 || h->prm.nu2 < 0 || h->prm.coarsest < 1 || h->prm.relax < BMG_RELAX_POINT ||
        h->prm.relax > BMG_RELAX_ALTLINES || (h->prm.cycle_sym != 0 && h->prm.cycle_sym != 1) ||
        (h->prm.affine != 0 && h->prm.affine != 1)) {
        delete h;
        return fail(BMG_EINVAL, "bad params");
    }
    bmg_status_t rc = setup_impl(h, st, (cudaStream_t)cuda_stream);
    if (rc != BMG_OK) {
        std::string d = abi_detail();
        bmg_destroy(h);
        abi_detail() = d;
        return rc;
    }
    *out = h;
    return BMG_OK;
}

}  // extern "C"


// Whether level l runs the fused streaming kernels for these level-l arrays.
static bool use_fused(bmg_solver *h, int l, const void *f, const void *uin, const void *uout)
{
    if (!h->prm.fused || l >= 32 || l + 1 >= h->L)
        return false;
    if (h->tile[l])
        return uin != uout && f && uout;
    const LevelPlan &lp = h->fplan.lv[l];
    return lp.down && lp.up && al16(f) && al16(uin) && al16(uout) && uin != uout;
}

// nsweeps sweeps of the handle's relaxation on level l (c6 point or c11 line GS);
// rev: the adjoint ordering (c12)
static void relax_level(bmg_solver *h, int l, const double *f, double *u, int nsweeps, cudaStream_t s, int *n,
                        bool rev = false)
{
    if (h->prm.relax == BMG_RELAX_POINT)
        launch_relax(h->lv[l].op(), f, u, nsweeps, s, n, rev);
    else
        launch_relax_lines(h->lv[l].op(), f, u, nsweeps, h->prm.relax, h->line_scr, s, n, rev);
}

static void copy_level(bmg_solver *h, int l, double *dst, const double *src, cudaStream_t s)
{
    if (dst != src)
        cudaMemcpyAsync(dst, src, (size_t)(h->lv[l].ny + 2) * h->lv[l].pitch * sizeof(double),
                        cudaMemcpyDeviceToDevice, s);
}

// Down leg of level l: u_out = relax^nu1(u_in); fc = P^T (f - A u_out); uc = 0 (if non-null).
// u_in == nullptr: a zero start (c9) that is not read.
static void enqueue_down(bmg_solver *h, int l, bool fused, const double *f, const double *uin, double *uout,
                         double *fc, double *uc, cudaStream_t s, int *n)
{
    Level &v = h->lv[l];
    if (fused && h->tile[l]) {
        TileArgs t{v.op(), h->civ(l), f, uin, nullptr, uout, fc, uc, uin == nullptr};
        launch_tile_down(t, h->prm.nu1, s);
        *n += 1;
        return;
    }
    if (fused && fused_down(h->fplan, l, v.op(), h->civ(l), f, uin, uout, fc, uc, s, n))
        return;
    if (fused && uout == v.r) {  // the per-step path would need r, which is T here
        h->cycle_err = true;
        return;
    }
    if (uin)
        copy_level(h, l, uout, uin, s);
    else
        launch_zero_interior(v.op(), uout, s);
    relax_level(h, l, f, uout, h->prm.nu1, s, n);
    launch_residual(v.op(), f, uout, v.r, s);
    // after nu1 >= 1 point-GS sweeps the last colour's residual vanishes
    launch_restrict(v.op(), h->civ(l), v.r, fc, uc, s, h->prm.relax == BMG_RELAX_POINT && h->prm.nu1 > 0);
    *n += 2;
}

// Up leg of level l: u_out = relax^nu2(u_in + P ec).
static void enqueue_up(bmg_solver *h, int l, bool fused, const double *f, const double *uin, const double *ec,
                       double *uout, cudaStream_t s, int *n)
{
    Level &v = h->lv[l];
    if (fused && h->tile[l]) {
        TileArgs t{v.op(), h->civ(l), f, uin, ec, uout, nullptr, nullptr, 0};
        launch_tile_up(t, h->prm.nu2, h->prm.cycle_sym == 1, s);
        *n += 1;
        return;
    }
    if (fused && fused_up(h->fplan, l, v.op(), h->civ(l), f, uin, ec, 0, h->lv[l + 1].ny + 2, uout, s, n))
        return;
    copy_level(h, l, uout, uin, s);
    // c14: v.r still holds the residual restricted on this level's down leg
    launch_interp_add(v.op(), h->civ(l), ec, uout, s, h->prm.affine ? v.r : nullptr);
    *n += 1;
    relax_level(h, l, f, uout, h->prm.nu2, s, n, h->prm.cycle_sym == 1);
}

// Enqueue one V(nu1,nu2) cycle (fig:vcycle_flowchart; DESIGN §3 c9) on s.
// A fused level's iterate goes U -> T on the down leg and T -> U on the up leg.
// bmg_timing: the next free (start, end) event pair
static bool next_events(bmg_solver *h, cudaEvent_t *e)
{
    while (h->tev.size() < h->tev_used + 2) {
        cudaEvent_t ev;
        if (cudaEventCreate(&ev) != cudaSuccess)
            return false;
        h->tev.push_back(ev);
    }
    e[0] = h->tev[h->tev_used];
    e[1] = h->tev[h->tev_used + 1];
    h->tev_used += 2;
    return true;
}

// rec (bmg_timing): an event pair recorded around the level-0 down leg (external
// event-record nodes when captured)
// seg (bmg_profile_legs): 2*lt+2 events recorded at every leg boundary
static int enqueue_cycle(bmg_solver *h, const double *f0, double *u0, cudaStream_t s,
                         const cudaEvent_t *rec = nullptr, const cudaEvent_t *seg = nullptr)
{
    int n = 0;
    const int L = h->L;
    auto F = [&](int l) { return l == 0 ? f0 : (const double *)h->lv[l].f; };
    auto U = [&](int l) { return l == 0 ? u0 : h->lv[l].u; };
    bool fz[64];
    const int lt = h->tail_l0 < L ? h->tail_l0 : L - 1;  // levels >= lt: tail kernel / coarse solve
    for (int l = 0; l < lt; l++) {
        double *T = l < 32 ? h->fplan.tmp[l] : nullptr;
        fz[l] = T && use_fused(h, l, F(l), U(l), T);
    }
    for (int l = 0; l < lt; l++) {
        double *T = l < 32 ? h->fplan.tmp[l] : nullptr;
        // a coarse level's down leg starts from zero (c9): a fused one does not read it,
        // so the level above need not write that zero start either
        const bool uz = l > 0 && fz[l];
        double *uc = (l + 1 < lt && fz[l + 1]) ? nullptr : h->lv[l + 1].u;
        if (seg && l == 0)
            cudaEventRecordWithFlags(seg[0], s, cudaEventRecordExternal);
        if (rec && l == 0)
            cudaEventRecordWithFlags(rec[0], s, cudaEventRecordExternal);
        enqueue_down(h, l, fz[l], F(l), uz ? nullptr : U(l), fz[l] ? T : U(l), h->lv[l + 1].f, uc, s, &n);
        if (rec && l == 0)
            cudaEventRecordWithFlags(rec[1], s, cudaEventRecordExternal);
        if (seg)
            cudaEventRecordWithFlags(seg[l + 1], s, cudaEventRecordExternal);
    }
    if (seg && lt == 0)
        cudaEventRecordWithFlags(seg[0], s, cudaEventRecordExternal);
    // no level-0 down leg of its own (the tail or the coarse solve starts at level 0):
    // bmg_timing records around that launch instead
    const bool rec_here = rec && lt == 0;
    if (rec_here)
        cudaEventRecordWithFlags(rec[0], s, cudaEventRecordExternal);
    if (h->tail) {
        launch_tail(h->tail, h->nco, F(0), U(0), s, h->tail_sm);
        n += 1;
    } else {
        Level &c = h->lv[L - 1];
        launch_coarse_solve(c.op(), h->chol, F(L - 1), U(L - 1), s);
        n += 1;
    }
    if (rec_here)
        cudaEventRecordWithFlags(rec[1], s, cudaEventRecordExternal);
    if (seg)
        cudaEventRecordWithFlags(seg[lt + 1], s, cudaEventRecordExternal);
    for (int l = lt - 1; l >= 0; l--) {
        enqueue_up(h, l, fz[l], F(l), fz[l] ? h->fplan.tmp[l] : U(l), h->lv[l + 1].u, U(l), s, &n);
        if (seg)
            cudaEventRecordWithFlags(seg[lt + 2 + (lt - 1 - l)], s, cudaEventRecordExternal);
    }
    return n;
}

// The cycle's graph for (f, x).  timed: the variant with the two event-record
// nodes of bmg_timing (their events are re-pointed before every launch).
static bmg_status_t get_graph(bmg_solver *h, const double *f, double *x, bool timed, cudaGraphExec_t *out)
{
    auto key = std::make_pair((const void *)f, (const void *)x);
    auto &cache = timed ? h->tgraphs : h->graphs;
    auto it = cache.find(key);
    if (it != cache.end()) {
        *out = it->second.ex;
        return BMG_OK;
    }
    if (timed && !h->cev[0]) {
        CK(cudaEventCreate(&h->cev[0]));
        CK(cudaEventCreate(&h->cev[1]));
    }
    cudaGraph_t g;
    CK(cudaStreamBeginCapture(h->cap, cudaStreamCaptureModeThreadLocal));
    h->cycle_err = false;
    int n = enqueue_cycle(h, f, x, h->cap, timed ? h->cev : nullptr);
    cudaError_t e = cudaStreamEndCapture(h->cap, &g);
    if (e != cudaSuccess)
        return fail(BMG_ECUDA, std::string("graph capture: ") + cudaGetErrorString(e));
    if (h->cycle_err) {
        cudaGraphDestroy(g);
        return fail(BMG_ECUDA, "a fused leg was rejected while capturing the cycle (tensor-map encode?)");
    }
    GraphRec gr;
    gr.g = g;
    if (timed) {
        size_t nn = 0;
        CK(cudaGraphGetNodes(g, nullptr, &nn));
        std::vector<cudaGraphNode_t> nodes(nn);
        CK(cudaGraphGetNodes(g, nodes.data(), &nn));
        for (cudaGraphNode_t nd : nodes) {
            cudaGraphNodeType ty;
            CK(cudaGraphNodeGetType(nd, &ty));
            if (ty != cudaGraphNodeTypeEventRecord)
                continue;
            cudaEvent_t ev;
            CK(cudaGraphEventRecordNodeGetEvent(nd, &ev));
            for (int k = 0; k < 2; k++)
                if (ev == h->cev[k])
                    gr.ev_node[k] = nd;
        }
        if (!gr.ev_node[0] || !gr.ev_node[1])
            return fail(BMG_ECUDA, "timed graph: event-record nodes not found");
    }
    CK(cudaGraphInstantiate(&gr.ex, g, 0));
    if (!timed) {
        cudaGraphDestroy(g);
        gr.g = nullptr;
    }
    h->kernels_per_cycle = n;
    if (cache.size() > 16) {  // bound the cache
        for (auto &kv : cache)
            kv.second.destroy();
        cache.clear();
    }
    cache[key] = gr;
    *out = gr.ex;
    return BMG_OK;
}

// The device-side solve loop for (f, x): ONE graph whose conditional WHILE node
// runs [V-cycle, residual norm, k_solve_step] until the stopping test fails --
// no host round trip per cycle (conditional graph nodes).
static bmg_status_t get_solve_graph(bmg_solver *h, const double *f, double *x, cudaGraphExec_t *out)
{
    auto key = std::make_pair((const void *)f, (const void *)x);
    auto it = h->sgraphs.find(key);
    if (it != h->sgraphs.end()) {
        *out = it->second;
        return BMG_OK;
    }
    cudaGraph_t g;
    CK(cudaGraphCreate(&g, 0));
    cudaGraphConditionalHandle hd;
    CK(cudaGraphConditionalHandleCreate(&hd, g, 1, cudaGraphCondAssignDefault));  // enter the loop
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = hd;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t node;
    CK(cudaGraphAddNode(&node, g, nullptr, 0, &cp));
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    CK(cudaStreamBeginCaptureToGraph(h->cap, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    h->cycle_err = false;
    enqueue_cycle(h, f, x, h->cap);
    launch_resid_norm(h->lv[0].op(), f, x, nullptr, h->partials, h->d_norm, h->cap);
    launch_solve_step(hd, h->d_norm, h->solve_st, h->solve_hist, h->cap);
    cudaError_t e = cudaStreamEndCapture(h->cap, &body);
    if (e != cudaSuccess || h->cycle_err) {
        cudaGraphDestroy(g);
        return fail(BMG_ECUDA, std::string("solve graph capture: ") +
                                   (h->cycle_err ? "a fused leg was rejected" : cudaGetErrorString(e)));
    }
    cudaGraphExec_t ex;
    e = cudaGraphInstantiate(&ex, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess)
        return fail(BMG_ECUDA, std::string("solve graph instantiate: ") + cudaGetErrorString(e));
    if (h->sgraphs.size() > 16) {
        for (auto &kv : h->sgraphs)
            cudaGraphExecDestroy(kv.second);
        h->sgraphs.clear();
    }
    h->sgraphs[key] = ex;
    *out = ex;
    return BMG_OK;
}

extern "C" {

bmg_status_t bmg_vcycle(bmg_solver_t h, const double *rhs, double *x, int ncycles, void *cuda_stream)
{
    join_pcg(h, (cudaStream_t)cuda_stream);
    if (!h || !rhs || !x || ncycles < 0)
        return fail(BMG_EINVAL, "bad arguments to bmg_vcycle");
    if (h->dist) {
        std::string err;
        bmg_status_t rc = dist_vcycle(h->dist, rhs, x, ncycles, (cudaStream_t)cuda_stream, err);
        return rc == BMG_OK ? rc : fail(rc, err);
    }
    cudaGraphExec_t ex;
    TRY(get_graph(h, rhs, x, h->timing, &ex));
    const GraphRec &gr = (h->timing ? h->tgraphs : h->graphs)[std::make_pair((const void *)rhs, (const void *)x)];
    for (int k = 0; k < ncycles; k++) {
        if (h->timing) {  // a fresh event pair for this launch's level-0 down leg
            cudaEvent_t ev[2];
            if (!next_events(h, ev))
                return fail(BMG_ECUDA, "bmg_timing: cudaEventCreate failed");
            CK(cudaGraphExecEventRecordNodeSetEvent(ex, gr.ev_node[0], ev[0]));
            CK(cudaGraphExecEventRecordNodeSetEvent(ex, gr.ev_node[1], ev[1]));
        }
        CK(cudaGraphLaunch(ex, (cudaStream_t)cuda_stream));
    }
    return BMG_OK;
}

bmg_status_t bmg_timing(bmg_solver_t h, int enable)
{
    if (!h || h->dist)
        return fail(BMG_EINVAL, "bmg_timing: null or distributed handle");
    h->timing = enable != 0;
    h->tev_used = 0;
    return BMG_OK;
}

bmg_status_t bmg_timing_read(bmg_solver_t h, double *ms_total, int *launches)
{
    if (!h || h->dist || !ms_total || !launches)
        return fail(BMG_EINVAL, "bmg_timing_read: bad arguments");
    double tot = 0.0;
    for (size_t i = 0; i + 1 < h->tev_used; i += 2) {
        CK(cudaEventSynchronize(h->tev[i + 1]));
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, h->tev[i], h->tev[i + 1]));
        tot += ms;
    }
    *ms_total = tot;
    *launches = (int)(h->tev_used / 2);
    h->tev_used = 0;
    return BMG_OK;
}

bmg_status_t bmg_setup_time(bmg_solver_t h, double *device_ms)
{
    if (!h || h->dist || !device_ms || !h->setup_ev[0])
        return fail(BMG_EINVAL, "bmg_setup_time: bad arguments");
    float ms = 0.f;
    CK(cudaEventSynchronize(h->setup_ev[1]));
    CK(cudaEventElapsedTime(&ms, h->setup_ev[0], h->setup_ev[1]));
    *device_ms = ms;
    return BMG_OK;
}

bmg_status_t bmg_profile_legs(bmg_solver_t h, const double *rhs, double *x, int ncycles, double *ms_out, int cap,
                              int *nseg, void *cuda_stream)
{
    join_pcg(h, (cudaStream_t)cuda_stream);
    if (!h || h->dist || !rhs || !x || !ms_out || !nseg || ncycles < 1 || cap < 2 * h->L + 1)
        return fail(BMG_EINVAL, "bmg_profile_legs: bad arguments");
    const int lt = h->tail_l0 < h->L ? h->tail_l0 : h->L - 1;
    const int ne = 2 * lt + 2;
    std::vector<cudaEvent_t> ev(ne);
    for (auto &e : ev)
        CK(cudaEventCreate(&e));
    auto cleanup = [&]() {
        for (auto &e : ev)
            cudaEventDestroy(e);
    };
    cudaGraph_t g;
    CK(cudaStreamBeginCapture(h->cap, cudaStreamCaptureModeThreadLocal));
    h->cycle_err = false;
    enqueue_cycle(h, rhs, x, h->cap, nullptr, ev.data());
    cudaError_t e = cudaStreamEndCapture(h->cap, &g);
    if (e != cudaSuccess || h->cycle_err) {
        cleanup();
        return fail(BMG_ECUDA, "bmg_profile_legs: capture failed");
    }
    cudaGraphExec_t ex;
    e = cudaGraphInstantiate(&ex, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) {
        cleanup();
        return fail(BMG_ECUDA, std::string("bmg_profile_legs: ") + cudaGetErrorString(e));
    }
    std::vector<double> acc(ne - 1, 0.0);
    cudaStream_t s = (cudaStream_t)cuda_stream;
    for (int c = 0; c < ncycles && e == cudaSuccess; c++) {
        e = cudaGraphLaunch(ex, s);
        if (e == cudaSuccess)
            e = cudaStreamSynchronize(s);
        for (int k = 0; k + 1 < ne && e == cudaSuccess; k++) {
            float ms = 0.f;
            e = cudaEventElapsedTime(&ms, ev[k], ev[k + 1]);
            acc[k] += ms;
        }
    }
    cudaGraphExecDestroy(ex);
    cleanup();
    if (e != cudaSuccess)
        return fail(BMG_ECUDA, std::string("bmg_profile_legs: ") + cudaGetErrorString(e));
    for (int k = 0; k + 1 < ne; k++)
        ms_out[k] = acc[k] / ncycles;
    *nseg = ne - 1;
    return BMG_OK;
}

bmg_status_t bmg_vcycle_host(bmg_solver_t h, const double *rhs_host, double *x_host, int ncycles, void *cuda_stream)
{
    join_pcg(h, (cudaStream_t)cuda_stream);
    if (!h || !rhs_host || !x_host || ncycles < 0 || h->dist)
        return fail(BMG_EINVAL, "bad arguments to bmg_vcycle_host (not for distributed handles)");
    Level &v = h->lv[0];
    size_t bytes = (size_t)(v.ny + 2) * v.pitch * sizeof(double);
    if (!h->stage_f) {
        TRY(dalloc(h, &h->stage_f, bytes / sizeof(double)));
        TRY(dalloc(h, &h->stage_x, bytes / sizeof(double)));
    }
    cudaStream_t s = (cudaStream_t)cuda_stream;
    CK(cudaMemcpyAsync(h->stage_f, rhs_host, bytes, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(h->stage_x, x_host, bytes, cudaMemcpyHostToDevice, s));
    TRY(bmg_vcycle(h, h->stage_f, h->stage_x, ncycles, cuda_stream));
    CK(cudaMemcpyAsync(x_host, h->stage_x, bytes, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return BMG_OK;
}

// nprob independent problems with host data, pipelined over two device staging slots:
// problem i's host->device copies (stream hb_in) and problem i-1's device->host copy
// (stream hb_out) overlap the cycles of the problem in between (cuda_stream), so the
// batch runs at the PCIe rate instead of copy + compute + copy in series.
bmg_status_t bmg_vcycle_host_batch(bmg_solver_t h, int nprob, const double *const *rhs_host,
                                   double *const *x_host, int ncycles, void *cuda_stream)
{
    join_pcg(h, (cudaStream_t)cuda_stream);
    if (!h || nprob < 0 || (nprob > 0 && (!rhs_host || !x_host)) || ncycles < 0 || h->dist)
        return fail(BMG_EINVAL, "bad arguments to bmg_vcycle_host_batch (not for distributed handles)");
    for (int i = 0; i < nprob; i++)
        if (!rhs_host[i] || !x_host[i])
            return fail(BMG_EINVAL, "bmg_vcycle_host_batch: NULL host array");
    Level &v = h->lv[0];
    const size_t bytes = (size_t)(v.ny + 2) * v.pitch * sizeof(double);
    if (!h->stage_f) {
        TRY(dalloc(h, &h->stage_f, bytes / sizeof(double)));
        TRY(dalloc(h, &h->stage_x, bytes / sizeof(double)));
    }
    if (!h->stage_f2) {
        TRY(dalloc(h, &h->stage_f2, bytes / sizeof(double)));
        TRY(dalloc(h, &h->stage_x2, bytes / sizeof(double)));
        CK(cudaStreamCreateWithFlags(&h->hb_in, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&h->hb_out, cudaStreamNonBlocking));
        for (cudaEvent_t &e : h->hb_ev)
            CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    cudaStream_t s = (cudaStream_t)cuda_stream;
    double *fs[2] = {h->stage_f, h->stage_f2}, *xs[2] = {h->stage_x, h->stage_x2};
    cudaEvent_t *in_done = h->hb_ev, *cyc_done = h->hb_ev + 2, *out_done = h->hb_ev + 4;
    // the slots are free of earlier work on cuda_stream before the first copy into them
    CK(cudaEventRecord(cyc_done[0], s));
    CK(cudaStreamWaitEvent(h->hb_in, cyc_done[0], 0));
    for (int i = 0; i < nprob; i++) {
        const int k = i & 1;
        if (i >= 2)  // slot k's previous result has left (its D2H waited for its cycle)
            CK(cudaStreamWaitEvent(h->hb_in, out_done[k], 0));
        CK(cudaMemcpyAsync(fs[k], rhs_host[i], bytes, cudaMemcpyHostToDevice, h->hb_in));
        CK(cudaMemcpyAsync(xs[k], x_host[i], bytes, cudaMemcpyHostToDevice, h->hb_in));
        CK(cudaEventRecord(in_done[k], h->hb_in));
        CK(cudaStreamWaitEvent(s, in_done[k], 0));
        TRY(bmg_vcycle(h, fs[k], xs[k], ncycles, cuda_stream));
        CK(cudaEventRecord(cyc_done[k], s));
        CK(cudaStreamWaitEvent(h->hb_out, cyc_done[k], 0));
        CK(cudaMemcpyAsync(x_host[i], xs[k], bytes, cudaMemcpyDeviceToHost, h->hb_out));
        CK(cudaEventRecord(out_done[k], h->hb_out));
    }
    CK(cudaStreamSynchronize(h->hb_out));
    CK(cudaStreamSynchronize(s));
    return BMG_OK;
}

bmg_status_t bmg_residual_norm(bmg_solver_t h, const double *rhs, const double *x, double *r_out, double *norm_host,
                               void *cuda_stream)
{
    join_pcg(h, (cudaStream_t)cuda_stream);
    if (!h || !rhs || !x || !norm_host || (h->dist && r_out))
        return fail(BMG_EINVAL, "bad arguments to bmg_residual_norm");
    cudaStream_t s = (cudaStream_t)cuda_stream;
    if (h->dist) {
        std::string err;
        bmg_status_t rc = dist_resid_norm(h->dist, rhs, x, norm_host, s, err);
        return rc == BMG_OK ? rc : fail(rc, err);
    }
    launch_resid_norm(h->lv[0].op(), rhs, x, r_out, h->partials, h->d_norm, s);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(h->h_norm, h->d_norm, sizeof(double), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    *norm_host = h->h_norm[0];
    return BMG_OK;
}

bmg_status_t bmg_solve(bmg_solver_t h, const double *rhs, double *x, double tol, int maxiter, int *iters_out,
                       double *hist_host, void *cuda_stream)
{
    join_pcg(h, (cudaStream_t)cuda_stream);
    if (!h || !rhs || !x || maxiter < 0 || !(tol >= 0))
        return fail(BMG_EINVAL, "bad arguments to bmg_solve");
    cudaStream_t s = (cudaStream_t)cuda_stream;
    if (iters_out)
        *iters_out = 0;
    // history + state on the device (the graph loop's and the one-launch tail solve's)
    auto solve_buffers = [&]() -> bmg_status_t {
        if (h->solve_cap < maxiter + 1) {
            CK(cudaStreamSynchronize(s));
            for (auto &kv : h->sgraphs)  // their step nodes point at the old history
                cudaGraphExecDestroy(kv.second);
            h->sgraphs.clear();
            if (h->solve_hist)
                cudaFree(h->solve_hist);
            h->solve_hist = nullptr;
            h->solve_cap = 0;
            const int cap = maxiter + 1 > 1024 ? maxiter + 1 : 1024;  // rarely reallocated (graphs go with it)
            void *q;
            CK(cudaMalloc(&q, sizeof(double) * (size_t)cap + sizeof(SolveState) + 64));
            h->solve_hist = (double *)q;
            h->solve_cap = cap;
            h->solve_st = (SolveState *)(h->solve_hist + h->solve_cap + 1);
            if (!h->solve_st_h)
                CK(cudaMallocHost(&h->solve_st_h, sizeof(SolveState)));
        }
        return BMG_OK;
    };
    // the whole hierarchy in the shared-memory tail (small problems, config 1): norms, cycles
    // and stopping test in ONE launch, the data staged once; bitwise the
    // graph loop's iterate and history (tests/test_gpu_solve.py)
    const char *tso = getenv("BMG_TAIL_SOLVE");  // 0: the graph loop (A/B, tests)
    const bool tail_solve_off = tso && atoi(tso) == 0;
    if (!h->dist && !h->timing && h->tail && h->tail_l0 == 0 && h->tail_sm > 0 && !tail_solve_off) {
        TRY(solve_buffers());
        *h->solve_st_h = SolveState{0.0, tol, 0, maxiter};
        CK(cudaMemcpyAsync(h->solve_st, h->solve_st_h, sizeof(SolveState), cudaMemcpyHostToDevice, s));
        launch_tail_solve(h->tail, rhs, x, h->solve_st, h->solve_hist, s, h->tail_sm);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(h->solve_st_h, h->solve_st, sizeof(SolveState), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        const int k = h->solve_st_h->k;
        const double fn0 = h->solve_st_h->fn;
        std::vector<double> hv(k + 1);
        CK(cudaMemcpy(hv.data(), h->solve_hist, sizeof(double) * (k + 1), cudaMemcpyDeviceToHost));
        if (hist_host)
            for (int i = 0; i <= k; i++)
                hist_host[i] = hv[i];
        if (iters_out)
            *iters_out = k;
        return (fn0 == 0.0 || hv[k] <= tol * fn0) ? BMG_OK : fail(BMG_ENOTCONV, "maxiter reached");
    }
    double fn;
    if (h->dist) {  // ||rhs|| = residual norm of x = 0
        std::string err;
        int row0, nrows;
        dist_local_rows(h->dist, &row0, &nrows, nullptr, nullptr, nullptr);
        if (!h->stage_x) {
            TRY(dalloc(h, &h->stage_x, (size_t)h->dist_rows_total));
            CK(cudaMemsetAsync(h->stage_x, 0, sizeof(double) * (size_t)h->dist_rows_total, s));
        }
        bmg_status_t rc = dist_resid_norm(h->dist, rhs, h->stage_x, &fn, s, err);
        if (rc != BMG_OK)
            return fail(rc, err);
    } else {
        Level &v = h->lv[0];
        launch_norm(v.op(), rhs, h->partials, h->d_norm, s);
        CK(cudaMemcpyAsync(h->h_norm, h->d_norm, sizeof(double), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        fn = h->h_norm[0];
    }
    if (fn == 0.0) {  // b = 0 -> x = 0 immediately
        if (h->dist)
            CK(cudaMemsetAsync(x, 0, sizeof(double) * (size_t)h->dist_rows_total, s));
        else
            launch_zero_interior(h->lv[0].op(), x, s);
        CK(cudaStreamSynchronize(s));
        if (hist_host)
            hist_host[0] = 0.0;
        return BMG_OK;
    }
    double rn;
    TRY(bmg_residual_norm(h, rhs, x, nullptr, &rn, cuda_stream));
    if (hist_host)
        hist_host[0] = rn;
    int k = 0;
    if (h->dist || h->timing) {  // host loop: one synchronised norm per cycle
        while (rn > tol * fn && k < maxiter) {
            TRY(bmg_vcycle(h, rhs, x, 1, cuda_stream));
            k++;
            TRY(bmg_residual_norm(h, rhs, x, nullptr, &rn, cuda_stream));
            if (hist_host)
                hist_host[k] = rn;
        }
    } else if (rn > tol * fn && maxiter > 0) {  // device loop: one graph launch, one wait
        TRY(solve_buffers());
        cudaGraphExec_t ex;
        TRY(get_solve_graph(h, rhs, x, &ex));
        *h->solve_st_h = SolveState{fn, tol, 0, maxiter};
        CK(cudaMemcpyAsync(h->solve_st, h->solve_st_h, sizeof(SolveState), cudaMemcpyHostToDevice, s));
        CK(cudaGraphLaunch(ex, s));
        CK(cudaMemcpyAsync(h->solve_st_h, h->solve_st, sizeof(SolveState), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        k = h->solve_st_h->k;
        std::vector<double> hv(k + 1);
        CK(cudaMemcpy(hv.data(), h->solve_hist, sizeof(double) * (k + 1), cudaMemcpyDeviceToHost));
        rn = hv[k];
        if (hist_host)
            for (int i = 1; i <= k; i++)
                hist_host[i] = hv[i];
    }
    if (iters_out)
        *iters_out = k;
    return rn <= tol * fn ? BMG_OK : fail(BMG_ENOTCONV, "maxiter reached");
}

/*
 * c13: conjugate gradients preconditioned by one V(nu,nu) cycle from a zero
 * guess (symmetric with cycle_sym = 1, c12) -- the textbook PCG recurrences
 * as DESIGN §3 c13 states them, every vector step a kernel.  The scalars
 * alpha = rho/(p.q) and beta = rho'/rho are formed on the device from the
 * deterministic dot products (slots of sc[]), so the host waits once per
 * iteration, for ||r|| (the stopping test); the next iteration's
 * preconditioner, rho' and direction -- which touch only z, p and sc -- are
 * enqueued before that wait, so the GPU does not idle during it.
 */
bmg_status_t bmg_pcg(bmg_solver_t h, const double *rhs, double *x, double tol, int maxiter, int *iters_out,
                     double *hist_host, void *cuda_stream)
{
    join_pcg(h, (cudaStream_t)cuda_stream);
    if (!h || !rhs || !x || maxiter < 0 || !(tol >= 0))
        return fail(BMG_EINVAL, "bad arguments to bmg_pcg");
    if (h->dist)
        return fail(BMG_EINVAL, "bmg_pcg: single-GPU handles only");
    if (h->prm.nu1 != h->prm.nu2 || h->prm.cycle_sym != 1)
        return fail(BMG_EINVAL, "bmg_pcg: the preconditioner must be symmetric (nu1 == nu2, cycle_sym = 1)");
    cudaStream_t s = (cudaStream_t)cuda_stream;
    if (iters_out)
        *iters_out = 0;
    const Level &v = h->lv[0];
    const Op A = v.op();
    const size_t np = (size_t)(v.ny + 2) * (size_t)v.pitch;
    if (!h->pcg_ws) {
        TRY(dalloc(h, &h->pcg_ws, 4 * np + 32));
        CK(cudaMemsetAsync(h->pcg_ws, 0, (4 * np + 32) * sizeof(double), s));
        CK(cudaEventCreateWithFlags(&h->pcg_ev, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&h->pcg_tail, cudaEventDisableTiming));
    }
    double *r = h->pcg_ws, *z = r + np, *p = z + np, *q = p + np, *sc = q + np;
    enum { PQ = 1, RN = 2 };  // sc slots; rho alternates between slots 0 and 3
    double fn;
    launch_norm(A, rhs, h->partials, h->d_norm, s);
    CK(cudaMemcpyAsync(h->h_norm, h->d_norm, sizeof(double), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    fn = h->h_norm[0];
    if (fn == 0.0) {
        launch_zero_interior(A, x, s);
        CK(cudaStreamSynchronize(s));
        if (hist_host)
            hist_host[0] = 0.0;
        return BMG_OK;
    }
    double rn;
    TRY(bmg_residual_norm(h, rhs, x, r, &rn, cuda_stream));  // r = f - A x0
    if (hist_host)
        hist_host[0] = rn;
    int k = 0;
    if (rn > tol * fn && maxiter > 0) {
        auto precondition = [&]() -> bmg_status_t {  // z = one V-cycle on r from z = 0
            launch_zero_interior(A, z, s);
            return bmg_vcycle(h, r, z, 1, cuda_stream);
        };
        int cur = 0;  // slot of the current rho
        TRY(precondition());
        CK(cudaMemcpyAsync(p, z, np * sizeof(double), cudaMemcpyDeviceToDevice, s));
        launch_dot(A, r, z, h->partials, sc + cur, s);
        while (k < maxiter) {
            launch_matvec_dot(A, p, q, h->partials, sc + PQ, s);                     // q = A p, p.q
            launch_cg_update_norm(A, sc, cur, PQ, p, q, x, r, h->partials, sc + RN, s);  // alpha = rho / (p.q)
            k++;
            CK(cudaMemcpyAsync(h->h_norm, sc + RN, sizeof(double), cudaMemcpyDeviceToHost, s));
            CK(cudaEventRecord(h->pcg_ev, s));
            // the next direction, speculatively (z, p and sc only; x and r are final),
            // unless this was the last allowed iteration
            const int nxt = 3 - cur;
            const bool spec = k < maxiter;
            if (spec) {
                TRY(precondition());
                launch_dot(A, r, z, h->partials, sc + nxt, s);
                launch_cg_direction(A, sc, nxt, cur, z, p, s);  // beta = rho' / rho
            }
            CK(cudaGetLastError());
            CK(cudaEventSynchronize(h->pcg_ev));
            rn = h->h_norm[0];
            if (hist_host)
                hist_host[k] = rn;
            if (rn <= tol * fn) {
                if (spec) {  // left queued: later calls on any stream join it (join_pcg)
                    CK(cudaEventRecord(h->pcg_tail, s));
                    h->pcg_pending = true;
                }
                break;
            }
            cur = nxt;
        }
    }
    CK(cudaGetLastError());
    if (iters_out)
        *iters_out = k;
    return rn <= tol * fn ? BMG_OK : fail(BMG_ENOTCONV, "maxiter reached");
}

}  // extern "C"

extern "C" {

bmg_status_t bmg_num_levels(bmg_solver_t h, int *L)
{
    if (!h || !L)
        return fail(BMG_EINVAL, "null argument");
    if (h->dist) {
        int K, Li;
        dist_local_rows(h->dist, nullptr, nullptr, nullptr, nullptr, &K);
        bmg_num_levels(h->dist_inner, &Li);
        *L = K + Li;
        return BMG_OK;
    }
    *L = h->L;
    return BMG_OK;
}

bmg_status_t bmg_level_shape(bmg_solver_t h, int level, int *nx, int *ny, int *kind)
{
    if (!h || h->dist || level < 0 || level >= h->L)
        return fail(BMG_EINVAL, "bad level");
    if (nx)
        *nx = h->lv[level].nx;
    if (ny)
        *ny = h->lv[level].ny;
    if (kind)
        *kind = h->lv[level].kind;
    return BMG_OK;
}

bmg_status_t bmg_level_pitch(bmg_solver_t h, int level, long long *pitch)
{
    if (!h || h->dist || !pitch || level < 0 || level >= h->L)
        return fail(BMG_EINVAL, "bad level");
    *pitch = h->lv[level].pitch;
    return BMG_OK;
}

bmg_status_t bmg_cycle_kernel_count(bmg_solver_t h, int *count)
{
    if (!h || !count)
        return fail(BMG_EINVAL, "null argument");
    if (h->dist) {  // two fused legs per slab level (per rank) + the inner cycle
        int K, ni = 0;
        dist_local_rows(h->dist, nullptr, nullptr, nullptr, nullptr, &K);
        TRY(bmg_cycle_kernel_count(h->dist_inner, &ni));
        *count = 2 * K * h->dist_local_ranks + ni;
        return BMG_OK;
    }
    if (h->kernels_per_cycle == 0) {  // count by a dry capture
        cudaGraph_t g;
        CK(cudaStreamBeginCapture(h->cap, cudaStreamCaptureModeThreadLocal));
        // dry capture on two distinct, 16-byte-aligned level-0 arrays that are not the
        // fused ping-pong partner (T = lv[0].r), so the count is that of the cycle
        // bmg_vcycle runs on caller arrays
        Level &v0 = h->lv[0];
        const size_t nb = (size_t)(v0.ny + 2) * v0.pitch;
        if (!h->stage_f) {
            TRY(dalloc(h, &h->stage_f, nb));
            TRY(dalloc(h, &h->stage_x, nb));
        }
        int n = enqueue_cycle(h, h->stage_f, h->stage_x, h->cap);
        CK(cudaStreamEndCapture(h->cap, &g));
        cudaGraphDestroy(g);
        h->kernels_per_cycle = n;
    }
    *count = h->kernels_per_cycle;
    return BMG_OK;
}

bmg_status_t bmg_export_level(bmg_solver_t h, int level, double *stencil_host, double *ci_host)
{
    if (!h || h->dist || level < 0 || level >= h->L || !stencil_host)
        return fail(BMG_EINVAL, "bad arguments to bmg_export_level");
    CK(cudaDeviceSynchronize());
    Level &v = h->lv[level];
    size_t w = (size_t)v.nx + 2, rows = (size_t)v.ny + 2;
    for (int k = 0; k < 5; k++) {
        double *dst = stencil_host + k * w * rows;
        if (v.pl[k])
            CK(cudaMemcpy2D(dst, w * sizeof(double), v.pl[k], v.pitch * sizeof(double), w * sizeof(double), rows,
                            cudaMemcpyDeviceToHost));
        else
            memset(dst, 0, w * rows * sizeof(double));
    }
    if (ci_host && level + 1 < h->L) {
        Level &c = h->lv[level + 1];
        size_t cw = (size_t)c.nx + 2, crows = (size_t)c.ny + 2;
        const int api_order[8] = {CI_LNE, CI_LA, CI_LNW, CI_LR, CI_LL, CI_LSE, CI_LB, CI_LSW};
        for (int k = 0; k < 8; k++)
            CK(cudaMemcpy2D(ci_host + k * cw * crows, cw * sizeof(double), v.ci[api_order[k]],
                            c.pitch * sizeof(double), cw * sizeof(double), crows, cudaMemcpyDeviceToHost));
    }
    return BMG_OK;
}

static bmg_status_t check_level(bmg_solver_t h, int level, bool need_coarse)
{
    if (!h || h->dist || level < 0 || level >= h->L || (need_coarse && level + 1 >= h->L))
        return fail(BMG_EINVAL, "bad level");
    return BMG_OK;
}

bmg_status_t bmg_relax(bmg_solver_t h, int level, const double *f, double *u, int nsweeps, void *cuda_stream)
{
    join_pcg(h, (cudaStream_t)cuda_stream);
    TRY(check_level(h, level, false));
    relax_level(h, level, f, u, nsweeps, (cudaStream_t)cuda_stream, nullptr);
    CK(cudaGetLastError());
    return BMG_OK;
}

bmg_status_t bmg_residual(bmg_solver_t h, int level, const double *f, const double *u, double *r, void *cuda_stream)
{
    join_pcg(h, (cudaStream_t)cuda_stream);
    TRY(check_level(h, level, false));
    launch_residual(h->lv[level].op(), f, u, r, (cudaStream_t)cuda_stream);
    CK(cudaGetLastError());
    return BMG_OK;
}

bmg_status_t bmg_restrict(bmg_solver_t h, int level, const double *r, double *fc, void *cuda_stream)
{
    join_pcg(h, (cudaStream_t)cuda_stream);
    TRY(check_level(h, level, true));
    launch_restrict(h->lv[level].op(), h->civ(level), r, fc, nullptr, (cudaStream_t)cuda_stream);
    CK(cudaGetLastError());
    return BMG_OK;
}

bmg_status_t bmg_interp_add(bmg_solver_t h, int level, const double *ec, double *u, void *cuda_stream)
{
    join_pcg(h, (cudaStream_t)cuda_stream);
    TRY(check_level(h, level, true));
    launch_interp_add(h->lv[level].op(), h->civ(level), ec, u, (cudaStream_t)cuda_stream);
    CK(cudaGetLastError());
    return BMG_OK;
}

bmg_status_t bmg_smooth_restrict(bmg_solver_t h, int level, const double *f, const double *u_in, double *u_out,
                                 double *fc, double *uc, void *cuda_stream)
{
    join_pcg(h, (cudaStream_t)cuda_stream);
    TRY(check_level(h, level, true));
    if (!f || !u_in || !u_out || !fc || u_in == u_out)
        return fail(BMG_EINVAL, "bmg_smooth_restrict: null pointer or u_in == u_out");
    int n = 0;
    enqueue_down(h, level, use_fused(h, level, f, u_in, u_out), f, u_in, u_out, fc, uc, (cudaStream_t)cuda_stream,
                 &n);
    CK(cudaGetLastError());
    return BMG_OK;
}

bmg_status_t bmg_correct_smooth(bmg_solver_t h, int level, const double *f, const double *u_in, const double *ec,
                                double *u_out, void *cuda_stream)
{
    join_pcg(h, (cudaStream_t)cuda_stream);
    TRY(check_level(h, level, true));
    if (!f || !u_in || !u_out || !ec || u_in == u_out)
        return fail(BMG_EINVAL, "bmg_correct_smooth: null pointer or u_in == u_out");
    int n = 0;
    enqueue_up(h, level, use_fused(h, level, f, u_in, u_out), f, u_in, ec, u_out, (cudaStream_t)cuda_stream, &n);
    CK(cudaGetLastError());
    return BMG_OK;
}

bmg_status_t bmg_partition(int nx, int ny, int nranks, const bmg_params_t *params, int *ybounds, int *kdist)
{
    bmg_status_t rc = dist_partition(nx, ny, nranks, params, ybounds, kdist);
    return rc == BMG_OK ? rc : fail(rc, "grid too small for this many slabs");
}

bmg_status_t bmg_setup_dist(const bmg_stencil_t *st, const bmg_comm_t *comm, const bmg_params_t *params,
                            void *cuda_stream, bmg_solver_t *out)
{
    if (!st || !comm || !out)
        return fail(BMG_EINVAL, "null argument to bmg_setup_dist");
    *out = nullptr;
    if (st->nx < 1 || st->ny < 1 || (st->kind != 5 && st->kind != 9) || st->pitch < (long long)st->nx + 2 ||
        comm->nranks < 1 || (!comm->loopback && (comm->rank < 0 || comm->rank >= comm->nranks)))
        return fail(BMG_EINVAL, "bad sizes or communicator");
    std::string err;
    DistSolver *d = nullptr;
    bmg_status_t rc = dist_setup(st, comm, params, (cudaStream_t)cuda_stream, &d, err);
    if (rc != BMG_OK)
        return fail(rc, err);
    bmg_solver *h = new bmg_solver();
    if (params)
        h->prm = *params;
    else
        bmg_params_default(&h->prm);
    h->dist = d;
    h->dist_inner = dist_inner_solver(d);
    int row0, nrows;
    dist_local_rows(d, &row0, &nrows, nullptr, nullptr, nullptr);
    h->dist_rows_total = comm->loopback ? (long long)(st->ny + 2) * st->pitch : (long long)nrows * st->pitch;
    h->dist_local_ranks = comm->loopback ? comm->nranks : 1;
    *out = h;
    return BMG_OK;
}

bmg_status_t bmg_local_rows(bmg_solver_t h, int *row0, int *nrows, int *ylo, int *yhi, int *kdist)
{
    if (!h)
        return fail(BMG_EINVAL, "null handle");
    if (h->dist) {
        dist_local_rows(h->dist, row0, nrows, ylo, yhi, kdist);
        return BMG_OK;
    }
    if (row0)
        *row0 = 0;
    if (nrows)
        *nrows = h->lv[0].ny + 2;
    if (ylo)
        *ylo = 1;
    if (yhi)
        *yhi = h->lv[0].ny + 1;
    if (kdist)
        *kdist = 0;
    return BMG_OK;
}

}  // extern "C"

