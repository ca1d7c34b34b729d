// abi_block.cu -- the c15 block multi-RHS entry points of libbmg.so
// (include/bmg.h: bmg_vcycle_block, bmg_residual_norm_block, bmg_solve_block,
// bmg_pcg_block): workspace, the block cycle's graph, its solve loop and PCG.
#include <stdlib.h>
#include <string.h>

#include <string>
#include <vector>

#include "solver.cuh"

// The block workspace for K columns (reallocated when K changes; block graphs
// hold its pointers, so they go with it).
static bmg_status_t block_workspace(bmg_solver *h, int K, cudaStream_t s)
{
    if (h->blk_K == K)
        return BMG_OK;
    CK(cudaStreamSynchronize(s));
    CK(cudaDeviceSynchronize());
    for (auto &kv : h->bgraphs)
        cudaGraphExecDestroy(kv.second);
    h->bgraphs.clear();
    for (auto &kv : h->sbgraphs)
        cudaGraphExecDestroy(kv.second);
    h->sbgraphs.clear();
    if (h->blk_arena)
        cudaFree(h->blk_arena);
    h->blk_arena = nullptr;
    h->blk_K = 0;
    const int L = h->L;
    h->blk_f.assign(L, nullptr);
    h->blk_u.assign(L, nullptr);
    h->blk_r.assign(L, nullptr);
    size_t used = 0;
    double *arena = nullptr;
    auto take = [&](size_t n) {
        double *p = arena ? arena + used : nullptr;
        used += (n + 31) / 32 * 32;
        return p;
    };
    for (int pass = 0; pass < 2; pass++) {
        if (pass == 1) {
            CK(cudaMalloc(&h->blk_arena, used * sizeof(double)));
            arena = (double *)h->blk_arena;
            CK(cudaMemsetAsync(arena, 0, used * sizeof(double), s));
            used = 0;
        }
        for (int l = 0; l < L; l++) {
            const size_t np = (size_t)(h->lv[l].ny + 2) * (size_t)h->lv[l].pitch * (size_t)K;
            if (l + 1 < L)
                h->blk_r[l] = take(np);
            if (l > 0) {
                h->blk_f[l] = take(np);
                h->blk_u[l] = take(np);
            }
        }
        h->blk_partials = take((size_t)K * NORM_BLOCKS);
        h->blk_norm = take(K);
    }
    h->blk_K = K;
    return BMG_OK;
}

// One block V(nu1,nu2) cycle on s: the per-step path of enqueue_cycle (fused = 0)
// with every step's kernel in its K-column form.
static int enqueue_cycle_block(bmg_solver *h, int K, const double *f0, double *u0, cudaStream_t s)
{
    int n = 0;
    const int L = h->L;
    auto F = [&](int l) { return l == 0 ? f0 : (const double *)h->blk_f[l]; };
    auto U = [&](int l) { return l == 0 ? u0 : h->blk_u[l]; };
    // forward colour order, no affine term: kb_rb5 (5-point, one pass) / kb_r9pair (9-point,
    // two launches) sweeps, the
    // iterate ping-ponging between U(l) and blk_r[l] (r is never stored on this path)
    auto onepass = [&](int l) { return !h->prm.affine && h->prm.cycle_sym == 0; };
    std::vector<double *> cur(L);
    for (int l = 0; l + 1 < L; l++) {
        const Op A = h->lv[l].op();
        cur[l] = U(l);
        if (onepass(l)) {
            for (int sw = 0; sw < h->prm.nu1; sw++) {
                double *to = cur[l] == U(l) ? h->blk_r[l] : U(l);
                launch_rb5_block(K, A, F(l), cur[l], to, s);
                cur[l] = to;
                n += A.kind == 5 ? 1 : 2;
            }
        } else {
            launch_relax_block(K, A, F(l), U(l), h->prm.nu1, s, &n);
        }
        if (h->prm.nu1 > 0 && !h->prm.affine) {  // the vanishing restriction, residual fused in (r not stored)
            launch_resid_restrict_block(K, A, h->civ(l), F(l), cur[l], h->blk_f[l + 1], h->blk_u[l + 1], s);
            n += 1;
        } else {  // c14 needs r on the up leg; nu1 = 0 restricts every residual
            launch_residual_block(K, A, F(l), U(l), h->blk_r[l], s);
            launch_restrict_block(K, A, h->civ(l), h->blk_r[l], h->blk_f[l + 1], h->blk_u[l + 1], s, h->prm.nu1 > 0);
            n += 2;
        }
    }
    launch_coarse_solve_block(K, h->lv[L - 1].op(), h->chol, F(L - 1), U(L - 1), s);
    n += 1;
    for (int l = L - 2; l >= 0; l--) {
        const Op A = h->lv[l].op();
        // the post-smoother's first colour overwrites its points from their neighbours
        // alone: those need no correction (exact; DESIGN §5.2 / §5.7)
        const int skip = (h->prm.nu2 > 0 && !h->prm.affine) ? (h->prm.cycle_sym == 1 ? 2 : 1) : 0;
        if (onepass(l)) {
            // the corrected iterate goes where the nu2 sweeps then end in U(l); the points
            // the first colour overwrites are skipped (kb_rb5 never reads them from uin)
            double *start = (h->prm.nu2 % 2 == 0) ? U(l) : h->blk_r[l];
            if (h->prm.nu2 == 0 && cur[l] != U(l))
                start = U(l);
            launch_interp_add_block(K, A, h->civ(l), U(l + 1), cur[l], s, nullptr, h->prm.nu2 > 0 ? skip : 0,
                                    start);
            n += 1;
            double *it = start;
            for (int sw = 0; sw < h->prm.nu2; sw++) {
                double *to = it == U(l) ? h->blk_r[l] : U(l);
                launch_rb5_block(K, A, F(l), it, to, s);
                it = to;
                n += A.kind == 5 ? 1 : 2;
            }
            continue;
        }
        launch_interp_add_block(K, A, h->civ(l), U(l + 1), U(l), s, h->prm.affine ? h->blk_r[l] : nullptr, skip);
        n += 1;
        launch_relax_block(K, A, F(l), U(l), h->prm.nu2, s, &n, h->prm.cycle_sym == 1);
    }
    return n;
}

static bmg_status_t block_args(bmg_solver *h, int K, const void *rhs, const void *x, const char *who)
{
    if (!h || !rhs || !x || K < 1 || K > BMG_MAX_NRHS)
        return fail(BMG_EINVAL, std::string("bad arguments to ") + who + " (nrhs in 1.." +
                                    std::to_string(BMG_MAX_NRHS) + ")");
    if (h->dist)
        return fail(BMG_EINVAL, std::string(who) + ": single-GPU handles only");
    if (h->prm.relax != BMG_RELAX_POINT)
        return fail(BMG_EINVAL, std::string(who) + ": point relaxation only");
    if (K % 2 == 0 && (!al16(rhs) || !al16(x)))
        return fail(BMG_EINVAL, std::string(who) + ": rhs/x must be 16-byte aligned for even nrhs");
    return BMG_OK;
}

static bmg_status_t block_norms(bmg_solver *h, int K, const double *rhs, const double *x, double *out,
                                cudaStream_t s)
{
    if (x)
        launch_resid_norm_block(K, h->lv[0].op(), rhs, x, h->blk_partials, h->blk_norm, s);
    else
        launch_norm_block(K, h->lv[0].op(), rhs, h->blk_partials, h->blk_norm, s);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(h->h_norm, h->blk_norm, K * sizeof(double), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    memcpy(out, h->h_norm, K * sizeof(double));
    return BMG_OK;
}

extern "C" {

bmg_status_t bmg_vcycle_block(bmg_solver_t h, int nrhs, const double *rhs, double *x, int ncycles, void *cuda_stream)
{
    join_pcg(h, (cudaStream_t)cuda_stream);
    TRY(block_args(h, nrhs, rhs, x, "bmg_vcycle_block"));
    if (ncycles < 0)
        return fail(BMG_EINVAL, "bmg_vcycle_block: ncycles < 0");
    cudaStream_t s = (cudaStream_t)cuda_stream;
    TRY(block_workspace(h, nrhs, s));
    auto key = std::make_pair((const void *)rhs, (const void *)x);
    auto it = h->bgraphs.find(key);
    if (it == h->bgraphs.end()) {
        cudaGraph_t g;
        CK(cudaStreamBeginCapture(h->cap, cudaStreamCaptureModeThreadLocal));
        enqueue_cycle_block(h, nrhs, rhs, x, h->cap);
        cudaError_t e = cudaStreamEndCapture(h->cap, &g);
        if (e != cudaSuccess)
            return fail(BMG_ECUDA, std::string("block graph capture: ") + cudaGetErrorString(e));
        cudaGraphExec_t ex;
        e = cudaGraphInstantiate(&ex, g, 0);
        cudaGraphDestroy(g);
        if (e != cudaSuccess)
            return fail(BMG_ECUDA, std::string("block graph instantiate: ") + cudaGetErrorString(e));
        if (h->bgraphs.size() > 16) {
            for (auto &kv : h->bgraphs)
                cudaGraphExecDestroy(kv.second);
            h->bgraphs.clear();
        }
        it = h->bgraphs.emplace(key, ex).first;
    }
    for (int k = 0; k < ncycles; k++)
        CK(cudaGraphLaunch(it->second, s));
    return BMG_OK;
}

bmg_status_t bmg_residual_norm_block(bmg_solver_t h, int nrhs, const double *rhs, const double *x,
                                     double *norms_host, void *cuda_stream)
{
    join_pcg(h, (cudaStream_t)cuda_stream);
    TRY(block_args(h, nrhs, rhs, x, "bmg_residual_norm_block"));
    if (!norms_host)
        return fail(BMG_EINVAL, "bmg_residual_norm_block: null norms_host");
    cudaStream_t s = (cudaStream_t)cuda_stream;
    TRY(block_workspace(h, nrhs, s));
    return block_norms(h, nrhs, rhs, x, norms_host, s);
}

bmg_status_t bmg_solve_block(bmg_solver_t h, int nrhs, const double *rhs, double *x, double tol, int maxiter,
                             int *iters_out, double *hist_host, void *cuda_stream)
{
    join_pcg(h, (cudaStream_t)cuda_stream);
    TRY(block_args(h, nrhs, rhs, x, "bmg_solve_block"));
    if (maxiter < 0 || !(tol >= 0))
        return fail(BMG_EINVAL, "bad arguments to bmg_solve_block");
    cudaStream_t s = (cudaStream_t)cuda_stream;
    TRY(block_workspace(h, nrhs, s));
    if (iters_out)
        *iters_out = 0;
    const int K = nrhs;
    double fn[BMG_MAX_NRHS], rn[BMG_MAX_NRHS];
    TRY(block_norms(h, K, rhs, nullptr, fn, s));
    for (int c = 0; c < K; c++)
        if (fn[c] == 0.0)  // SPEC S:444 per column
            launch_zero_col_block(K, h->lv[0].op(), x, c, s);
    TRY(block_norms(h, K, rhs, x, rn, s));
    if (hist_host)
        memcpy(hist_host, rn, K * sizeof(double));
    auto done = [&]() {
        for (int c = 0; c < K; c++)
            if (rn[c] > tol * fn[c])
                return false;
        return true;
    };
    int k = 0;
    if (!done() && maxiter > 0) {  // device loop: one graph launch (as bmg_solve), one wait
        const size_t need = (size_t)(maxiter + 1) * K;
        if (h->sb_cap < need) {
            CK(cudaStreamSynchronize(s));
            for (auto &kv : h->sbgraphs)
                cudaGraphExecDestroy(kv.second);
            h->sbgraphs.clear();
            if (h->sb_hist)
                cudaFree(h->sb_hist);
            h->sb_hist = nullptr;
            h->sb_cap = 0;
            const size_t cap = need > 8192 ? need : 8192;
            void *q;
            CK(cudaMalloc(&q, sizeof(double) * cap + sizeof(SolveStateBlock) + 64));
            h->sb_hist = (double *)q;
            h->sb_cap = cap;
            h->sb_st = (SolveStateBlock *)(h->sb_hist + cap + 1);
            if (!h->sb_st_h)
                CK(cudaMallocHost(&h->sb_st_h, sizeof(SolveStateBlock)));
        }
        auto key = std::make_pair((const void *)rhs, (const void *)x);
        auto it = h->sbgraphs.find(key);
        if (it == h->sbgraphs.end()) {
            cudaGraph_t g;
            CK(cudaGraphCreate(&g, 0));
            cudaGraphConditionalHandle hd;
            CK(cudaGraphConditionalHandleCreate(&hd, g, 1, cudaGraphCondAssignDefault));
            cudaGraphNodeParams cp = {};
            cp.type = cudaGraphNodeTypeConditional;
            cp.conditional.handle = hd;
            cp.conditional.type = cudaGraphCondTypeWhile;
            cp.conditional.size = 1;
            cudaGraphNode_t node;
            CK(cudaGraphAddNode(&node, g, nullptr, 0, &cp));
            cudaGraph_t body = cp.conditional.phGraph_out[0];
            CK(cudaStreamBeginCaptureToGraph(h->cap, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
            enqueue_cycle_block(h, K, rhs, x, h->cap);
            launch_resid_norm_block(K, h->lv[0].op(), rhs, x, h->blk_partials, h->blk_norm, h->cap);
            launch_solve_step_block(hd, h->blk_norm, h->sb_st, h->sb_hist, h->cap);
            cudaError_t e = cudaStreamEndCapture(h->cap, &body);
            if (e == cudaSuccess) {
                cudaGraphExec_t ex;
                e = cudaGraphInstantiate(&ex, g, 0);
                if (e == cudaSuccess)
                    it = h->sbgraphs.emplace(key, ex).first;
            }
            cudaGraphDestroy(g);
            if (e != cudaSuccess)
                return fail(BMG_ECUDA, std::string("block solve graph: ") + cudaGetErrorString(e));
        }
        SolveStateBlock &st = *h->sb_st_h;
        for (int c = 0; c < K; c++)
            st.fn[c] = fn[c];
        st.tol = tol;
        st.k = 0;
        st.maxiter = maxiter;
        st.K = K;
        CK(cudaMemcpyAsync(h->sb_st, h->sb_st_h, sizeof(SolveStateBlock), cudaMemcpyHostToDevice, s));
        CK(cudaGraphLaunch(it->second, s));
        CK(cudaMemcpyAsync(h->sb_st_h, h->sb_st, sizeof(SolveStateBlock), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        k = h->sb_st_h->k;
        std::vector<double> hv((size_t)(k + 1) * K);
        CK(cudaMemcpy(hv.data(), h->sb_hist, sizeof(double) * hv.size(), cudaMemcpyDeviceToHost));
        for (int c = 0; c < K; c++)
            rn[c] = hv[(size_t)k * K + c];
        if (hist_host)
            memcpy(hist_host + K, hv.data() + K, sizeof(double) * (size_t)k * K);
    }
    if (iters_out)
        *iters_out = k;
    return done() ? BMG_OK : fail(BMG_ENOTCONV, "maxiter reached");
}

/*
 * Block PCG (c13 on every column of a c15 block): column c runs exactly the
 * recurrences of bmg_pcg on (rhs_c, x_c) -- alpha_c, beta_c from its own dot
 * products (device slots), the preconditioner the block V(nu,nu) cycle from
 * zero -- and stops updating once ||r_c|| <= tol ||rhs_c|| (its x_c and r_c are
 * then frozen: the column's result is its single-column PCG's).  The host
 * waits once per step for the K norms.
 */
bmg_status_t bmg_pcg_block(bmg_solver_t h, int nrhs, const double *rhs, double *x, double tol, int maxiter,
                           int *iters_out, double *hist_host, void *cuda_stream)
{
    join_pcg(h, (cudaStream_t)cuda_stream);
    TRY(block_args(h, nrhs, rhs, x, "bmg_pcg_block"));
    if (maxiter < 0 || !(tol >= 0))
        return fail(BMG_EINVAL, "bad arguments to bmg_pcg_block");
    if (h->prm.nu1 != h->prm.nu2 || h->prm.cycle_sym != 1)
        return fail(BMG_EINVAL, "bmg_pcg_block: the preconditioner must be symmetric (nu1 == nu2, cycle_sym = 1)");
    const int K = nrhs;
    cudaStream_t s = (cudaStream_t)cuda_stream;
    TRY(block_workspace(h, K, s));
    if (iters_out)
        *iters_out = 0;
    const Level &v = h->lv[0];
    const Op A = v.op();
    const size_t np = (size_t)(v.ny + 2) * (size_t)v.pitch * (size_t)K;
    if (h->pcgb_K != K) {
        CK(cudaStreamSynchronize(s));
        if (h->pcgb_ws)
            cudaFree(h->pcgb_ws);
        h->pcgb_ws = nullptr;
        h->pcgb_K = 0;
        void *q;
        CK(cudaMalloc(&q, sizeof(double) * (4 * np + 8 * BMG_MAX_NRHS)));
        h->pcgb_ws = (double *)q;
        CK(cudaMemsetAsync(q, 0, sizeof(double) * (4 * np + 8 * BMG_MAX_NRHS), s));
        h->pcgb_K = K;
    }
    double *r = h->pcgb_ws, *z = r + np, *p = z + np, *q = p + np, *sc = q + np;
    // scalar slots (K each): rho in slot 0 / 1 alternately, p.q in slot 2
    const int PQ = 2 * K;
    auto host_norms = [&](const double *src, double *out) -> bmg_status_t {
        CK(cudaMemcpyAsync(h->h_norm, src, K * sizeof(double), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        memcpy(out, h->h_norm, K * sizeof(double));
        return BMG_OK;
    };
    double fn[BMG_MAX_NRHS], rn[BMG_MAX_NRHS];
    launch_norm_block(K, A, rhs, h->blk_partials, h->blk_norm, s);
    TRY(host_norms(h->blk_norm, fn));
    for (int c = 0; c < K; c++)
        if (fn[c] == 0.0)  // SPEC S:444 per column
            launch_zero_col_block(K, A, x, c, s);
    launch_residual_block(K, A, rhs, x, r, s);  // r = f - A x0 (ring 0)
    launch_norm_block(K, A, r, h->blk_partials, h->blk_norm, s);
    TRY(host_norms(h->blk_norm, rn));
    if (hist_host)
        memcpy(hist_host, rn, K * sizeof(double));
    unsigned mask = 0;
    for (int c = 0; c < K; c++)
        if (rn[c] > tol * fn[c])
            mask |= 1u << c;
    int k = 0;
    if (mask && maxiter > 0) {
        auto precondition = [&]() -> bmg_status_t {  // z = one block V-cycle on r from z = 0
            launch_zero_block(K, A, z, s);
            return bmg_vcycle_block(h, K, r, z, 1, cuda_stream);
        };
        int cur = 0;
        TRY(precondition());
        CK(cudaMemcpyAsync(p, z, np * sizeof(double), cudaMemcpyDeviceToDevice, s));
        launch_dot_block(K, A, r, z, h->blk_partials, sc + cur * K, s);
        while (k < maxiter) {
            launch_matvec_block(K, A, p, q, s);
            launch_dot_block(K, A, p, q, h->blk_partials, sc + PQ, s);
            launch_cg_update_block(K, A, sc, cur * K, PQ, mask, p, q, x, r, s);  // alpha_c = rho_c / (p.q)_c
            k++;
            launch_norm_block(K, A, r, h->blk_partials, h->blk_norm, s);
            TRY(host_norms(h->blk_norm, rn));
            if (hist_host)
                memcpy(hist_host + (size_t)k * K, rn, K * sizeof(double));
            for (int c = 0; c < K; c++)
                if (rn[c] <= tol * fn[c])
                    mask &= ~(1u << c);
            if (!mask)
                break;
            const int nxt = 1 - cur;
            TRY(precondition());
            launch_dot_block(K, A, r, z, h->blk_partials, sc + nxt * K, s);
            launch_cg_direction_block(K, A, sc, nxt * K, cur * K, mask, z, p, s);  // beta_c = rho'_c / rho_c
            cur = nxt;
        }
    }
    CK(cudaGetLastError());
    if (iters_out)
        *iters_out = k;
    return mask == 0 ? BMG_OK : fail(BMG_ENOTCONV, "maxiter reached");
}

}  // extern "C"
