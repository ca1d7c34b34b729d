// solver.cuh -- the handle behind bmg_solver_t and the host-side helpers the
// ABI translation units share (abi.cu: setup, cycle, solve, PCG, single steps;
// abi_block.cu: the c15 block multi-RHS entry points).  Internal to libbmg.so.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <map>
#include <string>
#include <utility>
#include <vector>

#include "bmg.h"
#include "bmg_internal.cuh"
#include "dist.cuh"
#include "fused.cuh"

namespace bmg {

// the thread-local detail text of bmg_last_error_detail (defined in abi.cu)
std::string &abi_detail();

inline bmg_status_t fail(bmg_status_t s, const std::string &msg)
{
    abi_detail() = msg;
    return s;
}

inline bool al16(const void *p) { return ((uintptr_t)p & 15) == 0; }

}  // namespace bmg

#define CK(call)                                                                                    \
    do {                                                                                            \
        cudaError_t e_ = (call);                                                                    \
        if (e_ != cudaSuccess)                                                                      \
            return bmg::fail(e_ == cudaErrorMemoryAllocation ? BMG_ENOMEM : BMG_ECUDA,              \
                             std::string(#call) + ": " + cudaGetErrorString(e_));                   \
    } while (0)

#define TRY(x)                    \
    do {                          \
        bmg_status_t s_ = (x);    \
        if (s_ != BMG_OK)         \
            return s_;            \
    } while (0)

namespace bmg {

struct Level {
    int nx = 0, ny = 0, kind = 5;
    long long pitch = 0;
    double *pl[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};  // O W S SW NW
    double *u = nullptr, *f = nullptr, *r = nullptr;                // u,f unused on level 0
    double *ci[8] = {nullptr};                                       // weights from level l+1 (coarse pitch)
    Op op() const
    {
        Op A;
        A.nx = nx;
        A.ny = ny;
        A.kind = kind;
        A.pitch = pitch;
        A.O = pl[0];
        A.W = pl[1];
        A.S = pl[2];
        A.SW = pl[3];
        A.NW = pl[4];
        A.ylo = 1;
        A.yhi = ny + 1;
        A.roff = 0;
        A.nrows = ny + 2;
        return A;
    }
};


struct GraphRec {
    cudaGraphExec_t ex = nullptr;
    cudaGraph_t g = nullptr;                         // kept for the timed variant's node handles
    cudaGraphNode_t ev_node[2] = {nullptr, nullptr};  // event-record nodes (timed variant)
    void destroy()
    {
        if (ex)
            cudaGraphExecDestroy(ex);
        if (g)
            cudaGraphDestroy(g);
    }
};

}  // namespace bmg

using namespace bmg;

struct bmg_solver {
    bmg_params_t prm;
    int L = 0;
    std::vector<Level> lv;
    std::vector<void *> allocs;
    double *chol = nullptr;  // coarsest factor
    int nco = 0;
    int *d_err = nullptr;
    double *partials = nullptr, *d_norm = nullptr, *h_norm = nullptr;  // h_norm: a pinned slot (pinned_slot)
    cudaEvent_t setup_ev[2] = {nullptr, nullptr};  // around the S0-S3 kernels (bmg_setup_time)
    double *stage_f = nullptr, *stage_x = nullptr;                     // bmg_vcycle_host staging
    double *stage_f2 = nullptr, *stage_x2 = nullptr;                   // bmg_vcycle_host_batch: 2nd slot
    cudaStream_t hb_in = nullptr, hb_out = nullptr;                    // its copy streams
    cudaEvent_t hb_ev[6] = {};                                         // in/compute/out done per slot
    cudaStream_t cap = nullptr;                                        // capture stream
    std::map<std::pair<const void *, const void *>, GraphRec> graphs, tgraphs;  // plain / timed
    cudaEvent_t cev[2] = {nullptr, nullptr};  // placeholders captured into timed graphs
    int kernels_per_cycle = 0;
    FusedPlan fplan;
    DistSolver *dist = nullptr;  // row-slab distributed solver (bmg_setup_dist)
    bmg_solver_t dist_inner = nullptr;  // its replicated coarse solver (owned by dist)
    long long dist_rows_total = 0;      // doubles of a level-0 rhs/x array of this handle
    int dist_local_ranks = 1;
    double *line_scr = nullptr;       // c11 line relaxation scratch (line modes only)
    double *pcg_ws = nullptr;         // c13 PCG vectors r, z, p, q (level-0 arrays) + scalars, lazily
    cudaEvent_t pcg_ev = nullptr;     // marks the residual norm's arrival in h_norm
    cudaEvent_t pcg_tail = nullptr;   // end of the speculative work a returning bmg_pcg left queued
    bool pcg_pending = false;         // pcg_tail recorded and not yet joined by another entry point
    // device-side solve loop: per (rhs, x) a graph [WHILE: cycle, residual norm, k_solve_step]
    std::map<std::pair<const void *, const void *>, cudaGraphExec_t> sgraphs;
    SolveState *solve_st = nullptr;   // device state
    SolveState *solve_st_h = nullptr; // pinned staging
    double *solve_hist = nullptr;     // device history, solve_cap doubles
    int solve_cap = 0;
    int tail_l0 = 1 << 30;            // first level of the tail kernel (none: > L)
    bool tile[32] = {};               // level runs the shared-memory tile legs (kernels_tile.cu)
    TailPlan *tail = nullptr;         // its device-side plan
    int tail_sm = 0;                  // > 0: k_tail_sm with this many doubles of shared memory
    bool timing = false;              // bmg_timing: timed graph variant, event pair per launch
    bool cycle_err = false;           // a planned fused leg was rejected while enqueuing a cycle
    std::vector<cudaEvent_t> tev;     // event pairs (start, end) per recorded launch
    size_t tev_used = 0;
    // c15 block multi-RHS workspace (bmg_vcycle_block) for blk_K columns: per level
    // r (all but the coarsest), f and u (below level 0), K-interleaved, one arena
    int blk_K = 0;
    void *blk_arena = nullptr;
    std::vector<double *> blk_f, blk_u, blk_r;
    double *blk_partials = nullptr, *blk_norm = nullptr;
    std::map<std::pair<const void *, const void *>, cudaGraphExec_t> bgraphs;  // block cycle graphs (blk_K)
    double *pcgb_ws = nullptr;  // block PCG: r, z, p, q (K-interleaved level-0 arrays) + scalar slots
    int pcgb_K = 0;
    // device-side block solve loop (blk_K columns): graphs per (rhs, x), state, history
    std::map<std::pair<const void *, const void *>, cudaGraphExec_t> sbgraphs;
    SolveStateBlock *sb_st = nullptr, *sb_st_h = nullptr;
    double *sb_hist = nullptr;
    size_t sb_cap = 0;

    CIv civ(int l) const
    {
        CIv v;
        v.pitch = lv[l + 1].pitch;
        v.roff = 0;
        v.nrows = lv[l + 1].ny + 2;
        for (int k = 0; k < 8; k++)
            v.w[k] = lv[l].ci[k];
        return v;
    }
};

// A call on another stream must not overtake the speculative preconditioner
// V-cycle a returning bmg_pcg may have left queued (it writes the hierarchy
// arrays and the PCG workspace): every entry point that enqueues work joins it.
inline void join_pcg(bmg_solver *h, cudaStream_t s)
{
    if (h && h->pcg_pending) {
        cudaStreamWaitEvent(s, h->pcg_tail, 0);
        h->pcg_pending = false;
    }
}

double *pinned_slot();
void pinned_release(double *p);

inline bmg_status_t dalloc(bmg_solver *h, double **p, size_t n)
{
    void *q = nullptr;
    CK(cudaMalloc(&q, n * sizeof(double)));
    h->allocs.push_back(q);
    *p = (double *)q;
    return BMG_OK;
}


