// fused.cuh -- fused streaming ("wavefront temporal blocking") kernels for
// the large levels (kernels_fused.cu).  DESIGN.md §5.2.
//
// Down leg of a level in ONE pass over HBM: nu1 multicolour GS sweeps +
// residual + restriction (+ zeroing the coarse correction).  Up leg in ONE
// pass: interpolation + correction + nu2 sweeps.  Each CTA owns a strip of
// TX output columns and a chunk of rows and streams the rows bottom-up:
// tensor-map TMA boxes (u, f, one 3-D box of the operator's plane block, the
// weight planes) land in a staging ring; warp-specialised task groups (split,
// colour stages 2 rows apart, residual, restriction, store) each wait on ONE
// mbarrier ring per row step (their producers' step completions).  u is
// ping-ponged (u_in -> u_out) because neighbouring CTAs read each other's halo
// rows/columns.
#pragma once
#include "bmg.h"
#include "bmg_internal.cuh"

namespace bmg {

struct FusedGeom {
    int TX = 0;      // output columns per strip (multiple of 4)
    int H = 0;       // x halo (even)
    int WD = 0;      // smem row width = TX + 2H
    int WC = 0;      // smem coarse row width = TX/2 + 6
    int R = 0;       // fine ring rows
    int D = 0;       // fine-row prefetch distance (rows)
    int NS = 0;      // colour stages (2 per sweep)
    int nstrips = 0, nchunks = 0, chunk = 0;
    int threads = 0;
    size_t smem = 0;
    bool ok = false;
    bool rev = false;   // up leg: colours in reverse order (cycle_sym, c12)
};

struct LevelPlan {
    bool down = false, up = false;
    FusedGeom gd, gu;
};

struct FusedPlan {
    int nlev = 0;
    LevelPlan lv[32];
    double *tmp[32] = {nullptr};  // ping-pong partner of each fused level's u
};

// Decide per level whether the fused kernels run and with which geometry.
// rev: the up legs run the colours in reverse order (cycle_sym = 1, c12)
bmg_status_t fused_plan_level(FusedPlan &fp, int l, int nx, int ny, long long pitch, int kind, int nu1, int nu2,
                              bool aligned, bool rev = false);

// In-kernel ghost-row push (the row-slab solver's peer mode, dist.cu; SURVEY §8(e)
// lever 3): the leg's store task also writes each owned row within `halo` rows of the
// slab's lower / upper edge into the neighbour's copy of the output array (peer
// pointers, global-row indexed), and the restriction task likewise each coarse row of
// f_c within `halo` rows of the coarse slab's edges -- the ghost rows the neighbours'
// next legs read, moved by the kernel that produces them instead of a separate
// send/recv.  A null pointer: no neighbour on that side.
struct Push {
    double *lo = nullptr, *hi = nullptr;
    int ylo = 0, yhi = 0;
    double *clo = nullptr, *chi = nullptr;
    int cylo = 0, cyhi = 0;
    int halo = 0;
};

// Down leg of level l: nu1 sweeps on (f, uin) -> uout, fc = P^T(f - A uout), uc = 0 (if non-null).
// uin == nullptr: a zero start (the correction scheme's coarse levels, c9) that is not read.
// Returns false if level l is not fused.
bool fused_down(const FusedPlan &fp, int l, const Op &A, const CIv &ci, const double *f, const double *uin,
                double *uout, double *fc, double *uc, cudaStream_t s, int *nlaunch, const Push *push = nullptr);
// Up leg: uout = relax^nu2(uin + P ec).
// ec: coarse correction, global-row indexed, stored rows [eroff, eroff+enrows).
bool fused_up(const FusedPlan &fp, int l, const Op &A, const CIv &ci, const double *f, const double *uin,
              const double *ec, int eroff, int enrows, double *uout, cudaStream_t s, int *nlaunch,
              const Push *push = nullptr);

}  // namespace bmg
