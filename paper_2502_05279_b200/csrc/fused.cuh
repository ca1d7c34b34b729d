// fused.cuh -- fused streaming kernels for large levels (kernels_fused.cu).
#pragma once
#include "bmg.h"
#include "bmg_internal.cuh"

namespace bmg {

struct FusedPlan {
    int nlev = 0;          // levels [0, nlev) use the fused down/up kernels
};

bmg_status_t fused_plan(FusedPlan &fp, int nx, int ny, long long pitch, int kind, const bmg_params_t &prm);

// Down leg of level l: nu1 sweeps + residual + restriction (+ zero of the coarse u), one pass.
// Returns false if level l is not handled by the fused path.
bool fused_down(const FusedPlan &fp, int l, const Op &A, const CIv &ci, const double *f, double *u, double *fc,
                double *uc, const Op &Ac, int nu1, cudaStream_t s, int *nlaunch);
// Up leg of level l: interpolation + correction + nu2 sweeps, one pass.
bool fused_up(const FusedPlan &fp, int l, const Op &A, const CIv &ci, const double *f, double *u, const double *ec,
              int nu2, cudaStream_t s, int *nlaunch);

}  // namespace bmg
