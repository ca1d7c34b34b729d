// dist.cuh -- row-slab distributed solver (dist.cu), used by abi.cu.
#pragma once
#include <string>

#include "bmg.h"

namespace bmg {

struct DistSolver;

bmg_status_t dist_partition(int nx, int ny, int nranks, const bmg_params_t *prm, int *ybounds, int *kdist);
bmg_status_t dist_setup(const bmg_stencil_t *st, const bmg_comm_t *cm, const bmg_params_t *prm, cudaStream_t s,
                        DistSolver **out, std::string &err);
void dist_destroy(DistSolver *d);
bmg_solver_t dist_inner_solver(DistSolver *d);
void dist_local_rows(DistSolver *d, int *row0, int *nrows, int *ylo, int *yhi, int *kdist);
bmg_status_t dist_vcycle(DistSolver *d, const double *rhs, double *x, int ncycles, cudaStream_t s, std::string &err);
bmg_status_t dist_resid_norm(DistSolver *d, const double *rhs, const double *x, double *norm, cudaStream_t s,
                             std::string &err);

}  // namespace bmg
