// kernels_fused.cu -- fused streaming kernels for large levels (placeholder: disabled).
#include "fused.cuh"

namespace bmg {

bmg_status_t fused_plan(FusedPlan &fp, int, int, long long, int, const bmg_params_t &)
{
    fp.nlev = 0;
    return BMG_OK;
}

bool fused_down(const FusedPlan &fp, int l, const Op &, const CIv &, const double *, double *, double *, double *,
                const Op &, int, cudaStream_t, int *)
{
    return l < fp.nlev && false;
}

bool fused_up(const FusedPlan &fp, int l, const Op &, const CIv &, const double *, double *, const double *, int,
              cudaStream_t, int *)
{
    return l < fp.nlev && false;
}

}  // namespace bmg
