"""compute-sanitizer target: the fused streaming legs (5- and 9-point, down and up, forward
and REV), the tile legs and both tail kernels, launched DIRECTLY (no CUDA graph: racecheck
and synccheck track direct launches) on small grids.  MODE=legs|cycle."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2502_05279_b200 import bmg, problems as P  # noqa: E402

for wl, nx, ny in [("lognormal", 300, 257), ("random9", 200, 131)]:
    for sym in (0, 1):
        prm = bmg.bmg_params_default()
        prm.cycle_sym = sym
        if sym:
            prm.nu1 = prm.nu2 = 1
        st = P.workload(wl, nx, ny)
        s = bmg.Solver(st, prm)
        f = s.grid(P.field_uniform(nx, ny, seed=1))
        u0 = s.grid(P.field_uniform(nx, ny, seed=2))
        uo = s.grid()
        fc, uc = s.level_grid(1), s.level_grid(1)
        ec = s.level_grid(1, P.field_uniform(nx // 2, ny // 2, seed=3))
        # level-0 legs through the single-leg ABI: direct launches of k_fused_down / k_fused_up
        bmg.bmg_smooth_restrict(s.h, 0, f, u0, uo, fc, uc)
        bmg.bmg_correct_smooth(s.h, 0, f, u0, ec, uo)
        torch.cuda.synchronize()
        s.close()
# a small hierarchy whose levels run the tile legs and the shared-memory tail (direct launches
# through the single-leg ABI on each level)
os.environ["BMG_TILE_POINTS"] = "70000"
st = P.workload("aniso", 255, 255)
s = bmg.Solver(st)
for l in range(bmg.bmg_num_levels(s.h) - 1):
    nx, ny, _ = bmg.bmg_level_shape(s.h, l)
    f = s.level_grid(l, P.field_uniform(nx, ny, seed=4))
    u0 = s.level_grid(l, P.field_uniform(nx, ny, seed=5))
    uo = s.level_grid(l)
    fc, uc = s.level_grid(l + 1), s.level_grid(l + 1)
    ec = s.level_grid(l + 1, P.field_uniform(nx // 2, ny // 2, seed=6))
    bmg.bmg_smooth_restrict(s.h, l, f, u0, uo, fc, uc)
    bmg.bmg_correct_smooth(s.h, l, f, u0, ec, uo)
torch.cuda.synchronize()
s.close()
print("sanitize fused done", flush=True)
