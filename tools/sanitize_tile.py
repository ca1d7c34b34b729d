"""compute-sanitizer target (racecheck): the kernels synchronised by __syncthreads / named
barriers only -- the tile legs of the small levels, both tail kernels (a full cycle of a
hierarchy whose fused levels are skipped by the tile threshold) -- on small grids."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["BMG_TILE_POINTS"] = "1000000000"  # every level above the tail runs the tile legs
import torch  # noqa: E402

from paper_2502_05279_b200 import bmg, problems as P  # noqa: E402

for wl, n in [("aniso", 127), ("lognormal", 100)]:
    for sym in (0, 1):
        for tsm in ("1", "0"):
            os.environ["BMG_TAIL_SM"] = tsm
            prm = bmg.bmg_params_default()
            prm.cycle_sym = sym
            if sym:
                prm.nu1 = prm.nu2 = 1
            s = bmg.Solver(P.workload(wl, n, n), prm)
            f, x = s.grid(P.field_uniform(n, n, seed=1)), s.grid(P.field_uniform(n, n, seed=2))
            for l in range(bmg.bmg_num_levels(s.h) - 1):  # direct launches of each level's legs
                nx, ny, _ = bmg.bmg_level_shape(s.h, l)
                fl = s.level_grid(l, P.field_uniform(nx, ny, seed=4))
                u0 = s.level_grid(l, P.field_uniform(nx, ny, seed=5))
                uo = s.level_grid(l)
                fc, uc = s.level_grid(l + 1), s.level_grid(l + 1)
                ec = s.level_grid(l + 1, P.field_uniform(nx // 2, ny // 2, seed=6))
                bmg.bmg_smooth_restrict(s.h, l, fl, u0, uo, fc, uc)
                bmg.bmg_correct_smooth(s.h, l, fl, u0, ec, uo)
            s.vcycle(f, x, 1)  # the tail kernel (graph)
            torch.cuda.synchronize()
            s.close()
print("sanitize tile done", flush=True)
