"""compute-sanitizer target: the 3-D path (setup kernels, k3_rb7, the colour-major 27-point
sweeps, transfers, plane relaxation incl. the plane tail) on small grids.  bmg3_relax and
setup launch directly (racecheck/synccheck track those); the cycle replays its graph."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2502_05279_b200 import bmg3, problems3d as p3  # noqa: E402

for wl, shape, relax in [("poisson7", (33, 29, 35), "point"), ("checker27", (15, 15, 15), "point"),
                         ("aniso7", (31, 31, 31), "planes"), ("checker27", (20, 17, 26), "planes")]:
    nx, ny, nz = shape
    s = p3.fv7(p3.d3_lognormal(nx, ny, nz)) if wl == "poisson7" else (
        p3.q1_27(p3.d3_checkerboard(nx, ny, nz, 4, 1e4)) if wl == "checker27" else p3.fv7(p3.d3_constant(nx, ny, nz), az=1e-3))
    S = bmg3.Solver3(s, relax=relax)
    f = S.grid(p3.random_interior(nx, ny, nz, seed=1))
    x = S.grid(p3.random_interior(nx, ny, nz, seed=2))
    S.relax(f, x, 3)
    S.vcycle(f, x, 1)
    torch.cuda.synchronize()
    S.close()
print("sanitize3d done")
