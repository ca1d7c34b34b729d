"""compute-sanitizer target: the block multi-RHS cycle / solve / PCG, the device
solve loop and PCG on small odd-sized problems (out-of-bounds / race checks)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2502_05279_b200 import bmg, problems as P  # noqa: E402

for wl, nx, ny, K in (("lognormal", 45, 38, 3), ("random9", 70, 33, 8), ("checker_off3", 95, 47, 2)):
    st = P.workload(wl, nx, ny)
    s = bmg.Solver(st)
    F = [P.field_uniform(nx, ny, seed=1 + c) for c in range(K)]
    fb, xb = s.block_grid(K, F), s.block_grid(K)
    s.vcycle_block(fb, xb, 2)
    xb.zero_()
    s.solve_block(fb, xb, 1e-8, 20)
    f, x = s.grid(F[0]), s.grid()
    s.solve(f, x, 1e-8, 20)
    s.close()
    prm = bmg.bmg_params_default()
    prm.nu1, prm.nu2, prm.cycle_sym = 1, 1, 1
    s = bmg.Solver(st, prm)
    fb, xb = s.block_grid(K, F), s.block_grid(K)
    s.pcg_block(fb, xb, 1e-8, 20)
    f, x = s.grid(F[0]), s.grid()
    s.pcg(f, x, 1e-8, 20)
    s.close()
torch.cuda.synchronize()
print("sanitize run done")
