"""racecheck target: block cycle kernels only (per-step handle, no solve loop)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2502_05279_b200 import bmg, problems as P  # noqa: E402

prm = bmg.bmg_params_default()
prm.fused = 0
for wl, nx, ny, K in (("lognormal", 45, 38, 3), ("random9", 70, 33, 8)):
    s = bmg.Solver(P.workload(wl, nx, ny), prm)
    F = [P.field_uniform(nx, ny, seed=1 + c) for c in range(K)]
    fb, xb = s.block_grid(K, F), s.block_grid(K)
    s.vcycle_block(fb, xb, 1)
    torch.cuda.synchronize()
    s.close()
print("racecheck run done", flush=True)
