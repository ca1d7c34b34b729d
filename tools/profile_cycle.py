"""One V(2,1) cycle (NRHS=K: one block cycle) between cudaProfilerStart/Stop (for ncu --profile-from-start off)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2502_05279_b200 import bmg, problems as P

n = int(os.environ.get("N", "8191")); wl = os.environ.get("WL", "poisson")
st = P.workload(wl, n, n)
prm = bmg.bmg_params_default()
prm.relax = int(os.environ.get("RELAX", "0"))
s = bmg.Solver(st, prm)
K = int(os.environ.get("NRHS", "0"))  # > 0: the block multi-RHS cycle (c15) with K columns
if K:
    f = s.block_grid(K); f[1:-1, 1:n + 1, :] = 1.0 / (n + 1) ** 2; x = s.block_grid(K)
    run = lambda c: s.vcycle_block(f, x, c)  # noqa: E731
else:
    f = s.grid(P.rhs_const(n, n)); x = s.grid()
    run = lambda c: s.vcycle(f, x, c)  # noqa: E731
run(3)
torch.cuda.synchronize()
torch.cuda.profiler.start()
run(int(os.environ.get("NCYC", "1")))
torch.cuda.synchronize()
torch.cuda.profiler.stop()
