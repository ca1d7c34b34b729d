"""One V(2,1) cycle between cudaProfilerStart/Stop (for ncu --profile-from-start off)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch
from paper_2502_05279_b200 import bmg, problems as P

n = int(os.environ.get("N", "8191")); wl = os.environ.get("WL", "poisson")
st = P.workload(wl, n, n)
prm = bmg.bmg_params_default()
prm.relax = int(os.environ.get("RELAX", "0"))
s = bmg.Solver(st, prm)
f = s.grid(P.rhs_const(n, n)); x = s.grid()
s.vcycle(f, x, 3)
torch.cuda.synchronize()
torch.cuda.profiler.start()
s.vcycle(f, x, int(os.environ.get("NCYC", "1")))
torch.cuda.synchronize()
torch.cuda.profiler.stop()
