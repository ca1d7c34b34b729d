"""Micro-benchmark of the level-0 legs (bmg_smooth_restrict / bmg_correct_smooth)."""
import os, sys, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2502_05279_b200 import bmg, problems as P

n = int(os.environ.get("N", "8191"))
wl = os.environ.get("WL", "poisson")
legs = os.environ.get("LEGS", "down,up,cycle").split(",")
st = P.workload(wl, n, n)
s = bmg.Solver(st)
f = s.grid(P.rhs_const(n, n)); u = s.grid(); u2 = s.grid()
fc = s.level_grid(1); uc = s.level_grid(1)
def timeit(fn, rep=10):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); [fn() for _ in range(rep)]; e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / rep
out = {"lib": os.environ.get("BMG_LIB", "").split("/")[-1], "wl": wl, "n": n}
N = n * n
if "down" in legs:
    out["down_ms"] = timeit(lambda: bmg.bmg_smooth_restrict(s.h, 0, f, u, u2, fc, uc))
    out["down_GBps_68B"] = 68 * N / out["down_ms"] / 1e6
if "up" in legs:
    out["up_ms"] = timeit(lambda: bmg.bmg_correct_smooth(s.h, 0, f, u, uc, u2))
    out["up_GBps_66B"] = 66 * N / out["up_ms"] / 1e6
if "cycle" in legs:
    out["cycle_ms"] = timeit(lambda: s.vcycle(f, u, 1))
print(json.dumps(out))
