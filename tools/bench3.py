"""3-D BoxMG timing: V(2,1) cycles of a problems3d workload on one GPU,
CUDA-event timed graph replays; with PROFILE=1 one cycle between cudaProfilerStart/Stop
(for ncu --profile-from-start off).  usage: python tools/bench3.py WORKLOAD N [relax] [cycles]"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2502_05279_b200 import bmg3, problems3d as p3

wl, n = sys.argv[1], int(sys.argv[2])
relax = sys.argv[3] if len(sys.argv) > 3 else p3.WORKLOADS3[wl][1]
K = int(sys.argv[4]) if len(sys.argv) > 4 else 10
s = p3.WORKLOADS3[wl][0](n)
t0 = time.perf_counter()
S = bmg3.Solver3(s, relax=relax)
setup_ms = (time.perf_counter() - t0) * 1e3
f = S.grid(p3.rhs_const(n, n, n)); x = S.grid()
S.vcycle(f, x, 3); torch.cuda.synchronize()
if os.environ.get("PROFILE"):
    torch.cuda.profiler.start(); S.vcycle(f, x, 1); torch.cuda.synchronize(); torch.cuda.profiler.stop()
    sys.exit(0)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); S.vcycle(f, x, K); e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / K
x2 = S.grid()
t0 = time.perf_counter(); it, hist, rc = S.solve(f, x2, 1e-8, 100); solve_ms = (time.perf_counter() - t0) * 1e3
N = n ** 3
print(json.dumps({"workload": wl, "n": n, "relax": relax, "levels": S.L, "ms_per_cycle": ms,
                  "munknowns_per_s": N / ms / 1e3, "kernels_per_cycle": bmg3.bmg3_cycle_kernel_count(S.h),
                  "setup_ms": setup_ms, "solve_iters": it, "solve_ms": solve_ms,
                  "factor": float((hist[-1] / hist[0]) ** (1 / max(it, 1)))}))
