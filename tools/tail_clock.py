"""Per-phase cycle stamps of the tail kernel (variant lib built with -DBMG_TAIL_CLOCK):
BMG_LIB=tools/vlib/libbmg_tclk.so python tools/tail_clock.py [wl n]"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2502_05279_b200 import bmg, problems as P

wl = sys.argv[1] if len(sys.argv) > 1 else "poisson"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 31
s = bmg.Solver(P.workload(wl, n, n))
f = s.grid(P.rhs_const(n, n)); u = s.grid()
for _ in range(5):
    s.vcycle(f, u, 1)
torch.cuda.synchronize()
buf = (ctypes.c_longlong * 256)()
k = bmg.lib().bmg_debug_tail_clock(buf)
t = np.array(buf[:k])
d = np.diff(t)
print(wl, n, "phases", len(d), "total cycles", t[-1] - t[0], "us@1.965GHz", (t[-1] - t[0]) / 1965)
print(" ".join(str(x) for x in d))
