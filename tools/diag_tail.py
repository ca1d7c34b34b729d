import sys, numpy as np
sys.path.insert(0, '.')
from tests.test_gpu_tail import _cycle, CASES
import torch
for wl, nx, ny in CASES:
    for nu1, nu2, sym, aff in [(2, 1, 0, 0), (1, 1, 1, 0)]:
        a = _cycle(wl, nx, ny, 1, nu1, nu2, sym, aff)
        b = _cycle(wl, nx, ny, 0, nu1, nu2, sym, aff)
        c = _cycle(wl, nx, ny, 1, nu1, nu2, sym, aff, tail_sm=False)
        print(wl, nx, ny, nu1, nu2, sym, "sm-vs-step", np.abs(a - b).max(), "old-vs-step", np.abs(c - b).max(), "sm-vs-old", np.abs(a-c).max(), flush=True)
