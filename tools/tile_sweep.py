"""Cycle time vs the tile-leg threshold (BMG_TILE_POINTS, read at each bmg_setup)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2502_05279_b200 import bmg, problems as P

for wl, n in [("poisson", 8191), ("checker", 1023), ("aniso", 4095), ("poisson", 31), ("poisson", 255)]:
    st = P.workload(wl, n, n)
    for lim in [0, 5000, 20000, 70000, 300000, 1100000]:
        os.environ["BMG_TILE_POINTS"] = str(lim)
        s = bmg.Solver(st)
        f = s.grid(P.rhs_const(n, n)); x = s.grid()
        s.vcycle(f, x, 5); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 20 if n > 2000 else 200
        e0.record(); s.vcycle(f, x, reps); e1.record(); torch.cuda.synchronize()
        down, tail, up = bmg.bmg_profile_legs(s.h, f, x, 5)
        print(json.dumps({"wl": wl, "n": n, "tile_points": lim, "cycle_ms": e0.elapsed_time(e1) / reps,
                          "down": [round(v, 4) for v in down], "up": [round(v, 4) for v in up], "tail": round(tail, 4)}),
              flush=True)
        s.close()
