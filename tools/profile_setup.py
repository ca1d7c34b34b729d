"""bmg_setup wall clock, repeated (first call pays allocation / module load), for ncu."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2502_05279_b200 import bmg, problems as P

n = int(os.environ.get("N", "8191")); wl = os.environ.get("WL", "poisson")
st = P.workload(wl, n, n)
planes = [bmg.to_device(p, bmg.default_pitch(n)) for p in st.plane_list()]
torch.cuda.synchronize()
for k in range(3):
    t = time.perf_counter()
    h = bmg.bmg_setup(planes, st.kind, n, n, bmg.default_pitch(n))
    dt = time.perf_counter() - t
    print(f"setup {k}: {dt * 1e3:.2f} ms", flush=True)
    bmg.bmg_destroy(h)
