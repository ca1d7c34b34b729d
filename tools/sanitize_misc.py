"""compute-sanitizer target: line relaxation (x/y/alternating, symmetric), the
row-slab solver (loopback, 3 slabs) and the affine variant on small odd grids."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2502_05279_b200 import bmg, dist as D, problems as P  # noqa: E402

for mode in (bmg.BMG_RELAX_XLINES, bmg.BMG_RELAX_YLINES, bmg.BMG_RELAX_ALTLINES):
    for sym in (0, 1):
        prm = bmg.bmg_params_default()
        prm.relax, prm.cycle_sym = mode, sym
        if sym:
            prm.nu1 = prm.nu2 = 1
        st = P.workload("aniso", 67, 45)
        s = bmg.Solver(st, prm)
        f, x = s.grid(P.rhs_const(67, 45)), s.grid()
        s.vcycle(f, x, 2)
        if sym:
            x.zero_()
            s.pcg(f, x, 1e-8, 10)
        s.close()
prm = bmg.bmg_params_default()
prm.affine = 1
s = bmg.Solver(P.workload("lognormal", 90, 77), prm)
f, x = s.grid(P.rhs_const(90, 77)), s.grid()
s.vcycle(f, x, 2)
s.close()
prm = bmg.bmg_params_default()
prm.agglom_rows = 16
st = P.workload("random9", 255, 255)
d = D.DistSolver(st, 3, 0, None, params=prm, loopback=True)
f, x = d.local(P.rhs_const(255, 255)), d.local()
d.vcycle(f, x, 2)
d.close()
torch.cuda.synchronize()
print("sanitize misc done", flush=True)
