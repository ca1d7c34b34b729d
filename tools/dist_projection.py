"""Multi-GPU evidence on ONE GPU: the row-slab solver with the loopback
transport runs all P slabs of the 8191^2 problem on this GPU, one after another.

  T_lb(P)   = loopback cycle time (every slab's legs + the replicated inner cycle
              once + device-to-device ghost-row copies)
  T_inner   = the replicated inner hierarchy's cycle (a single-GPU solver on the
              level-K operator, measured on its own)
  slabs(P)  = T_lb(P) - T_inner  (all slabs' work, summed)

On P GPUs each rank runs its slab concurrently, so the per-cycle time is about
  T_P ~ slabs(P)/P * imbalance + T_inner + T_exch,
T_exch = 2K grouped NCCL ghost-row exchanges (8191^2, P=8: K levels; each a
one-row-per-neighbour send/recv over NVLink) + one all-gather of level K's rhs --
NOT measured here (one GPU); the printed projection takes them as a parameter.
Also the weak-scaling counterpart (BASELINE config 5: 4095 x 4096P-1 global, ~4096 rows
x nx per GPU): E = T(1) / T_P.  Prints one JSON line.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2502_05279_b200 import bmg, dist as D, problems as P  # noqa: E402

N = int(os.environ.get("N", "8191"))
EXCH_US = float(os.environ.get("EXCH_US", "25"))  # assumed latency of one grouped NCCL exchange
SIG_US = float(os.environ.get("SIG_US", "5"))  # assumed cost of one peer-mode signal + wait pair
AGGLOM = os.environ.get("AGGLOM")  # params.agglom_rows (default: the library's)


def time_cycles(fn, ncyc=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(ncyc):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / ncyc


st = P.workload("poisson", N, N)
f_np = P.rhs_const(N, N)
out = {"n": N, "exch_us_assumed": EXCH_US, "peer_sig_us_assumed": SIG_US}
prm = bmg.bmg_params_default()
if AGGLOM:
    prm.agglom_rows = int(AGGLOM)
out["agglom_rows"] = prm.agglom_rows
s = bmg.Solver(st)
f, x = s.grid(f_np), s.grid()
out["single_ms"] = time_cycles(lambda: s.vcycle(f, x, 1))
s.close()
for nr in (2, 4, 8):
    yb, K = bmg.bmg_partition(N, N, nr, prm)
    d = D.DistSolver(st, nr, 0, None, params=prm, loopback=True)
    f, x = d.local(f_np), d.local()
    t_lb = time_cycles(lambda: d.vcycle(f, x, 1))
    d.close()
    nK = N >> K
    si = bmg.Solver(P.workload("poisson", nK, nK))  # the replicated inner hierarchy
    fi, xi = si.grid(P.rhs_const(nK, nK)), si.grid()
    t_in = time_cycles(lambda: si.vcycle(fi, xi, 1))
    si.close()
    slabs = t_lb - t_in
    t_p = slabs / nr + t_in + (2 * K + 1) * EXCH_US / 1e3
    # peer mode (bmg_comm_t.peer): the legs store their ghost rows into the neighbours'
    # arrays themselves; left: the cycle-start level-0 exchange and the level-K all-gather
    # (NCCL) and one signal/wait pair per leg (2K)
    d = D.DistSolver(st, nr, 0, None, params=prm, loopback=True, peer=True)
    f, x = d.local(f_np), d.local()
    t_pe = time_cycles(lambda: d.vcycle(f, x, 1))
    d.close()
    slabs_pe = t_pe - t_in
    t_pp = slabs_pe / nr + t_in + 2 * EXCH_US / 1e3 + 2 * K * SIG_US / 1e3
    out[f"p{nr}"] = {"kdist": K, "loopback_ms": t_lb, "inner_ms": t_in, "slabs_ms": slabs,
                     "slab_overhead_vs_single": slabs / (out["single_ms"] - t_in) if out["single_ms"] > t_in else None,
                     "projected_ms": t_p, "projected_efficiency": out["single_ms"] / (nr * t_p),
                     "peer_loopback_ms": t_pe, "peer_projected_ms": t_pp,
                     "peer_projected_efficiency": out["single_ms"] / (nr * t_pp)}
# weak scaling (BASELINE config 5): ~4096 rows x nx per GPU, 512-cell 1e6 checkerboard
if os.environ.get("WEAK", "1") == "1":
    weak = {}
    t1 = None
    for nr, (gx, gy) in ((1, (4095, 4095)), (2, (4095, 8191)), (4, (8191, 8191)), (8, (8191, 16383))):
        stw = P.workload("checker512", gx, gy)
        fw = P.rhs_const(gx, gy)
        if nr == 1:
            s1 = bmg.Solver(stw)
            a, b = s1.grid(fw), s1.grid()
            t1 = time_cycles(lambda: s1.vcycle(a, b, 1))
            s1.close()
            weak["p1"] = {"global": [gx, gy], "single_ms": t1}
            continue
        yb, K = bmg.bmg_partition(gx, gy, nr, prm)
        d = D.DistSolver(stw, nr, 0, None, params=prm, loopback=True)
        a, b = d.local(fw), d.local()
        t_lb = time_cycles(lambda: d.vcycle(a, b, 1), ncyc=10)
        d.close()
        del d, a, b
        torch.cuda.empty_cache()
        ix, iy = gx >> K, gy >> K
        si = bmg.Solver(P.workload("checker512", ix, iy))
        fi, xi = si.grid(P.rhs_const(ix, iy)), si.grid()
        t_in = time_cycles(lambda: si.vcycle(fi, xi, 1))
        si.close()
        slabs = t_lb - t_in
        t_p = slabs / nr + t_in + (2 * K + 1) * EXCH_US / 1e3
        # peer mode, as for strong scaling above
        d = D.DistSolver(stw, nr, 0, None, params=prm, loopback=True, peer=True)
        a, b = d.local(fw), d.local()
        t_pe = time_cycles(lambda: d.vcycle(a, b, 1), ncyc=10)
        d.close()
        del d, a, b
        torch.cuda.empty_cache()
        t_pp = (t_pe - t_in) / nr + t_in + 2 * EXCH_US / 1e3 + 2 * K * SIG_US / 1e3
        weak[f"p{nr}"] = {"global": [gx, gy], "kdist": K, "loopback_ms": t_lb, "inner_ms": t_in,
                          "slabs_per_gpu_ms": slabs / nr, "projected_ms": t_p,
                          "projected_weak_efficiency": t1 / t_p, "peer_loopback_ms": t_pe,
                          "peer_projected_ms": t_pp, "peer_projected_weak_efficiency": t1 / t_pp}
    out["weak_config5"] = weak
print(json.dumps(out))
