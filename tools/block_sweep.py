"""Block multi-RHS throughput sweep (c15): ms per block cycle and per right-hand
side at N^2 for nrhs = 1, 2, 4, 8, against the single-RHS fused and per-step
cycles.  Device-timed with CUDA events (graph replays), inputs >> L2."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2502_05279_b200 import bmg, problems as P  # noqa: E402

N = int(os.environ.get("N", "8191"))
WL = os.environ.get("WL", "poisson")
KS = [int(k) for k in os.environ.get("KS", "1,2,4,8").split(",")]


def timed(fn, n=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


st = P.workload(WL, N, N)
out = {"n": N, "workload": WL}
for fused in (1, 0):
    prm = bmg.bmg_params_default()
    prm.fused = fused
    s = bmg.Solver(st, prm)
    f, x = s.grid(P.rhs_const(N, N)), s.grid()
    out["single_fused_ms" if fused else "single_perstep_ms"] = timed(lambda: s.vcycle(f, x, 1))
    if fused:
        for K in KS:
            fb = s.block_grid(K)
            fb[1:-1, 1:N + 1, :] = 1.0 / (N + 1) ** 2
            xb = s.block_grid(K)
            ms = timed(lambda: s.vcycle_block(fb, xb, 1))
            out[f"block{K}"] = {"ms_per_block_cycle": ms, "ms_per_rhs": ms / K}
            del fb, xb
            torch.cuda.empty_cache()
    s.close()
print(json.dumps(out))
