"""3-D bench lines for bench.py --config 3d-<workload>-<n>.

A step is one V(2,1) cycle of the 3-D hot path (every level: the hierarchy's
smoother, residual, restriction, coarsest Cholesky, interpolation-correction)
on a problems3d workload, f = h^2, x0 = 0, replayed as the captured CUDA graph.
Not a BASELINE.json configuration (BASELINE's five are 2-D): these lines
measure the 3-D row to the same bar (parity in tests/test_gpu3d.py).

roofline: the dominant step of a cycle is the fine-level smoother sweep
(bmg3_relax), timed live with CUDA events on the launching stream, `sweeps`
sweeps between the events, against SURVEY §8(d)'s model B bytes of that sweep:
point GS (k3_rb7t): (s+3)*8 B per unknown with s = 4 stored planes (a_O, W,
S, B read once; u, f read, u written) = 56 B; zebra plane GS: the plane
right-hand side (f, u, B read, g written: 4 doubles) plus one 2-D V(1,1) per
plane -- on the in-plane 5-point level 2(s+3) + (s+3) + 3.25 + 4.25 = 25.5
doubles (s = 3), on the 9-point plane levels below 23.5 doubles per their
unknowns (N/4 + N/16 + ... = N/3: 7.8) -- = 37.3 doubles = 298 B per unknown.
"""
from __future__ import annotations

import json
import os
import time

import numpy as np

WORKLOAD3 = {
    # name: (problems3d workload, n, relax)
    "3d-poisson7-255": ("poisson7", 255, "point"),
    "3d-poisson7-511": ("poisson7", 511, "point"),
    "3d-aniso7-255": ("aniso7", 255, "planes"),
    "3d-checkeraniso7-255": ("checkeraniso7", 255, "planes"),
    "3d-checker27-255": ("checker27", 255, "point"),
}

METRIC3 = "3-D V(2,1) cycles/s and Munknowns/s (SURVEY 8(f) row 4); HBM GB/s vs peak"


def model_bytes3(n, kind0, L):
    """Model-B bytes per cycle: per non-coarsest level, 3 sweeps + residual (s+3)N each,
    restriction (1 + 26/8 + 1/8)N, interpolation (2 + 26/8 + 1/8)N doubles; s = 4 (7-pt) or 14."""
    B = 0.0
    for l in range(L - 1):
        s = 4 if (l == 0 and kind0 == 7) else 14
        N = float(n) ** 3
        B += (4 * (s + 3) + 4.375 + 5.375) * N * 8
        n //= 2
    return B


def oracle3_sample(wl, relax, n=63, ncycles=2):
    """The 3-D oracle (single thread) on a bounded sample: n^3 of the same workload,
    setup untimed, ncycles timed; returns (Munknowns/s, sample text)."""
    from oracle import oracle3d as o3
    from paper_2502_05279_b200 import problems3d as p3

    s = p3.WORKLOADS3[wl][0](n)
    t0 = time.perf_counter()
    H = o3.Hierarchy3(s, relax=relax)
    setup = time.perf_counter() - t0
    f = p3.rhs_const(n, n, n)
    x = np.zeros_like(f)
    t0 = time.perf_counter()
    H.vcycle(f, x, ncycles)
    dt = (time.perf_counter() - t0) / ncycles
    return n ** 3 / dt / 1e6, (f"oracle V(2,1) [{relax}] on {wl} {n}^3 (bounded sample of the same workload "
                               f"family), {ncycles} timed cycles after an untimed setup ({setup:.1f} s), "
                               f"single thread; value in Munknowns/s")


def run3d(args, name, clocks_cls, peaks, host_info):
    import torch

    from paper_2502_05279_b200 import bmg3, problems3d as p3

    wl, n, relax = WORKLOAD3[name]
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:  # replicas only: every rank solves its own copy, no collective on the data path
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if args.impl == "reference":
        if rank == 0:
            val, sample = oracle3_sample(wl, relax, n=min(n, 63), ncycles=max(1, args.steps))
            model, cores = host_info()
            print(json.dumps({"impl": "reference", "metric": METRIC3, "value": val, "unit": "Munknowns/s",
                              "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
                              "config": {"workload": f"{wl} {n}^3 ({relax} relaxation)"},
                              "cpu_baseline": {"value": val, "unit": "Munknowns/s", "cores": 1, "kind": "oracle",
                                               "sample": sample},
                              "e2e": {"value": val, "unit": "Munknowns/s", "h2d_bytes_per_step": 0,
                                      "d2h_bytes_per_step": 0}}), flush=True)
        return
    s = p3.WORKLOADS3[wl][0](n)
    bmg3.Solver3(p3.WORKLOADS3[wl][0](15), relax=relax).close()  # loads the kernels (not timed)
    S = bmg3.Solver3(s, relax=relax)
    setup_ms = S.setup_ms  # bmg3_setup wall clock (planes already on the device)
    f = S.grid(p3.rhs_const(n, n, n))
    x = S.grid()
    stream = torch.cuda.current_stream()
    S.vcycle(f, x, args.warmup)
    torch.cuda.synchronize()
    clocks = clocks_cls(local)
    clocks.start()
    time.sleep(0.2)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks.mark("t0")
    e0.record(stream)
    S.vcycle(f, x, args.steps)
    e1.record(stream)
    torch.cuda.synchronize()
    clocks.mark("t1")
    ms = e0.elapsed_time(e1) / args.steps
    if dist:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    # dominant kernel: the fine-level smoother sweep, timed live on the launching stream
    sweeps = 10
    y = S.grid()
    S.relax(f, y, 2)
    torch.cuda.synchronize()
    e0.record(stream)
    S.relax(f, y, sweeps)
    e1.record(stream)
    torch.cuda.synchronize()
    sweep_ms = e0.elapsed_time(e1) / sweeps
    clocks.stop()
    peak, peak_src = peaks()
    N = float(n) ** 3
    bpu = 56.0 if relax == "point" else 298.0
    alg = bpu * N
    L = S.L
    kpc = bmg3.bmg3_cycle_kernel_count(S.h)
    B = model_bytes3(n, s.kind, L)
    # solve to 1e-8
    x2 = S.grid()
    t0 = time.perf_counter()
    it, hist, rc = S.solve(f, x2, 1e-8, 100)
    solve_ms = (time.perf_counter() - t0) * 1e3
    # e2e: pinned host rhs/x -> device, one cycle, x -> host, host wall clock
    fh = torch.from_numpy(p3.rhs_const(n, n, n)).pin_memory()
    xh = torch.zeros_like(fh).pin_memory()
    fd, xd = S.grid(), S.grid()
    nb = fh.numel() * 8
    e2e_steps = max(1, min(args.e2e_steps, 5))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        fd[:, :, : n + 2].copy_(fh, non_blocking=True)
        xd[:, :, : n + 2].copy_(xh, non_blocking=True)
        S.vcycle(fd, xd, 1)
        xh.copy_(xd[:, :, : n + 2], non_blocking=True)
    torch.cuda.synchronize()
    e2e_dt = time.perf_counter() - t0
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        val, sample = oracle3_sample(wl, relax)
        model, cores = host_info()
        cpu = {"value": val, "unit": "Munknowns/s", "cores": 1, "kind": "oracle", "sample": sample,
               "host_cpu": model, "host_cores": cores}
    cs = clocks.summary()
    line = {
        "metric": METRIC3,
        "value": world * 1e3 / ms,
        "unit": "cycles/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": f"3-D {p3.WORKLOADS3[wl][2]}, {n}^3 interior, V(2,1) [{relax} relaxation], "
                               f"f=h^2, x0=0", "n": n, "kind": s.kind, "levels": L, "relax": relax,
                   "parallelism": "single GPU" if world == 1 else f"{world} independent replicas (no collective)",
                   "l2": f"level-0 arrays {(n + 2) ** 2 * S.pitch * 8 / 1e6:.0f} MB each (> L2 at n >= 255); "
                         "no flush"},
        "munknowns_per_s": world * N / ms / 1e3,
        "model_B_GBps": world * B / (ms / 1e3) / 1e9,
        "model_B_frac": B / (ms / 1e3) / 1e9 / peak,
        "gpu_launches": kpc * args.steps,
        "kernels_per_cycle": kpc,
        "roofline": {"bound": "hbm", "kernel": f"fine-level {relax} GS sweep (bmg3_relax)",
                     "achieved": alg / (sweep_ms / 1e3) / 1e9, "peak": peak, "unit": "GB/s",
                     "frac": alg / (sweep_ms / 1e3) / 1e9 / peak, "traffic": None,
                     "algorithmic_bytes_per_unknown": bpu, "sweep_ms": sweep_ms,
                     "share_of_step": 3 * sweep_ms / ms, "peak_source": peak_src},
        "clocks": {"sm_mhz": cs["sm_mhz"], "sm_max_mhz": cs["sm_max_mhz"], "reasons": cs["reasons"],
                   "samples": cs["samples"]},
        "e2e": {"value": world * e2e_steps / e2e_dt, "unit": "cycles/s", "h2d_bytes_per_step": 2 * nb,
                "d2h_bytes_per_step": nb, "note": "pinned host rhs/x copied in, 1 cycle (bmg3_vcycle), x copied "
                                                   "out; host wall clock"},
        "solve": {"tol": 1e-8, "iterations": it, "converged": rc == 0, "ms": solve_ms,
                  "mean_factor": float((hist[-1] / hist[0]) ** (1.0 / max(it, 1))), "setup_ms": setup_ms,
                  "note": "setup_ms = bmg3_setup wall clock (allocation + S0-S3 + plane hierarchies, "
                          "synchronised; planes already on the device, kernels loaded by a 15^3 warm-up)"},
        "cpu_baseline": cpu,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    S.close()
    if dist:
        dist.destroy_process_group()
