#!/usr/bin/env python
"""Benchmark of the BoxMG V(2,1) cycle (BASELINE.json metric) on B200.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config NAME] [--impl reference]

A step is one V(2,1) cycle of the whole hot path (all levels, fine-level
relaxation through the coarsest Cholesky solve and back) on the N=1 workload
of BASELINE.json configs[3]: 2-D 5-point Poisson on 8193^2 (8191^2 interior
unknowns), f = h^2, x0 = 0.  Inputs (every level-0 array is 537 MB) are larger
than the 126 MB L2, so no explicit L2 flush is needed between steps.

Prints ONE JSON line on rank 0.  See DESIGN.md §8 for every field.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "V(2,1) cycles/s and Munknowns/s at 8193^2; HBM GB/s vs peak; 1/2/4/8 GPU"
CONFIG_KIND = {"aniso": 9}
# BASELINE config 3 solves to 1e-8; 1e-10 (configs 1, 2) is below the fp64 rounding
# floor of the residual at 4095^2 and 8191^2 with f = h^2 (measured floor ~6e-10 relative at 8191^2)
SOLVE_TOL = {"aniso4097": 1e-8, "checker4096": 1e-8, "poisson8193": 1e-8}
SOLVE_MAXIT = 100
TAIL_UNKNOWNS = 1024  # levels with at most this many unknowns run in the tail kernel

CONFIGS = {
    # name: (workload, nx, ny, description)
    "poisson33": ("poisson", 31, 31, "2D 5-point Poisson 33x33 (31^2 interior), Dirichlet, V(2,1) to 1e-10"),
    "poisson8193": ("poisson", 8191, 8191, "2D 5-point Poisson 8193^2 (8191^2 interior), V(2,1), f=h^2, x0=0"),
    "checker1025": ("checker", 1023, 1023, "2D 5-point 1e6 checkerboard (8x8 coarse-aligned blocks) 1025^2"),
    "aniso4097": ("aniso", 4095, 4095, "2D 9-point Q1 anisotropic eps=1e-3 4097^2"),
    "checker4096": ("checker512", 4095, 4095, "2D 5-point 512-cell 1e6 checkerboard 4096^2 per GPU"),
}


def l2_note(nx, ny):
    """Timing-rule statement: inputs larger than the 126 MB L2, or not (no flush is done)."""
    arr = (ny + 2) * ((nx + 2 + 31) // 32 * 32) * 8
    if arr > 126e6:
        return f"inputs > L2 (level-0 arrays {arr / 1e6:.0f} MB each); no flush needed"
    return (f"level-0 arrays {arr / 1e6:.1f} MB each: the working set can stay in the 126 MB L2 between "
            f"cycles (no flush; an L2-resident throughput, not an HBM one)")


def model_bytes(nx, ny, kind, L, fused_levels):
    """Algorithmic bytes per V(2,1) cycle.

    model B: (4s+19.5) N_l doubles per non-coarsest level; model A (two fused
    passes, CI stored): (2s+10.5) N_l.  s = 3 (5-pt level 0) or 5 (9-pt)."""
    B = A = 0.0
    for l in range(L - 1):
        s = 3 if (l == 0 and kind == 5) else 5
        N = float(nx) * float(ny)
        B += (4 * s + 19.5) * N * 8
        A += (2 * s + 10.5) * N * 8
        nx, ny = nx // 2, ny // 2
    return B, A


class ClockSampler:
    """nvidia-smi clocks/throttle sampling during the timed region (B200_PROFILING.md)."""

    FIELDS = ("timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.rows = []
        self.proc = None
        self.t0 = self.t1 = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._th = threading.Thread(target=self._read, daemon=True)
            self._th.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append((time.time(), [x.strip() for x in line.split(",")]))

    def mark(self, which):
        setattr(self, which, time.time())

    def stop(self):
        if self.proc is not None:
            time.sleep(0.12)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = [r for t, r in self.rows if self.t0 is not None and self.t0 - 0.06 <= t <= self.t1 + 0.06]
        if not rows:
            rows = [r for _, r in self.rows]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        import statistics

        def num(x):
            try:
                return float(x)
            except ValueError:
                return None

        sm = [num(r[1]) for r in rows if num(r[1]) is not None]
        mx = [num(r[2]) for r in rows if num(r[2]) is not None]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if len(r) > 4 + k and r[4 + k] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy burst)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def host_info():
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except Exception:
        pass
    return model, os.cpu_count()


# ------------------------------------------------------------------ oracle (CPU) legs
RELAX = {"point": 0, "xline": 1, "yline": 2, "altline": 3}


def oracle_cycles(wl, nx, ny, ncycles, warm=0, relax="point"):
    """Time the oracle's V(2,1) cycle on the FULL workload (same operator, f = h^2, x0 = 0;
    setup untimed): `warm` untimed cycles, then `ncycles` timed ones, single thread.
    Returns (cycles/s, seconds per cycle, setup seconds, sample string)."""
    import numpy as np

    import oracle
    from paper_2502_05279_b200 import problems as P

    st = P.workload(wl, nx, ny)
    f = P.rhs_const(nx, ny)
    t = time.perf_counter()
    h = oracle.Hierarchy(st, relax=relax)
    setup_s = time.perf_counter() - t
    del st
    u = np.zeros_like(f)
    if warm:
        u = h.vcycle(f, u, warm)
    t = time.perf_counter()
    u = h.vcycle(f, u, ncycles)
    dt = time.perf_counter() - t
    return ncycles / dt, dt / ncycles, setup_s, (f"oracle V(2,1) [{relax} relaxation] on the full {wl} {nx}x{ny} "
                                                 f"workload (f=h^2, x0=0), {ncycles} timed cycles after {warm} "
                                                 f"untimed, setup ({setup_s:.1f} s) untimed; single thread")


def run_reference(args, cfg):
    """--impl reference: the oracle (this tier's reference arm) on the same workload,
    K timed cycles after W untimed ones, rank 0 only (other ranks exit without work)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    wl, nx, ny, desc = CONFIGS[cfg]
    model, cores = host_info()
    val, per_cycle, setup_s, sample = oracle_cycles(wl, nx, ny, args.steps, warm=args.warmup, relax=args.relax)
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": "cycles/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": per_cycle * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": desc, "nx": nx, "ny": ny, "cycle": "V(2,1)", "relax": args.relax},
        "munknowns_per_s": val * nx * ny / 1e6,
        "cpu_baseline": {"value": val, "unit": "cycles/s", "cores": 1, "kind": "oracle", "sample": sample,
                         "host_cpu": model, "host_cores": cores, "setup_s": setup_s},
        "e2e": {"value": val, "unit": "cycles/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU leg
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    import bench3d

    ap.add_argument("--config", default="poisson8193", choices=sorted(CONFIGS) + sorted(bench3d.WORKLOAD3),
                    help="a BASELINE config, or a 3-D line (3d-*, SURVEY 8(f) row 4; bench3d.py)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--unfused", action="store_true", help="one kernel per method step (debug/comparison)")
    ap.add_argument("--dist", action="store_true", help="use the row-slab NCCL solver even on one GPU")
    ap.add_argument("--peer", action="store_true",
                    help="row slabs: ghost rows by in-kernel peer stores (bmg_comm_t.peer, CUDA IPC) instead of NCCL")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--relax", default="point", choices=sorted(RELAX),
                    help="relaxation: point GS (c6, default) or zebra line GS (c11)")
    ap.add_argument("--solve-tol", type=float, default=None, help="tolerance of the timed solve (default per config)")
    ap.add_argument("--pcg", type=int, default=0, metavar="NU",
                    help="also time V(NU,NU)-preconditioned CG (symmetric cycle, c12/c13) on the same problem")
    ap.add_argument("--nrhs", type=int, default=0, metavar="K",
                    help="also time the block multi-RHS cycle (c15, bmg_vcycle_block) with K right-hand sides")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.config in bench3d.WORKLOAD3:
        return bench3d.run3d(args, args.config, ClockSampler, measured_peaks, host_info)
    if args.impl == "reference":
        return run_reference(args, args.config)

    import torch

    from paper_2502_05279_b200 import bmg, problems as P

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    wl, nx, ny, desc = CONFIGS[args.config]
    st = P.workload(wl, nx, ny)
    prm = bmg.bmg_params_default()
    prm.fused = 0 if args.unfused else 1
    prm.relax = RELAX[args.relax]
    distributed = world > 1 or args.dist
    if distributed:
        # strong scaling (BASELINE config 4): one global problem in row slabs, NCCL ghost rows
        from paper_2502_05279_b200 import dist as D

        comm = D.nccl_comm(world, rank)
        solver = D.DistSolver(st, world, rank, comm, prm, peer=args.peer)
        f = solver.local(P.rhs_const(nx, ny))
        x = solver.local()
        parallelism = (f"{world} row slabs ({'in-kernel peer ghost-row stores' if args.peer else 'NCCL ghost-row exchange'}"
                       f", coarse levels all-gathered below level {solver.kdist})")
        scaling = "strong"
    else:
        # a throwaway setup + cycle on a small grid first, so that the timed setup
        # (solve.setup_ms) does not include the one-time lazy loading of the kernels
        # (1023^2: its level 0 plans the fused legs, whose first planning sets every fused
        # instance's attributes -- ~0.1 s of module loading measured inside a timed setup)
        wn = min(1023, nx, ny)
        warm = bmg.Solver(P.workload(wl, wn, wn), prm)
        wf = warm.grid(P.rhs_const(wn, wn))
        warm.vcycle(wf, warm.grid(), 1)
        torch.cuda.synchronize()
        warm.close()
        del warm, wf
        solver = bmg.Solver(st, prm)
        f = solver.grid(P.rhs_const(nx, ny))
        x = solver.grid()
        parallelism = "single GPU"
        scaling = "strong"  # the global problem is fixed; N GPUs split it
    del st
    L = bmg.bmg_num_levels(solver.h)
    kind = CONFIG_KIND.get(wl, 5)
    stream = torch.cuda.current_stream()

    # warm-up (untimed): builds and caches the CUDA graph(s)
    solver.vcycle(f, x, args.warmup)
    torch.cuda.synchronize()
    kpc = bmg.bmg_cycle_kernel_count(solver.h)

    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    if not distributed:
        # the timed cycles replay the cycle graph's variant with a CUDA event pair around
        # every level-0 down leg (the roofline kernel) on this stream; that variant is
        # captured and warmed here, outside the timed region, and its records cleared
        bmg.bmg_timing(solver.h, True)
        solver.vcycle(f, x, 1)
        bmg.bmg_timing_read(solver.h)
        torch.cuda.synchronize()
    clocks.mark("t0")
    ev0.record(stream)
    solver.vcycle(f, x, args.steps)
    ev1.record(stream)
    torch.cuda.synchronize()
    clocks.mark("t1")
    leg = None
    if not distributed:
        leg = bmg.bmg_timing_read(solver.h)
        bmg.bmg_timing(solver.h, False)
    if dist:
        dist.barrier()
    ms = ev0.elapsed_time(ev1)
    if dist:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    clocks.stop()
    ms_per_step = ms / args.steps
    # whole-job throughput: V-cycles of the global problem per second (strong scaling)
    cycles_per_s = args.steps / (ms / 1e3)

    peak, peak_src = measured_peaks()
    rl = None
    if not distributed:
        # roofline: the dominant kernel = level-0 down leg, launched alone through the ABI
        rl = roofline(leg, nx, ny, kind, peak, peak_src, ms_per_step, args)
        # for reference: the same cycles replayed as one CUDA graph each
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ng = max(10, args.steps // 4)
        torch.cuda.synchronize()
        g0.record(stream)
        solver.vcycle(f, x, ng)
        g1.record(stream)
        torch.cuda.synchronize()
        rl["graph_replay_ms_per_step"] = g0.elapsed_time(g1) / ng
        levels = per_level(bmg, solver, f, x, stream)
        cyc = cycle_traffic(nx, ny, args)
        if cyc is not None:
            rl["cycle_dram_bytes"] = cyc
            rl["cycle_dram_GBps"] = cyc / (ms_per_step / 1e3) / 1e9
            rl["cycle_dram_frac"] = rl["cycle_dram_GBps"] / peak
    else:
        levels = None

    # convergence sanity of the timed run (residual at the rounding floor after many cycles)
    rnorm = solver.residual_norm(f, x)
    fnorm = P.h_of(max(nx, ny)) ** 2 * (float(nx) * ny) ** 0.5

    # the solve loop (bmg_solve: V-cycles + residual norm per cycle, host-checked stopping
    # test) from x0 = 0, timed separately (SURVEY §8(d) "GPU timing")
    solve = None
    if not distributed:
        tol = args.solve_tol or SOLVE_TOL.get(args.config, 1e-10)
        xs = solver.grid()
        solver.solve(f, xs, tol, 2)  # warm-up: captures the device-side solve loop's graph for (f, xs)
        xs.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        it, hist, rc = solver.solve(f, xs, tol, SOLVE_MAXIT)
        dt = time.perf_counter() - t0
        k = len(hist) - 1
        solve = {"tol": tol, "iterations": it, "converged": rc == 0, "ms": dt * 1e3,
                 "final_rel_residual": float(hist[-1] / fnorm) if len(hist) else None,
                 "mean_factor": float((hist[-1] / hist[0]) ** (1.0 / k)) if k > 0 and hist[0] > 0 else None,
                 "last_factor": float(hist[-1] / hist[-2]) if k > 0 and hist[-2] > 0 else None,
                 "setup_ms": solver.setup_ms,
                 "setup_device_ms": bmg.bmg_setup_time(solver.h),
                 "note": "x0 = 0; ms = wall clock of bmg_solve (device-side loop: one graph launch whose conditional "
                         "WHILE node runs cycle + norm + stopping test; graph captured by an untimed warm-up solve); "
                         "setup_ms = wall clock of bmg_setup (S0-S3 + allocation, synchronised; kernels already loaded by a "
                         "warm-up setup on 255^2); setup_device_ms = device time of the S0-S3 kernels "
                         "(bmg_setup_time)"}
        del xs
        if args.pcg > 0:
            # V-cycle-preconditioned CG (bmg_pcg) with the symmetric V(NU,NU) cycle
            prm2 = bmg.bmg_params_default()
            prm2.nu1 = prm2.nu2 = args.pcg
            prm2.cycle_sym = 1
            prm2.relax = prm.relax
            s2 = bmg.Solver(P.workload(wl, nx, ny), prm2)
            f2 = s2.grid(P.rhs_const(nx, ny))
            x2 = s2.grid()
            s2.pcg(f2, x2, tol, 2)  # warm-up: workspace + graph
            x2.zero_()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            it2, h2, rc2 = s2.pcg(f2, x2, tol, SOLVE_MAXIT)
            dt2 = time.perf_counter() - t0
            solve["pcg"] = {"preconditioner": f"V({args.pcg},{args.pcg}) symmetric (cycle_sym=1)", "iterations": it2,
                            "converged": rc2 == 0, "ms": dt2 * 1e3,
                            "final_rel_residual": float(h2[-1] / fnorm) if len(h2) else None,
                            "setup_ms": s2.setup_ms}
            s2.close()
            del f2, x2

    # block multi-RHS (c15): K right-hand sides per cycle, every kernel
    # reading the operator / weights once for all K; device-timed block cycles from the
    # same rhs in every column, then a block solve from x0 = 0
    block = None
    if args.nrhs > 0 and not distributed and args.relax == "point":
        K = args.nrhs
        fb = solver.block_grid(K)
        fb.copy_(f.unsqueeze(-1).expand(-1, -1, K))
        xb = solver.block_grid(K)
        solver.vcycle_block(fb, xb, args.warmup)
        nb = max(10, args.steps // 4)
        b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        b0.record(stream)
        solver.vcycle_block(fb, xb, nb)
        b1.record(stream)
        torch.cuda.synchronize()
        bms = b0.elapsed_time(b1) / nb
        xb.zero_()
        solver.solve_block(fb, xb, 1e-3, 2)  # warm-up: captures the block solve loop's graph for (fb, xb)
        xb.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        itb, hb, rcb = solver.solve_block(fb, xb, args.solve_tol or SOLVE_TOL.get(args.config, 1e-10), SOLVE_MAXIT)
        dtb = time.perf_counter() - t0
        if args.pcg > 0:  # block PCG with the symmetric block V(NU,NU) cycle
            prm3 = bmg.bmg_params_default()
            prm3.nu1 = prm3.nu2 = args.pcg
            prm3.cycle_sym = 1
            s3 = bmg.Solver(P.workload(wl, nx, ny), prm3)
            fb3, xb3 = s3.block_grid(K), s3.block_grid(K)
            fb3.copy_(fb)
            s3.pcg_block(fb3, xb3, 1e-3, 2)  # warm-up: workspaces + block graph
            xb3.zero_()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            itp, hp, rcp = s3.pcg_block(fb3, xb3, args.solve_tol or SOLVE_TOL.get(args.config, 1e-10), SOLVE_MAXIT)
            pcg_block = {"preconditioner": f"block V({args.pcg},{args.pcg}) symmetric", "steps": itp,
                         "converged": rcp == 0, "ms": (time.perf_counter() - t0) * 1e3}
            s3.close()
            del fb3, xb3
        else:
            pcg_block = None
        block = {"nrhs": K, "ms_per_block_cycle": bms, "ms_per_rhs_cycle": bms / K,
                 "rhs_cycles_per_s": K * 1e3 / bms, "vs_single_rhs_cycle": ms_per_step / (bms / K),
                 "solve": {"steps": itb, "converged": rcb == 0, "ms": dtb * 1e3,
                           "final_rel_residual": float(hb[-1].max() / fnorm) if len(hb) else None},
                 "pcg": pcg_block,
                 "note": ("K columns interleaved per point; per-step block kernels (one read of the stencil and "
                          "weights per block), CUDA-graph replay, device-timed; vs_single_rhs_cycle = the "
                          "single-RHS cycle time of this line / the block cycle time per right-hand side")}
        del fb, xb
        torch.cuda.empty_cache()

    # e2e: the same metric through the public API with HOST buffers (pinned): per step
    # H2D of rhs and x, one V(2,1) cycle, D2H of x; host wall clock, max over ranks
    e2e = None
    if args.e2e_steps > 0:
        fh = f.cpu().pin_memory()
        xh = torch.zeros_like(fh).pin_memory()
        # one GPU: the steps are a batch of independent problems through
        # bmg_vcycle_host_batch (each step's rhs and x H2D, its cycle, its x D2H; the copies
        # of neighbouring steps overlap the cycle in between), two host x buffers alternating
        xh2 = torch.zeros_like(fh).pin_memory() if not distributed else None

        def e2e_step():
            if distributed:
                fd, xd = f, x
                fd.copy_(fh, non_blocking=True)
                xd.copy_(xh, non_blocking=True)
                solver.vcycle(fd, xd, 1)
                xh.copy_(xd, non_blocking=True)
                torch.cuda.current_stream().synchronize()
            else:
                bmg.bmg_vcycle_host(solver.h, fh, xh, 1)

        def e2e_batch(n):
            bmg.bmg_vcycle_host_batch(solver.h, [fh] * n, [(xh, xh2)[i & 1] for i in range(n)], 1)

        if distributed:
            e2e_step()
        else:
            e2e_batch(2)
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if distributed:
            for _ in range(args.e2e_steps):
                e2e_step()
        else:
            e2e_batch(args.e2e_steps)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        if dist:
            t = torch.tensor([dt], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt = float(t.item())
        nbytes = fh.numel() * 8
        e2e = {"value": args.e2e_steps / dt, "unit": "cycles/s", "h2d_bytes_per_step": 2 * nbytes * world,
               "d2h_bytes_per_step": nbytes * world,
               "note": ("per step: H2D rhs+x (pinned), 1 V(2,1) cycle, D2H x (1 GPU: the steps as one "
                        "bmg_vcycle_host_batch call -- each step's copies overlap the neighbouring steps' "
                        "cycles; otherwise torch copies + bmg_vcycle on the rank-local slabs, in series); "
                        "host wall clock")}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        # bounded: 2 full-size cycles (~7 s each at 8191^2 on the B200 host) after an untimed setup
        nc = 2 if nx * ny > 4e6 else (8 if nx * ny > 2e5 else 50)
        val, per_cycle, setup_s, sample = oracle_cycles(wl, nx, ny, nc, warm=0, relax=args.relax)
        model, cores = host_info()
        cpu = {"value": val, "unit": "cycles/s", "cores": 1, "kind": "oracle", "sample": sample,
               "host_cpu": model, "host_cores": cores, "setup_s": setup_s}

    B, A = model_bytes(nx, ny, kind, L, 0)
    cs = clocks.summary()
    line = {
        "metric": METRIC,
        "value": cycles_per_s,
        "unit": "cycles/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_per_step,
        "higher_is_better": True,
        "scaling": scaling,
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": desc, "nx": nx, "ny": ny, "levels": L, "cycle": "V(2,1)",
                   "parallelism": parallelism,
                   "l2": l2_note(nx, ny),
                   "fused": bool(prm.fused) and args.relax == "point", "relax": args.relax},
        "munknowns_per_s": cycles_per_s * nx * ny / 1e6,
        "model_B_GBps": B / (ms_per_step / 1e3) / 1e9,
        "model_B_frac": B / (ms_per_step / 1e3) / 1e9 / (peak * world),
        "model_A_frac": A / (ms_per_step / 1e3) / 1e9 / (peak * world),
        "final_rel_residual": rnorm / fnorm,
        "gpu_launches": kpc * args.steps,
        "kernels_per_cycle": kpc,
        "roofline": rl,
        "clocks": {"sm_mhz": cs["sm_mhz"], "sm_max_mhz": cs["sm_max_mhz"], "reasons": cs["reasons"],
                   "samples": cs["samples"]},
        "e2e": e2e,
        "solve": solve,
        "cpu_baseline": cpu,
    }
    if levels is not None:
        line["levels"] = levels
    if block is not None:
        line["block"] = block
    if rank == 0:
        print(json.dumps(line), flush=True)
    solver.close()
    if dist:
        dist.destroy_process_group()


def per_level(bmg, solver, f, x, stream, ncycles=10):
    """Per-leg device times of one cycle (bmg_profile_legs: an event between every two
    legs; the paper's per-level kernel timings, fig:kernel_timings P:492-500), measured
    after the timed region on the same arrays."""
    torch = sys.modules["torch"]
    down, tail, up = bmg.bmg_profile_legs(solver.h, f, x, ncycles, stream=stream.cuda_stream)
    torch.cuda.synchronize()
    out = {"legs": [], "tail_ms": tail, "tail_levels_from": len(down), "cycles_averaged": ncycles}
    for l in range(len(down)):
        lnx, lny, kind = bmg.bmg_level_shape(solver.h, l)
        out["legs"].append({"level": l, "nx": lnx, "ny": lny, "kind": kind, "down_ms": down[l], "up_ms": up[l]})
    out["sum_ms"] = sum(down) + sum(up) + tail
    return out


def cycle_traffic(nx, ny, args):
    """Sum of ncu dram read+write bytes over every kernel of one cycle at this size
    (profiles/traffic.json 'cycles' rows, from the committed launch list), or None."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as fh:
            rows = json.load(fh).get("cycles", [])
    except (OSError, ValueError):
        return None
    for r in rows:
        if r.get("nx") == nx and r.get("ny") == ny and r.get("relax", "point") == args.relax and \
                r.get("fused", True) == (not args.unfused):
            return r["dram_bytes_per_cycle"]
    return None


def traffic_per_launch(kernel: str, nx: int, ny: int):
    """dram__bytes_read.sum + dram__bytes_write.sum of one launch of `kernel` at this
    size, from the committed ncu --set full summary (profiles/traffic.json), or None."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "traffic.json")
    try:
        with open(path) as fh:
            rows = json.load(fh)["launches"]
    except (OSError, ValueError, KeyError):
        return None
    for r in rows:
        if r.get("kernel") == kernel and r.get("nx") == nx and r.get("ny") == ny:
            return r["dram_bytes_read"] + r["dram_bytes_write"]
    return None


def roofline(leg, nx, ny, kind, peak, peak_src, ms_per_step, args):
    """Dominant kernel: the level-0 down leg (one fused launch per cycle), timed by the
    library's event pairs inside the timed region.  Algorithmic bytes per launch =
    per-fine-unknown bytes x nx*ny."""
    ms_total, launches = leg
    dur_ms = ms_total / max(launches, 1)
    if nx * ny <= 4096:
        # the whole cycle is the single-CTA tail kernel: latency-bound, the
        # HBM roofline does not apply; report its share and duration only
        return {"bound": "latency", "kernel": "k_tail (every level in one CTA)", "achieved": None, "peak": None,
                "unit": "GB/s", "frac": None, "traffic": None, "launch_ms": dur_ms, "launches_timed": launches,
                "share_of_step": dur_ms / ms_per_step}
    s_planes = 3 if kind == 5 else 5
    # algorithmic bytes of the down leg per fine unknown = SURVEY §8(d) model A's
    # down-leg share: read u, f and the s operator planes, write u, read the
    # 2N-double CI planes of fig:restrict_kernel, write f_c and zero u_c (N/4 each).
    # The kernel itself reads only the half of the CI planes whose residual does not
    # vanish, so this is an effective bandwidth; `traffic` is the real one.
    # u_c: a fused coarse down leg never reads its zero start (C4), so the fused level-0
    # leg writes no u_c when level 1 is fused too (levels above the tail threshold)
    uc_written = args.unfused or args.relax != "point" or (nx // 2) * (ny // 2) <= TAIL_UNKNOWNS
    per_unk = 8.0 * (s_planes + 2 + 1 + 2 + 0.25 + (0.25 if uc_written else 0.0))
    if args.relax != "point":
        # per-step kernels: every line sweep direction reads the s planes, f and
        # u and writes u once ((s+3) doubles); then residual (s+3) and restriction (3.25)
        ndir = 2 if args.relax == "altline" else 1
        per_unk = 8.0 * (2 * ndir * (s_planes + 3) + (s_planes + 3) + 3.25)
    algo = per_unk * nx * ny
    achieved = algo / (dur_ms / 1e3) / 1e9
    kname = f"k_fused_down<{kind}, 4>" if not args.unfused and args.relax == "point" else None
    traffic = traffic_per_launch(kname, nx, ny) if kname else None
    what = ("nu1 GS sweeps + residual + restriction" if args.relax == "point" else
            f"nu1 {args.relax} GS sweeps (3 line kernels per colour) + residual + restriction")
    return {"bound": "hbm", "kernel": f"level-0 down leg (bmg_smooth_restrict: {what})", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
            "algorithmic_bytes_per_launch": algo, "algorithmic_bytes_per_unknown": per_unk,
            "launch_ms": dur_ms, "launches_timed": launches, "share_of_step": dur_ms / ms_per_step}


if __name__ == "__main__":
    main()
