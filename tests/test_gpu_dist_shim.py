"""The NCCL transport of the row-slab solver (csrc/dist.cu, NCCL mode: one rank per
PROCESS, rank-local slab arrays, grouped ncclSend/ncclRecv ghost-row exchange,
send/recv all-gather of the agglomerated level, ncclAllReduce of the norms) with
P = 2..4 ranks on ONE GPU.  Real NCCL refuses two ranks on one device, so the ranks
dlopen tests/ncclshim (a CUDA-IPC implementation of the NCCL entry points dist.cu
uses) through bmg_comm_t.nccl_lib; everything on the library side is the NCCL-mode
code path unchanged.

Checks: every rank's owned rows after two V(2,1) cycles are BITWISE equal to the
single-GPU solver's (same kernels, same per-point arithmetic), the
distributed residual norm agrees to 1e-12, and the distributed solve takes the
single-GPU solve's iteration count with the same history (1e-10) -- and against the
oracle's cycle at 1e-12 (normwise).
"""
import multiprocessing as mp
import os
import subprocess
import tempfile

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SHIM_SRC = os.path.join(ROOT, "tests", "ncclshim", "ncclshim.cu")
SHIM_LIB = os.path.join(ROOT, "tests", "ncclshim", "libncclshim.so")


def build_shim() -> str:
    if not os.path.exists(SHIM_LIB) or os.path.getmtime(SHIM_LIB) < os.path.getmtime(SHIM_SRC):
        import __graft_entry__ as ge

        tmp = SHIM_LIB + f".tmp{os.getpid()}"
        subprocess.check_call([ge._nvcc(), "-O2", "-std=c++17", "-Xcompiler", "-fPIC", "-shared",
                               "-Wno-deprecated-gpu-targets", "-I", ge._nccl_include(), SHIM_SRC, "-o", tmp])
        os.replace(tmp, SHIM_LIB)
    return SHIM_LIB


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__ as ge

    ge.build_lib()
    build_shim()


def _rank_main(rank, P, wl, n, agg, path, out_dir, q, peer=False):
    try:
        import ctypes
        import sys

        sys.path.insert(0, ROOT)
        import torch

        from paper_2502_05279_b200 import bmg, dist as D, problems as Pr

        torch.cuda.set_device(0)
        shim = ctypes.CDLL(SHIM_LIB)
        shim.shimCommInit.restype = ctypes.c_void_p
        shim.shimCommInit.argtypes = [ctypes.c_char_p, ctypes.c_int, ctypes.c_int, ctypes.c_longlong]
        comm = shim.shimCommInit(path.encode(), rank, P, 64 << 20)
        assert comm, "shimCommInit failed"
        st = Pr.workload(wl, n, n)
        prm = bmg.bmg_params_default()
        prm.agglom_rows = agg
        ds = D.DistSolver(st, P, rank, ctypes.c_void_p(comm), prm, pitch=bmg.default_pitch(n), nccl_lib=SHIM_LIB,
                          peer=peer)
        f = Pr.field_uniform(n, n, seed=91)
        x0 = Pr.field_uniform(n, n, seed=92)
        fl, xl = ds.local(f), ds.local(x0)
        ds.vcycle(fl, xl, 2)
        torch.cuda.synchronize()
        rn = ds.residual_norm(fl, xl)
        # the solve loop (host loop, all-reduced norms) from x = 0 on f = h^2
        fs = ds.local(Pr.rhs_const(n, n))
        xs = ds.local()
        it, hist, rc = bmg.bmg_solve(ds.h, fs, xs, 1e-9, 60)
        torch.cuda.synchronize()
        lo, hi = ds.ylo - ds.row0, ds.yhi - ds.row0
        np.save(os.path.join(out_dir, f"x{rank}.npy"), xl[lo:hi].cpu().numpy())
        np.save(os.path.join(out_dir, f"s{rank}.npy"), xs[lo:hi].cpu().numpy())
        q.put((rank, ds.ylo, ds.yhi, ds.kdist, rn, it, list(hist), rc, None))
        ds.close()
    except Exception as e:  # noqa: BLE001 -- reported to the parent
        import traceback

        q.put((rank, None, None, None, None, None, None, None, traceback.format_exc() + repr(e)))


def _shim_main(rank, P, path, q):
    """The shim alone: grouped send/recv of several messages to every peer + all-reduce."""
    try:
        import ctypes

        import torch

        torch.cuda.set_device(0)
        shim = ctypes.CDLL(SHIM_LIB)
        shim.shimCommInit.restype = ctypes.c_void_p
        shim.shimCommInit.argtypes = [ctypes.c_char_p, ctypes.c_int, ctypes.c_int, ctypes.c_longlong]
        comm = ctypes.c_void_p(shim.shimCommInit(path.encode(), rank, P, 1 << 20))
        assert comm.value, "shimCommInit failed"
        vp, sz = ctypes.c_void_p, ctypes.c_size_t
        shim.ncclSend.argtypes = [vp, sz, ctypes.c_int, ctypes.c_int, vp, vp]
        shim.ncclRecv.argtypes = [vp, sz, ctypes.c_int, ctypes.c_int, vp, vp]
        shim.ncclAllReduce.argtypes = [vp, vp, sz, ctypes.c_int, ctypes.c_int, vp, vp]
        NCCL_DOUBLE, NCCL_SUM = 8, 0
        stream = vp(torch.cuda.current_stream().cuda_stream)
        bad = []
        for rnd in range(3):
            send = {o: [torch.full((100 + 10 * m,), float(1000 * rank + 10 * o + m + rnd), dtype=torch.float64,
                                   device="cuda") for m in range(3)] for o in range(P) if o != rank}
            recv = {o: [torch.zeros(100 + 10 * m, dtype=torch.float64, device="cuda") for m in range(3)]
                    for o in range(P) if o != rank}
            assert shim.ncclGroupStart() == 0
            for m in range(3):
                for o in range(P):
                    if o == rank:
                        continue
                    assert shim.ncclRecv(vp(recv[o][m].data_ptr()), recv[o][m].numel(), NCCL_DOUBLE, o, comm, stream) == 0
                    assert shim.ncclSend(vp(send[o][m].data_ptr()), send[o][m].numel(), NCCL_DOUBLE, o, comm, stream) == 0
            assert shim.ncclGroupEnd() == 0
            torch.cuda.synchronize()
            for o in recv:
                for m in range(3):
                    want = float(1000 * o + 10 * rank + m + rnd)
                    if not bool((recv[o][m] == want).all()):
                        bad.append((rnd, o, m, float(recv[o][m][0]), want))
            a = torch.tensor([float(rank + 1), 2.0 * rank], dtype=torch.float64, device="cuda")
            b = torch.zeros(2, dtype=torch.float64, device="cuda")
            assert shim.ncclAllReduce(vp(a.data_ptr()), vp(b.data_ptr()), 2, NCCL_DOUBLE, NCCL_SUM, comm, stream) == 0
            torch.cuda.synchronize()
            if b.tolist() != [P * (P + 1) / 2, float(P * (P - 1))]:
                bad.append(("allreduce", b.tolist()))
        q.put((rank, bad))
    except Exception as e:  # noqa: BLE001
        import traceback

        q.put((rank, [traceback.format_exc() + repr(e)]))


@pytest.mark.parametrize("P", [2, 3])
def test_shim_itself(P):
    """The stand-in transport delivers grouped point-to-point messages in posting order
    and sums the all-reduce (so a failure below is the library's, not the shim's)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    with tempfile.TemporaryDirectory() as td:
        procs = [ctx.Process(target=_shim_main, args=(r, P, os.path.join(td, "shm"), q)) for r in range(P)]
        for p in procs:
            p.start()
        res = [q.get(timeout=300) for _ in range(P)]
        for p in procs:
            p.join(timeout=60)
    for rank, bad in res:
        assert not bad, (rank, bad[:3])


CASES = [("checker", 511, 2, 32), ("lognormal", 300, 3, 16), ("poisson", 1023, 4, 32), ("random9", 400, 2, 16)]


@pytest.mark.parametrize("peer", [False, True])
@pytest.mark.parametrize("wl,n,P,agg", CASES)
def test_nccl_mode_multi_rank(orc, wl, n, P, agg, peer):
    """peer = True: the in-kernel ghost-row stores into CUDA-IPC-mapped neighbour arrays and
    the system-scope signal/wait flags between processes (bmg_comm_t.peer)."""
    from paper_2502_05279_b200 import bmg, problems as Pr

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    with tempfile.TemporaryDirectory() as td:
        path = os.path.join(td, "shm")
        procs = [ctx.Process(target=_rank_main, args=(r, P, wl, n, agg, path, td, q, peer)) for r in range(P)]
        for p in procs:
            p.start()
        res = [q.get(timeout=600) for _ in range(P)]
        for p in procs:
            p.join(timeout=120)
        errs = [r[-1] for r in res if r[-1]]
        assert not errs, errs[0]
        res.sort()
        xs = [np.load(os.path.join(td, f"x{r}.npy")) for r in range(P)]
        ss = [np.load(os.path.join(td, f"s{r}.npy")) for r in range(P)]
    assert all(r[3] >= 1 for r in res)  # distributed levels exist
    # single-GPU reference (same inputs)
    st = Pr.workload(wl, n, n)
    prm = bmg.bmg_params_default()
    prm.agglom_rows = agg
    s = bmg.Solver(st, prm)
    f = Pr.field_uniform(n, n, seed=91)
    x0 = Pr.field_uniform(n, n, seed=92)
    x = s.grid(x0)
    fd = s.grid(f)
    s.vcycle(fd, x, 2)
    torch.cuda.synchronize()
    g = x.cpu().numpy()
    ns = s.residual_norm(fd, x)
    fs = s.grid(Pr.rhs_const(n, n))
    xsol = s.grid()
    it, hist, rc = s.solve(fs, xsol, 1e-9, 60)
    gs = xsol.cpu().numpy()
    s.close()
    for r, (rank, ylo, yhi, K, rn, itd, histd, rcd, _) in enumerate(res):
        assert np.array_equal(xs[r], g[ylo:yhi]), (rank, float(np.abs(xs[r] - g[ylo:yhi]).max()))
        assert abs(rn - ns) <= 1e-12 * ns
        assert itd == it and rcd == rc
        assert np.all(np.abs(np.array(histd) - hist) <= 1e-10 * hist + 1e-13 * hist[0])
        assert np.array_equal(ss[r], gs[ylo:yhi])
    # and the distributed iterate against the oracle
    o = orc.Hierarchy(st).vcycle(f, x0, 2)
    full = np.zeros_like(o)
    for r, (rank, ylo, yhi, *_rest) in enumerate(res):
        full[ylo:yhi] = xs[r][:, : n + 2]
    assert np.abs(full - o).max() <= 1e-12 * np.abs(o).max()
