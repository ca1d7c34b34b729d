"""Multi-GPU path on ONE GPU through the loopback transport:
P row slabs in this process, ghost rows exchanged device-to-device with the
same schedule the NCCL path uses, the coarse levels all-gathered and solved by
the replicated inner solver.  The distributed iterate must be BITWISE equal
to the single-GPU iterate (same kernels, same per-point arithmetic), norms
within 1e-12 relative (different reduction trees)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from paper_2502_05279_b200 import bmg, problems as P  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__ as ge

    ge.build_lib()


def loopback(st, nranks, prm, pitch, peer=0):
    planes = [bmg.to_device(p, pitch) for p in st.plane_list()]
    comm = bmg.bmg_comm_t()
    comm.nranks, comm.rank, comm.nccl_comm, comm.nccl_lib, comm.loopback = nranks, 0, None, None, 1
    comm.peer = peer
    h = bmg.bmg_setup_dist(planes, st.kind, st.nx, st.ny, pitch, comm, prm)
    return h


CASES = [("checker_off3", 255, 2, 16), ("lognormal", 300, 2, 16), ("poisson", 511, 4, 16), ("checker", 511, 3, 32),
         ("aniso", 255, 2, 16), ("lognormal", 300, 3, 16), ("random9", 400, 5, 16), ("poisson", 1023, 8, 32)]


@pytest.mark.parametrize("peer", [0, 1])
@pytest.mark.parametrize("wl,n,nranks,agg", CASES)
def test_loopback_bitwise_vcycle(wl, n, nranks, agg, peer):
    """peer = 1: the ghost rows move by the fused legs' in-kernel stores into the
    neighbouring slabs (bmg_comm_t.peer) instead of the exchange copies."""
    st = P.workload(wl, n, n)
    prm = bmg.bmg_params_default()
    prm.agglom_rows = agg
    single = bmg.Solver(st, prm)
    pitch = single.pitch
    h = loopback(st, nranks, prm, pitch, peer)
    row0, nrows, ylo, yhi, K = bmg.bmg_local_rows(h)
    assert K >= 1
    f = single.grid(P.field_uniform(n, n, seed=51))
    x0 = P.field_uniform(n, n, seed=52)
    xs, xd = single.grid(x0), single.grid(x0)
    single.vcycle(f, xs, 2)
    bmg.bmg_vcycle(h, f, xd, 2)
    torch.cuda.synchronize()
    assert torch.equal(xs, xd), float((xs - xd).abs().max())
    ns, nd = single.residual_norm(f, xs), bmg.bmg_residual_norm(h, f, xd)
    assert abs(ns - nd) <= 1e-12 * ns
    assert bmg.bmg_num_levels(h) == single.L
    bmg.bmg_destroy(h)
    single.close()


@pytest.mark.parametrize("max_levels", [5, 6, 7])
def test_loopback_max_levels(max_levels):
    """A truncated hierarchy (max_levels) has the same levels distributed or not: the
    replicated inner solver gets max_levels - K (K distributed levels), so the level
    count and the iterate match the single-GPU solver bitwise."""
    n = 511
    st = P.workload("checker", n, n)
    prm = bmg.bmg_params_default()
    prm.agglom_rows, prm.max_levels = 16, max_levels
    single = bmg.Solver(st, prm)
    h = loopback(st, 2, prm, single.pitch)
    assert bmg.bmg_num_levels(h) == single.L == max_levels
    f = single.grid(P.field_uniform(n, n, seed=53))
    x0 = P.field_uniform(n, n, seed=54)
    xs, xd = single.grid(x0), single.grid(x0)
    single.vcycle(f, xs, 2)
    bmg.bmg_vcycle(h, f, xd, 2)
    torch.cuda.synchronize()
    assert torch.equal(xs, xd), float((xs - xd).abs().max())
    bmg.bmg_destroy(h)
    single.close()


@pytest.mark.parametrize("wl,n,nranks,agg", [("poisson", 511, 3, 16), ("checker", 511, 2, 64)])
def test_loopback_solve(wl, n, nranks, agg):
    st = P.workload(wl, n, n)
    prm = bmg.bmg_params_default()
    prm.agglom_rows = agg
    single = bmg.Solver(st, prm)
    h = loopback(st, nranks, prm, single.pitch)
    f = single.grid(P.rhs_const(n, n))
    xs, xd = single.grid(), single.grid()
    its, hs, rcs = single.solve(f, xs, 1e-10, 100)
    itd, hd, rcd = bmg.bmg_solve(h, f, xd, 1e-10, 100)
    assert rcs == rcd == 0 and its == itd
    assert np.all(np.abs(hs - hd) <= 1e-10 * hs + 1e-13 * hs[0])
    assert torch.equal(xs, xd)
    bmg.bmg_destroy(h)
    single.close()


def test_dist_rejects_tiny_grid():
    st = P.workload("poisson", 31, 31)
    with pytest.raises(bmg.BmgError):
        loopback(st, 8, bmg.bmg_params_default(), bmg.default_pitch(31))


def test_den_nonpositive_rejected_like_oracle(orc):
    """Reading c3(iii): an interpolation denominator <= 0 is EINVAL.  For the
    lognormal field (sigma=2, seed 42) at 255^2 the level-2 Galerkin operator
    has such a row; the oracle and the library both reject it."""
    st = P.workload("lognormal", 255, 255)
    with pytest.raises(ValueError):
        orc.Hierarchy(st)
    with pytest.raises(bmg.BmgError) as ei:
        bmg.Solver(st)
    assert ei.value.status == bmg.BMG_EINVAL


def test_nccl_mode_single_rank():
    """The NCCL transport path (dlopen'ed libnccl, rank-local arrays, grouped
    send/recv + all-gather code) with a 1-rank communicator: bitwise equal to
    the single-GPU solver; the partition-derived local layout matches the ABI."""
    from paper_2502_05279_b200 import dist as D

    n = 511
    st = P.workload("checker", n, n)
    prm = bmg.bmg_params_default()
    single = bmg.Solver(st, prm)
    comm = D.nccl_comm(1, 0)
    ds = D.DistSolver(st, 1, 0, comm, prm, pitch=single.pitch)
    assert bmg.bmg_local_rows(ds.h) == D.local_layout(n, n, 1, 0, prm)
    f = P.field_uniform(n, n, seed=61)
    x0 = P.field_uniform(n, n, seed=62)
    xs = single.grid(x0)
    single.vcycle(single.grid(f), xs, 2)
    fl, xl = ds.local(f), ds.local(x0)
    ds.vcycle(fl, xl, 2)
    torch.cuda.synchronize()
    assert torch.equal(xs[1:-1], xl[1:-1])
    assert abs(ds.residual_norm(fl, xl) - single.residual_norm(single.grid(f), xs)) <= 1e-12 * single.residual_norm(
        single.grid(f), xs)
    ds.close()
    single.close()
