"""bmg_solve's device-side loop: one graph launch whose conditional
WHILE node runs cycle + residual norm + stopping test.  Checked against the
host loop (the path a handle with bmg_timing enabled takes; same kernels) bit
for bit, against the oracle's solve (iterations and history), and
for graph reuse across calls with other tol / maxiter on the same arrays."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from paper_2502_05279_b200 import bmg, problems as P  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__ as ge

    ge.build_lib()


@pytest.mark.parametrize("wl,n,tol", [("poisson", 31, 1e-10), ("lognormal", 63, 1e-9), ("random9", 127, 1e-9),
                                      ("checker", 255, 1e-8)])
def test_device_loop_equals_host_loop_and_oracle(orc, wl, n, tol):
    st = P.workload(wl, n, n)
    s = bmg.Solver(st)
    f = s.grid(P.rhs_const(n, n))
    xd = s.grid()
    itd, hd, rcd = s.solve(f, xd, tol, 100)
    bmg.bmg_timing(s.h, True)  # host loop
    xh = s.grid()
    ith, hh, rch = s.solve(f, xh, tol, 100)
    bmg.bmg_timing(s.h, False)
    assert (itd, rcd) == (ith, rch) and np.array_equal(hd, hh) and torch.equal(xd, xh)
    u, ito, histo, rco = orc.Hierarchy(st).solve(P.rhs_const(n, n), np.zeros((n + 2, n + 2)), tol, 100)
    assert rco == rcd and ito == itd
    assert np.all(np.abs(hd - histo) <= 1e-10 * histo + 1e-12 * histo[0])
    s.close()


def test_device_loop_reuse_and_limits():
    n = 63
    s = bmg.Solver(P.workload("lognormal", n, n))
    f = s.grid(P.rhs_const(n, n))
    x = s.grid()
    it, hist, rc = s.solve(f, x, 1e-12, 3)  # maxiter reached
    assert rc == bmg.BMG_ENOTCONV and it == 3 and len(hist) == 4
    x.zero_()
    it0, h0, rc0 = s.solve(f, x, 1e-8, 50)  # same graph (same arrays), other tol / maxiter
    assert rc0 == 0 and 0 < it0 < 50 and h0[-1] <= 1e-8 * np.linalg.norm(P.rhs_const(n, n))
    it1, h1, rc1 = s.solve(f, x, 1e-8, 50)  # already converged: no cycle
    assert rc1 == 0 and it1 == 0 and len(h1) == 1
    x.zero_()
    it2, h2, rc2 = s.solve(f, x, 1e-8, 0)  # maxiter 0: no cycle, not converged
    assert rc2 == bmg.BMG_ENOTCONV and it2 == 0
    x.zero_()
    it3, h3, rc3 = s.solve(f, x, 1e-8, 2000)  # a larger history than the first allocation
    assert rc3 == 0 and it3 == it0 and np.array_equal(h3, h0)
    s.close()


def test_vcycle_host_batch_bitwise_per_problem():
    """bmg_vcycle_host_batch (include/bmg.h): each problem's result is bitwise that of
    bmg_vcycle_host on the same host arrays, with copies overlapping across problems
    (pinned) -- 5 problems, two staging slots reused, distinct rhs and starts."""
    n = 255
    s = bmg.Solver(P.workload("checker", n, n))
    rhs = [P.field_uniform(n, n, seed=10 + i) for i in range(5)]
    x0 = [P.field_uniform(n, n, seed=20 + i) for i in range(5)]
    fh = [s.grid(a).cpu().pin_memory() for a in rhs]
    xb = [s.grid(a).cpu().pin_memory() for a in x0]
    bmg.bmg_vcycle_host_batch(s.h, fh, xb, 2)
    for i in range(5):
        xr = s.grid(x0[i]).cpu().pin_memory()
        bmg.bmg_vcycle_host(s.h, fh[i], xr, 2)
        assert torch.equal(xb[i], xr), i
    bmg.bmg_vcycle_host_batch(s.h, [], [], 1)  # empty batch: a no-op
    s.close()
