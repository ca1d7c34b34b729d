"""The tail kernel (kernels_cycle.cu k_tail_sm): every small level of the
cycle in one single-CTA launch out of shared memory.  Its per-point arithmetic is the
per-step kernels' (relax5_pt / relax9_pt with 1/a_pp from the same rcp_pos, residual_pt,
restrict_store, interp_pt), and within one colour GS updates are independent, so a cycle
whose levels all run in the tail is BITWISE the global-memory tail's (BMG_TAIL_SM=0), and
within rounding of the per-step cycle (fused = 0), whose restriction keeps the terms of
the colour relaxed last (zero up to rounding; the tail drops them, c5a).  Shapes: square, ragged, odd/even, 5-/9-point level 0,
both smoother parities, the symmetric cycle (c12) and affine interpolation (c14)."""
import os

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


def _cycle(wl, nx, ny, fused, nu1, nu2, sym, affine, tail_sm=True, ncycles=2):
    prm = bmg.bmg_params_default()
    prm.fused = fused
    prm.nu1, prm.nu2 = nu1, nu2
    prm.cycle_sym = sym
    prm.affine = affine
    old = os.environ.get("BMG_TAIL_SM")
    os.environ["BMG_TAIL_SM"] = "1" if tail_sm else "0"
    try:
        s = bmg.Solver(P.workload(wl, nx, ny), prm)
    finally:
        if old is None:
            del os.environ["BMG_TAIL_SM"]
        else:
            os.environ["BMG_TAIL_SM"] = old
    f = s.grid(P.field_uniform(nx, ny, seed=1))
    u = s.grid(P.field_uniform(nx, ny, seed=2))
    s.vcycle(f, u, ncycles)
    torch.cuda.synchronize()
    return u.cpu().numpy()


CASES = [("poisson", 31, 31), ("aniso", 31, 31), ("checker", 30, 17), ("random9", 25, 32), ("lognormal", 3, 40),
         ("poisson", 1, 1), ("lognormal", 2, 2), ("checker_off3", 31, 33)]


@pytest.mark.parametrize("wl,nx,ny", CASES)
@pytest.mark.parametrize("nu1,nu2,sym,affine", [(2, 1, 0, 0), (1, 1, 1, 0), (2, 2, 0, 1), (1, 2, 0, 0)])
def test_tail_sm_bitwise(wl, nx, ny, nu1, nu2, sym, affine):
    t = _cycle(wl, nx, ny, 1, nu1, nu2, sym, affine)
    assert np.array_equal(t, _cycle(wl, nx, ny, 1, nu1, nu2, sym, affine, tail_sm=False))
    ps = _cycle(wl, nx, ny, 0, nu1, nu2, sym, affine)
    assert np.abs(t - ps).max() <= 1e-12 * np.abs(ps).max()


def _solve(wl, nx, ny, tol, maxiter, one_launch, rhs_zero=False):
    old = os.environ.get("BMG_TAIL_SOLVE")
    os.environ["BMG_TAIL_SOLVE"] = "1" if one_launch else "0"
    try:
        s = bmg.Solver(P.workload(wl, nx, ny))
        f = s.grid(np.zeros((ny + 2, nx + 2)) if rhs_zero else P.rhs_const(nx, ny))
        x = s.grid(P.field_uniform(nx, ny, seed=3))
        it, hist, rc = s.solve(f, x, tol, maxiter)
        torch.cuda.synchronize()
        out = (it, np.asarray(hist).copy(), rc, x.cpu().numpy())
        s.close()
        return out
    finally:
        if old is None:
            del os.environ["BMG_TAIL_SOLVE"]
        else:
            os.environ["BMG_TAIL_SOLVE"] = old


@pytest.mark.parametrize("wl,nx,ny,tol,maxiter", [("poisson", 31, 31, 1e-10, 100), ("aniso", 31, 31, 1e-8, 100),
                                                  ("checker", 30, 17, 1e-10, 100), ("random9", 25, 32, 1e-9, 100),
                                                  ("lognormal", 3, 40, 1e-10, 100), ("poisson", 31, 31, 1e-12, 3),
                                                  ("poisson", 31, 31, 1e-8, 0)])
def test_tail_solve_one_launch_bitwise_graph_loop(wl, nx, ny, tol, maxiter):
    """bmg_solve with the whole hierarchy in the tail runs as ONE k_tail_solve launch
    (norms in launch_resid_norm's reduction order): iterations, status, history and the
    iterate bitwise the graph loop's (BMG_TAIL_SOLVE=0), incl. maxiter reached / 0."""
    a = _solve(wl, nx, ny, tol, maxiter, True)
    b = _solve(wl, nx, ny, tol, maxiter, False)
    assert a[0] == b[0] and a[2] == b[2]
    assert np.array_equal(a[1], b[1]) and np.array_equal(a[3], b[3])


def test_tail_solve_zero_rhs():
    it, hist, rc, x = _solve("poisson", 31, 31, 1e-10, 100, True, rhs_zero=True)
    assert rc == 0 and it == 0 and hist[0] == 0.0 and np.all(x[1:-1, 1:32] == 0.0)
