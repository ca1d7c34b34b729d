"""GPU <-> oracle parity of zebra line relaxation (DESIGN §3 c11, kernels_line.cu)
through the C ABI (params.relax), tolerances as DESIGN §7:

* one relaxation call on level 0 (same operator on both sides): 1e-12
  relative per component with the max|u| floor (a line solve's rounding is
  amplified by the condition number of its tridiagonal block, ~1e3 on the
  anisotropic y-lines);
* one V-cycle iterate: 1e-12 (floor max|x|); per-cycle norms 1e-10;
* at the bench size (4095^2 anisotropic, the launch configuration bench.py
  times) a property that holds at any size: after a sweep the lines of the
  colour relaxed last have zero residual (each was solved exactly with its
  neighbours final).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from paper_2502_05279_b200 import bmg, problems as P  # noqa: E402

MODES = {"xline": bmg.BMG_RELAX_XLINES, "yline": bmg.BMG_RELAX_YLINES, "altline": bmg.BMG_RELAX_ALTLINES}


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__ as ge

    ge.build_lib()


def params(mode):
    prm = bmg.bmg_params_default()
    prm.relax = MODES[mode]
    return prm


def assert_iterate_close(g, o, rtol=1e-12):
    tol = rtol * np.maximum(np.abs(o), np.abs(o).max())
    err = np.abs(g - o)
    assert np.all(err <= tol), (err.max(), np.abs(o).max())


# sizes: single chunk (n <= 16), two chunks, many ragged chunks, lines of length 1..3
STEP_CASES = [("lognormal", 13, 9), ("random9", 17, 31), ("aniso", 63, 40), ("checker", 127, 127),
              ("lognormal", 300, 257), ("random9", 200, 131), ("aniso", 1, 7), ("lognormal", 33, 2),
              ("poisson", 16, 16), ("lognormal", 3, 100)]


@pytest.mark.parametrize("wl,nx,ny", STEP_CASES)
@pytest.mark.parametrize("mode", ["xline", "yline", "altline"])
def test_relax_lines_step(orc, wl, nx, ny, mode):
    st = P.workload(wl, nx, ny)
    s = bmg.Solver(st, params(mode))
    st9 = orc.expand_stencil(st)
    f = P.field_uniform(nx, ny, seed=51)
    u0 = P.field_uniform(nx, ny, seed=52)
    for nsw in (1, 2):
        u = s.grid(u0)
        bmg.bmg_relax(s.h, 0, s.grid(f), u, nsw)
        torch.cuda.synchronize()
        got = bmg.from_device(u, nx)
        assert_iterate_close(got, orc.relax_lines(st9, f, u0, nsw, mode))
        xg = u.cpu().numpy()
        assert np.all(xg[0, :] == 0) and np.all(xg[-1, :] == 0) and np.all(xg[:, 0] == 0)
        assert np.all(xg[:, nx + 1:] == 0)
    s.close()


VC_CASES = [("aniso", 63, 63), ("lognormal", 63, 63), ("checker", 127, 127), ("random9", 33, 33),
            ("aniso", 100, 37), ("poisson", 31, 31), ("lognormal", 5, 9)]


@pytest.mark.parametrize("wl,nx,ny", VC_CASES)
@pytest.mark.parametrize("mode", ["xline", "yline", "altline"])
def test_vcycle_lines_parity(orc, wl, nx, ny, mode):
    st = P.workload(wl, nx, ny)
    s = bmg.Solver(st, params(mode))
    h = orc.Hierarchy(st, relax=mode)
    f = P.field_uniform(nx, ny, seed=61)
    x0 = P.field_uniform(nx, ny, seed=62)
    x = s.grid(x0)
    s.vcycle(s.grid(f), x, 1)
    torch.cuda.synchronize()
    assert_iterate_close(bmg.from_device(x, nx), h.vcycle(f, x0, 1))
    s.close()


@pytest.mark.parametrize("wl,n,mode,tol,maxit", [("aniso", 63, "yline", 1e-10, 50), ("aniso", 127, "altline", 1e-10, 50),
                                                 ("lognormal", 63, "altline", 1e-10, 100)])
def test_solve_lines_parity(orc, wl, n, mode, tol, maxit):
    st = P.workload(wl, n, n)
    s = bmg.Solver(st, params(mode))
    h = orc.Hierarchy(st, relax=mode)
    f = P.rhs_const(n, n)
    x = s.grid()
    it, hist, rc = s.solve(s.grid(f), x, tol, maxit)
    uo, ito, histo, rco = h.solve(f, np.zeros_like(f), tol, maxit)
    assert rc == rco == 0 and it == ito
    floor = 1e-12 * histo[0]
    assert np.all(np.abs(hist - histo) <= 1e-10 * histo + floor), np.abs(hist / histo - 1).max()
    assert_iterate_close(bmg.from_device(x, n), uo, rtol=1e-10)
    s.close()


def line_indefinite_stencil(n=31):
    """Poisson with an indefinite x-line segment (row 5, i = 3..5: O = 1, W = -1,
    nearly decoupled in y): the oracle accepts it with point or y-line relaxation
    and reports ENOTSPD for x-lines (tests/test_oracle_lines.py p-L6)."""
    st = P.workload("poisson", n, n)
    st.planes = {k: v.copy() for k, v in st.planes.items()}
    st.planes["O"][5, 3:6] = 1.0
    st.planes["W"][5, 4:6] = -1.0
    st.planes["S"][5, 3:6] = -0.001
    st.planes["S"][6, 3:6] = -0.001
    return st


def test_line_not_spd_setup():
    bad = line_indefinite_stencil()
    with pytest.raises(bmg.BmgError) as ei:
        bmg.Solver(bad, params("xline"))
    assert ei.value.status == bmg.BMG_ENOTSPD
    bmg.Solver(bad, params("yline")).close()
    bmg.Solver(bad).close()
    prm = bmg.bmg_params_default()
    prm.relax = 7
    with pytest.raises(bmg.BmgError) as ei:
        bmg.Solver(P.workload("poisson", 15, 15), prm)
    assert ei.value.status == bmg.BMG_EINVAL


@pytest.mark.parametrize("mode,last_y", [("yline", True), ("xline", False), ("altline", True)])
def test_bench_size_last_colour_lines_exact(mode, last_y):
    """4095^2 anisotropic (BASELINE config 3, bench launch configuration): after one
    sweep, the residual vanishes on every line of colour 1 of the last direction."""
    n = 4095
    st = P.workload("aniso", n, n)
    s = bmg.Solver(st, params(mode))
    f = s.grid(P.rhs_const(n, n))
    u = s.grid(P.field_uniform(n, n, seed=71))
    bmg.bmg_relax(s.h, 0, f, u, 1)
    r = s.grid()
    bmg.bmg_residual(s.h, 0, f, u, r)
    torch.cuda.synchronize()
    rr = r[:, : n + 2]
    lines = rr[1:-1, 1::2] if last_y else rr[1::2, 1:-1]  # colour-1 columns / rows: odd 1..4095 (n+1 even)
    other = rr[1:-1, 2:-1:2] if last_y else rr[2:-1:2, 1:-1]
    scale = float(f.abs().max()) + float(u.abs().max()) * 8 / 3
    assert float(lines.abs().max()) <= 1e-11 * scale
    assert float(other.abs().max()) > 1e-6 * scale  # the other colour is not trivially zero
    s.close()
