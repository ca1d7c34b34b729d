"""3-D BoxMG: GPU <-> oracle parity through include/bmg3.h.

* level-0 ingest and interpolation weights: bitwise (same arithmetic, no
  contraction in setup; DESIGN §3 c19);
* coarse operators: 1e-12 relative per entry, floor = the row's |O|; coarse
  weights 1e-12 absolute (O(1) ratios); the anisotropic plane workload uses
  the DESIGN §7 fp64-drift reading where noted;
* one V-cycle / relaxation iterate: 1e-12 of max|x| per component (normwise);
* residual histories: 1e-10 relative.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from oracle import oracle3d as o3  # noqa: E402
from paper_2502_05279_b200 import bmg3, problems3d as p3  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__ as ge

    ge.build_lib()


def _wl(name, n, ny=None, nz=None):
    ny = n if ny is None else ny
    nz = n if nz is None else nz
    if name == "poisson7":
        return p3.fv7(p3.d3_constant(n, ny, nz))
    if name == "lognormal7":
        return p3.fv7(p3.d3_lognormal(n, ny, nz))
    if name == "aniso7":
        return p3.fv7(p3.d3_constant(n, ny, nz), az=1e-3)
    if name == "checkeraniso7":
        return p3.fv7(p3.d3_checkerboard(n, ny, nz, 4, 1e4), az=1e-3)
    if name == "lognormalaniso7":
        return p3.fv7(p3.d3_lognormal(n, ny, nz, sigma=0.5), az=1e-3)
    if name == "checker27":
        return p3.q1_27(p3.d3_checkerboard(n, ny, nz, max(1, (n + 1) // 8), 1e4))
    if name == "lognormal27":
        return p3.q1_27(p3.d3_lognormal(n, ny, nz), 1.0, 0.7, 1.3)
    raise KeyError(name)


def _full_of_planes(stg):
    """GPU export (14 planes: O + 13 lower) -> the lower half + centre of the 27-entry stencil."""
    out = {13: stg[0]}
    for e in range(13):
        out[e] = stg[1 + e]
    return out


def assert_level_close(stg, st_orc, exact=False, rtol=1e-12):
    floor = np.abs(st_orc[..., 13])
    for e, g in _full_of_planes(stg).items():
        o = st_orc[..., e]
        if exact:
            assert np.array_equal(g, o), e
        else:
            bad = np.abs(g - o) > rtol * np.maximum(np.abs(o), floor)
            assert not bad.any(), (e, np.abs(g - o).max(), np.argwhere(bad)[:3])


def assert_iterate_close(g, o, rtol=1e-12):
    err = np.abs(g - o)
    assert err.max() <= rtol * np.abs(o).max(), (err.max(), np.abs(o).max())


SHAPES = [(15, 15, 15), (31, 31, 31), (33, 29, 35), (20, 17, 26)]


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("name", ["lognormal7", "checker27", "lognormal27"])
def test_setup_every_level(name, shape):
    nx, ny, nz = shape
    s = _wl(name, nx, ny, nz)
    S = bmg3.Solver3(s)
    H = o3.Hierarchy3(s)
    assert S.L == H.num_levels
    for l in range(S.L):
        assert bmg3.bmg3_level_shape(S.h, l) == H.level_shape(l)
        stg, cig = bmg3.bmg3_export_level(S.h, l)
        sto, cio = H.export_level(l)
        assert_level_close(stg, sto, exact=(l == 0))
        if cio is not None:
            cig = np.moveaxis(cig, 0, -1)
            if l == 0:
                assert np.array_equal(cig, cio)
            else:
                assert np.abs(cig - cio).max() <= 1e-12
    S.close()


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("name,relax", [("poisson7", "point"), ("lognormal7", "point"), ("checker27", "point"),
                                        ("lognormal27", "point"), ("aniso7", "planes"), ("checker27", "planes"),
                                        ("lognormal7", "planes"), ("checkeraniso7", "planes")])
def test_vcycle_parity(name, relax, shape):
    nx, ny, nz = shape
    s = _wl(name, nx, ny, nz)
    f = p3.random_interior(nx, ny, nz, seed=1)
    x0 = p3.random_interior(nx, ny, nz, seed=2)
    S = bmg3.Solver3(s, relax=relax)
    x = S.grid(x0)
    S.vcycle(S.grid(f), x, 2)
    torch.cuda.synchronize()
    got = bmg3.from_device3(x, nx)
    ref = o3.Hierarchy3(s, relax=relax).vcycle(f, x0, 2)
    assert_iterate_close(got, ref)
    assert not got[0].any() and not got[-1].any() and not got[:, 0].any() and not got[:, :, 0].any()
    S.close()


@pytest.mark.parametrize("name,relax", [("lognormal7", "point"), ("checker27", "point"), ("aniso7", "planes"),
                                        ("lognormal27", "planes")])
def test_relax_parity(name, relax):
    n = 31
    s = _wl(name, n)
    f = p3.random_interior(n, n, n, seed=3)
    x0 = p3.random_interior(n, n, n, seed=4)
    S = bmg3.Solver3(s, relax=relax)
    x = S.grid(x0)
    S.relax(S.grid(f), x, 2)
    torch.cuda.synchronize()
    ref = o3.Hierarchy3(s, relax=relax).relax_fine(f, x0, 2)
    assert_iterate_close(bmg3.from_device3(x, n), ref)
    S.close()


@pytest.mark.parametrize("name,relax,tol", [("poisson7", "point", 1e-10), ("checker27", "point", 1e-10),
                                            ("aniso7", "planes", 1e-10)])
def test_solve_parity(name, relax, tol):
    n = 31
    s = _wl(name, n)
    f = p3.rhs_const(n, n, n)
    S = bmg3.Solver3(s, relax=relax)
    x = S.grid()
    it, hist, rc = S.solve(S.grid(f), x, tol, 60)
    xo, ito, histo, rco = o3.Hierarchy3(s, relax=relax).solve(f, np.zeros_like(f), tol, 60)
    assert rc == 0 and rco == 0 and it == ito
    floor = 1e-12 * histo[0]  # below this the norms are rounding noise of both sides
    assert np.all(np.abs(hist - histo) <= 1e-10 * histo + floor), np.abs(hist / histo - 1).max()
    assert_iterate_close(bmg3.from_device3(x, n), xo, 1e-11)
    S.close()


@pytest.mark.parametrize("shape,relax", [((63, 63, 63), "point"), ((63, 63, 63), "planes"), ((127, 127, 127), "point")])
def test_larger_cycle_every_point(shape, relax):
    nx, ny, nz = shape
    s = _wl("lognormal7" if relax == "point" else "checkeraniso7", nx, ny, nz)
    f = p3.random_interior(nx, ny, nz, seed=5)
    x0 = p3.random_interior(nx, ny, nz, seed=6)
    S = bmg3.Solver3(s, relax=relax)
    x = S.grid(x0)
    S.vcycle(S.grid(f), x, 1)
    torch.cuda.synchronize()
    ref = o3.Hierarchy3(s, relax=relax).vcycle(f, x0, 1)
    assert_iterate_close(bmg3.from_device3(x, nx), ref)
    S.close()


def test_single_level_and_zero_rhs():
    # 3x3x3: the fine level is the coarsest -> the cycle is the Cholesky solve
    s = _wl("lognormal27", 3)
    f = p3.random_interior(3, 3, 3, seed=7)
    S = bmg3.Solver3(s)
    assert S.L == 1
    x = S.grid()
    S.vcycle(S.grid(f), x, 1)
    torch.cuda.synchronize()
    ref = o3.Hierarchy3(s).vcycle(f, np.zeros_like(f), 1)
    assert_iterate_close(bmg3.from_device3(x, 3), ref)
    x = S.grid(p3.random_interior(3, 3, 3, seed=8))
    it, hist, rc = S.solve(S.grid(), x, 1e-8, 5)
    assert it == 0 and rc == 0 and not bmg3.from_device3(x, 3).any()
    S.close()


def test_errors_on_device():
    s = _wl("poisson7", 7)
    s.planes["O"][3, 3, 3] = -1.0
    from paper_2502_05279_b200.bmg import BmgError

    with pytest.raises(BmgError):
        bmg3.Solver3(s)
    assert bmg3.bmg3_cycle_kernel_count(bmg3.Solver3(_wl("poisson7", 15)).h) > 0


def test_rejection_matches_oracle():
    """c19's den <= 0 (a positive collapsed coupling on a Galerkin coarse level):
    lognormal D with z-coupling 1e-3 is rejected by both implementations (EINVAL)."""
    s = _wl("lognormalaniso7", 15)
    with pytest.raises(ValueError):
        o3.Hierarchy3(s)
    from paper_2502_05279_b200.bmg import BmgError

    with pytest.raises(BmgError) as ei:
        bmg3.Solver3(s)
    assert ei.value.status == 1 and "denominator" in str(ei.value)


@pytest.mark.parametrize("nu", [(1, 1), (1, 2), (3, 1), (2, 0), (0, 2)])
@pytest.mark.parametrize("name,relax", [("lognormal7", "point"), ("checker27", "point"), ("aniso7", "planes")])
def test_vcycle_nu_parity(name, relax, nu):
    """Every parity of nu1 / nu2: the one-pass 7-point sweep's ping-pong between x and its
    second buffer, and the up leg's out-of-place interpolation, end in x."""
    nx, ny, nz = 31, 27, 33
    s = _wl(name, nx, ny, nz)
    f = p3.random_interior(nx, ny, nz, seed=11)
    x0 = p3.random_interior(nx, ny, nz, seed=12)
    S = bmg3.Solver3(s, relax=relax, nu1=nu[0], nu2=nu[1])
    x = S.grid(x0)
    S.vcycle(S.grid(f), x, 2)
    S.relax(S.grid(f), x, 3)  # an odd number of sweeps through bmg3_relax
    torch.cuda.synchronize()
    H = o3.Hierarchy3(s, relax=relax, nu1=nu[0], nu2=nu[1])
    ref = H.relax_fine(f, H.vcycle(f, x0, 2), 3)
    assert_iterate_close(bmg3.from_device3(x, nx), ref)
    S.close()
