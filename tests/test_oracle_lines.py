"""Pins for the oracle's line relaxation (reading c11): zebra
line Gauss-Seidel, the "Line" box of fig:vcycle_flowchart, which the
paper names but does not define.

What fixes it independently of the oracle's Thomas code:
* p-L1 the definition as dense block Gauss-Seidel: every line of a colour is
  solved with numpy.linalg.solve for its block of A, the other lines' current
  values on the right-hand side (tests/dense.py assembles A from the ABI
  planes);
* p-L2 closed forms: a stencil with no x couplings (W = 0) is a set of
  decoupled columns, so ONE y-line sweep is the exact solve A^-1 f (and the
  same for S = 0 with x-lines); a single-row grid is one line;
* p-L3 transposition: an x-line sweep on A equals a y-line sweep on the
  transposed grid problem (every index of the y-line path is exercised), and
  so does a whole V-cycle (interpolation, RAP, restriction are transposition
  equivariant up to rounding);
* p-L4 the exact solution is a fixed point;
* p-L5 behaviour: on the anisotropic Q1 operator of config 3 (strong coupling
  in y) y-line relaxation turns the point-GS factor (~0.95) into ~0.02;
* p-L6 a line block with a non-positive pivot is reported (ENOTSPD).
"""
import numpy as np
import pytest

from paper_2502_05279_b200 import problems as P
from tests import dense


def line_masks(nx, ny, ylines):
    """Boolean masks (lexicographic interior order) of each line, grouped by colour
    (c11: colour = line index mod 2, colour 0 first)."""
    J, I = np.meshgrid(np.arange(1, ny + 1), np.arange(1, nx + 1), indexing="ij")
    coord = (I if ylines else J).reshape(-1)
    nl = nx if ylines else ny
    groups = []
    for c in (0, 1):
        groups.append([coord == line for line in range(1, nl + 1) if line % 2 == c])
    return groups


def dense_line_gs(A, f, u, nx, ny, mode, nsweeps):
    """c11 as dense block GS: u_L <- A_LL^{-1} (f_L - A_{L,rest} u_rest) per line L."""
    u = u.copy()
    dirs = {"xline": [False], "yline": [True], "altline": [False, True]}[mode]
    for _ in range(nsweeps):
        for ylines in dirs:
            for group in line_masks(nx, ny, ylines):
                for m in group:
                    rhs = f[m] - A[m][:, ~m] @ u[~m]
                    u[m] = np.linalg.solve(A[np.ix_(m, m)], rhs)
    return u


def transpose_stencil(stc: P.Stencil) -> P.Stencil:
    """The same operator on the transposed grid (x <-> y): A^T(i,j) couplings from
    A(j,i).  W^T = S, S^T = W, SW^T = SW, NW^T(i,j) = A[(j,i),(j+1,i-1)] = NW(j+1,i-1)."""
    nx, ny = stc.ny, stc.nx
    pl = stc.planes
    T = {"O": pl["O"].T.copy(), "W": pl["S"].T.copy(), "S": pl["W"].T.copy()}
    if stc.kind == 9:
        T["SW"] = pl["SW"].T.copy()
        nw = np.zeros((ny + 2, nx + 2))
        # nw[j, i] (point (i,j) of the transposed grid) = NW of original point (j+1, i-1)
        src = pl["NW"]  # src[b, a] = NW at original (a, b)
        for j in range(ny + 2):
            for i in range(nx + 2):
                a, b = j + 1, i - 1
                if 0 <= a < src.shape[1] and 0 <= b < src.shape[0]:
                    nw[j, i] = src[b, a]
        T["NW"] = nw
    return P.Stencil(stc.kind, nx, ny, T)


CASES = [("lognormal", 13, 9), ("random9", 12, 11), ("aniso", 9, 14), ("checker", 15, 15), ("poisson", 8, 5)]


@pytest.mark.parametrize("wl,nx,ny", CASES)
@pytest.mark.parametrize("mode", ["xline", "yline", "altline"])
def test_line_gs_equals_dense_block_gs(orc, wl, nx, ny, mode):
    """p-L1"""
    stc = P.workload(wl, nx, ny)
    st = orc.expand_stencil(stc)
    A = dense.dense_from_planes(stc)
    f = P.field_uniform(nx, ny, seed=5)
    u0 = P.field_uniform(nx, ny, seed=6)
    got = orc.relax_lines(st, f, u0, 2, mode)
    want = dense.to_grid(dense_line_gs(A, dense.to_vec(f), dense.to_vec(u0), nx, ny, mode, 2), nx, ny)
    scale = np.abs(want).max()
    assert np.abs(got - want).max() <= 1e-13 * scale
    assert np.all(got[0, :] == 0) and np.all(got[-1, :] == 0) and np.all(got[:, 0] == 0) and np.all(got[:, -1] == 0)


@pytest.mark.parametrize("nx,ny", [(7, 5), (16, 9), (1, 6)])
def test_decoupled_columns_one_yline_sweep_is_exact(orc, nx, ny):
    """p-L2: W = 0 (no x coupling) -> A is block diagonal in columns; one y-line
    sweep from any guess returns A^-1 f."""
    rng = np.random.default_rng(11)
    shape = (ny + 2, nx + 2)
    S = -rng.uniform(0.5, 2.0, shape)
    O = np.zeros(shape)
    O[1:-1, 1:-1] = -(S[1:-1, 1:-1] + S[2:, 1:-1]) + rng.uniform(0.01, 0.1, (ny, nx))
    stc = P.Stencil(5, nx, ny, {"O": O, "W": np.zeros(shape), "S": S})
    st = orc.expand_stencil(stc)
    A = dense.dense_from_planes(stc)
    f = P.field_uniform(nx, ny, seed=1)
    got = orc.relax_lines(st, f, P.field_uniform(nx, ny, seed=2), 1, "yline")
    want = dense.to_grid(np.linalg.solve(A, dense.to_vec(f)), nx, ny)
    assert np.abs(got - want).max() <= 1e-13 * np.abs(want).max()
    # transposed: S = 0, one x-line sweep is exact
    stT = transpose_stencil(stc)
    gotT = orc.relax_lines(orc.expand_stencil(stT), f.T.copy(), np.zeros((nx + 2, ny + 2)), 1, "xline")
    assert np.abs(gotT - want.T).max() <= 1e-13 * np.abs(want).max()


def test_single_row_is_one_line(orc):
    """p-L2: ny = 1: the grid is one x-line; one sweep solves the tridiagonal system."""
    nx = 23
    stc = P.workload("lognormal", nx, 1)
    st = orc.expand_stencil(stc)
    A = dense.dense_from_planes(stc)
    f = P.field_uniform(nx, 1, seed=4)
    got = orc.relax_lines(st, f, np.zeros_like(f), 1, "xline")
    want = dense.to_grid(np.linalg.solve(A, dense.to_vec(f)), nx, 1)
    assert np.abs(got - want).max() <= 1e-14 * np.abs(want).max()


@pytest.mark.parametrize("wl,nx,ny", [("lognormal", 11, 8), ("random9", 10, 13), ("aniso", 12, 7)])
def test_transposition_sweep(orc, wl, nx, ny):
    """p-L3: x-lines on A == y-lines on the transposed problem (and vice versa)."""
    stc = P.workload(wl, nx, ny)
    stT = transpose_stencil(stc)
    # the transposed operator really is A with x <-> y (dense check of the helper)
    idx = dense.interior_index(nx, ny)
    perm = idx[1:-1, 1:-1].T.reshape(-1)
    A = dense.dense_from_planes(stc)
    assert np.array_equal(dense.dense_from_planes(stT), A[np.ix_(perm, perm)])
    f = P.field_uniform(nx, ny, seed=7)
    u0 = P.field_uniform(nx, ny, seed=8)
    st, stt = orc.expand_stencil(stc), orc.expand_stencil(stT)
    for a, b in (("xline", "yline"), ("yline", "xline")):
        g1 = orc.relax_lines(st, f, u0, 2, a)
        g2 = orc.relax_lines(stt, f.T.copy(), u0.T.copy(), 2, b)
        assert np.abs(g1 - g2.T).max() <= 1e-14 * np.abs(g1).max()


@pytest.mark.parametrize("wl,n", [("aniso", 31), ("lognormal", 31)])
def test_transposition_vcycle(orc, wl, n):
    """p-L3 through the whole cycle: V(2,1) with x-lines on A == y-lines on A^T."""
    stc = P.workload(wl, n, n)
    stT = transpose_stencil(stc)
    f = P.field_uniform(n, n, seed=9, scale=1e-3)
    u0 = P.field_uniform(n, n, seed=10)
    a = orc.Hierarchy(stc, relax="xline").vcycle(f, u0, 2)
    b = orc.Hierarchy(stT, relax="yline").vcycle(f.T.copy(), u0.T.copy(), 2)
    assert np.abs(a - b.T).max() <= 1e-12 * np.abs(a).max()


@pytest.mark.parametrize("mode", ["xline", "yline", "altline"])
def test_exact_solution_fixed_point(orc, mode):
    """p-L4"""
    nx, ny = 14, 11
    stc = P.workload("random9", nx, ny)
    A = dense.dense_from_planes(stc)
    f = P.field_uniform(nx, ny, seed=3)
    xs = dense.to_grid(np.linalg.solve(A, dense.to_vec(f)), nx, ny)
    got = orc.relax_lines(orc.expand_stencil(stc), f, xs, 1, mode)
    assert np.abs(got - xs).max() <= 1e-13 * np.abs(xs).max()


def _factor(H, n, k0, k1):
    """mean per-cycle residual reduction between cycles k0 and k1 (f = 0, random x0)"""
    f = np.zeros((n + 2, n + 2))
    x = P.field_uniform(n, n, seed=3)
    rs = [H.residual_norm(f, x)]
    for _ in range(k1):
        x = H.vcycle(f, x, 1)
        rs.append(H.residual_norm(f, x))
    return (rs[k1] / rs[k0]) ** (1 / (k1 - k0)), rs


def test_yline_fixes_anisotropy(orc):
    """p-L5: Q1 -(1e-3 u_xx + u_yy), n=63: point GS ~0.93 per cycle, y-line GS ~0.02
    (measured 0.948 over cycles 20-25 / 0.018 over cycles 2-5 under c11), alternating
    lines at least as good."""
    n = 63
    stc = P.workload("aniso", n, n)
    fp, _ = _factor(orc.Hierarchy(stc, relax="point"), n, 20, 25)
    fx, _ = _factor(orc.Hierarchy(stc, relax="xline"), n, 20, 25)
    fy, _ = _factor(orc.Hierarchy(stc, relax="yline"), n, 2, 5)
    fa, _ = _factor(orc.Hierarchy(stc, relax="altline"), n, 2, 5)
    assert fp > 0.85 and fx > 0.85
    assert fy < 0.05 and fa < 0.05


def test_vcycle_line_matches_dense_vcycle(orc):
    """p-L1 through the cycle: V(1,1) with y-lines equals the dense recursive cycle
    built from the oracle's own operators/weights and dense block GS."""
    nx, ny = 15, 15
    stc = P.workload("lognormal", nx, ny)
    H = orc.Hierarchy(stc, nu1=1, nu2=1, relax="yline")
    L = H.num_levels
    As, Ps, dims = [], [], []
    for l in range(L):
        st, ci = H.export_level(l)
        lx, ly, _ = H.level_shape(l)
        As.append(dense.dense_from_full(st))
        dims.append((lx, ly))
        if ci is not None:
            Ps.append(dense.dense_P_from_restriction(orc, ci, lx, ly))
    f = P.field_uniform(nx, ny, seed=12)
    u0 = P.field_uniform(nx, ny, seed=13)

    def rec(l, fv, uv):
        if l == L - 1:
            return np.linalg.solve(As[l], fv)
        lx, ly = dims[l]
        uv = dense_line_gs(As[l], fv, uv, lx, ly, "yline", 1)
        fc = Ps[l].T @ (fv - As[l] @ uv)
        uv = uv + Ps[l] @ rec(l + 1, fc, np.zeros_like(fc))
        return dense_line_gs(As[l], fv, uv, lx, ly, "yline", 1)

    want = dense.to_grid(rec(0, dense.to_vec(f), dense.to_vec(u0)), nx, ny)
    got = H.vcycle(f, u0, 1)
    assert np.abs(got - want).max() <= 1e-12 * np.abs(want).max()


def test_line_not_spd_reported(orc):
    """p-L6: an x-line segment with O = 1, W = -1 (tridiag(-1, 1, -1) is singular:
    second pivot 0) inside a Poisson grid: x-line relaxation reports ENOTSPD (also
    at setup), while the hierarchy with point or y-line relaxation sets up fine."""
    n = 31
    stc = P.workload("poisson", n, n)
    stc.planes = {k: v.copy() for k, v in stc.planes.items()}
    stc.planes["O"][5, 3:6] = 1.0
    stc.planes["W"][5, 4:6] = -1.0
    stc.planes["S"][5, 3:6] = -0.001
    stc.planes["S"][6, 3:6] = -0.001
    st = orc.expand_stencil(stc)
    z = np.zeros((n + 2, n + 2))
    with pytest.raises(np.linalg.LinAlgError):
        orc.relax_lines(st, z, z, 1, "xline")
    orc.relax_lines(st, z, z, 1, "yline")
    with pytest.raises(ValueError, match="status 5"):
        orc.Hierarchy(stc, relax="xline")
    orc.Hierarchy(stc, relax="yline")
    orc.Hierarchy(stc, relax="point")
