"""Pins for the oracle's problem ingest, interpolation (c3) and Galerkin RAP (c4).

Every expected value here comes from the paper/SPEC (golden fixtures), a
closed form derived from the mathematics, or an independent dense
definition (tests/dense.py) -- never from the CUDA path.
"""
import json
import os

import numpy as np
import pytest

from paper_2502_05279_b200 import problems as P
from tests import dense

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def gold(name):
    with open(os.path.join(GOLD, name)) as fh:
        return json.load(fh)


# --------------------------------------------------------------- ingest (c0, c2)
def test_problem_build_golden(orc):
    g = gold("spec_problem_build.json")
    s = P.workload("poisson", 7, 7)
    st = orc.expand_stencil(s)
    for k, name in enumerate(orc.STENCIL_ORDER):
        assert st[4, 4, k] == g["poisson_interior"][name]
    f = P.rhs_const(3, 3)
    assert np.all(f[1:-1, 1:-1] == g["n3_rhs"])
    assert np.all(f[0, :] == 0) and np.all(f[:, 0] == 0)


@pytest.mark.parametrize("wl", ["poisson", "lognormal", "checker", "aniso", "random9"])
def test_expand_matches_dense_planes_and_is_symmetric(orc, wl):
    s = P.workload(wl, 15, 13)
    A_full = dense.dense_from_full(orc.expand_stencil(s))
    A_planes = dense.dense_from_planes(s)
    assert np.array_equal(A_full, A_planes)
    assert np.array_equal(A_full, A_full.T)
    assert np.all(np.linalg.eigvalsh(A_full) > 0)


def test_ghost_couplings_dropped_and_row_sums(orc):
    n = 9
    st = orc.expand_stencil(P.workload("poisson", n, n))
    assert np.all(st[0, :, :] == 0) and np.all(st[:, 0, :] == 0)
    assert np.all(st[1, :, 0:3] == 0)  # row j=1 has no south couplings
    assert np.all(st[:, n, [2, 5, 8]] == 0)  # column i=n has no east couplings
    rs = st.sum(axis=2)
    # interior rows sum to exactly 0; Poisson edge rows 1, corner rows 2 (c2 pins)
    assert np.all(rs[2:n, 2:n] == 0.0)
    assert rs[1, 1] == 2.0 and rs[n, n] == 2.0 and rs[1, n] == 2.0 and rs[n, 1] == 2.0
    assert np.all(rs[1, 2:n] == 1.0) and np.all(rs[2:n, 1] == 1.0)
    # variable D: interior row sums are 0 up to rounding of 5 terms
    st = orc.expand_stencil(P.workload("lognormal", n, n))
    rs = st.sum(axis=2)[2:n, 2:n]
    assert np.all(np.abs(rs) <= 8e-16 * np.abs(st[2:n, 2:n]).sum(axis=2))


def test_bad_diagonal_rejected(orc):
    s = P.workload("poisson", 7, 7)
    s.planes["O"][3, 3] = 0.0
    with pytest.raises(ValueError):
        orc.expand_stencil(s)


def test_level_ladder(orc):
    assert orc.count_levels(7, 7) == gold("spec_convergence.json")["levels_n7"]
    assert orc.count_levels(31, 31) == 4
    assert orc.count_levels(1023, 1023) == 9  # "levels 3-9" at N=1024^2
    assert orc.count_levels(8191, 8191) == 12
    assert orc.count_levels(8191, 16383) == 12
    assert orc.count_levels(3, 3) == 1


# --------------------------------------------------------------- interpolation (c3)
def bilinear_ci(ncx, ncy):
    """Bilinear weights (edge 1/2, cell-centre 1/4), zero toward ghost coarse points."""
    ci = np.zeros((ncy + 2, ncx + 2, 8))
    for J in range(ncy + 2):
        for I in range(ncx + 2):
            w = ci[J, I]
            inI = 1 <= I <= ncx
            inIm = 1 <= I - 1 <= ncx
            inJ = 1 <= J <= ncy
            inJm = 1 <= J - 1 <= ncy
            w[3] = 0.5 if (inI and inJ) else 0.0  # LR -> (I,J)
            w[4] = 0.5 if (inIm and inJ) else 0.0  # LL -> (I-1,J)
            w[1] = 0.5 if (inI and inJ) else 0.0  # LA -> (I,J)
            w[6] = 0.5 if (inI and inJm) else 0.0  # LB -> (I,J-1)
            w[0] = 0.25 if (inI and inJ) else 0.0  # LNE
            w[2] = 0.25 if (inIm and inJ) else 0.0  # LNW
            w[5] = 0.25 if (inI and inJm) else 0.0  # LSE
            w[7] = 0.25 if (inIm and inJm) else 0.0  # LSW
    return ci


def ci_interior_view(ci, nx, ny):
    """Mask of CI entries that belong to (interior fine point, interior coarse target)."""
    ncx, ncy = nx // 2, ny // 2
    m = np.zeros(ci.shape, dtype=bool)
    for J in range(ncy + 2):
        for I in range(ncx + 2):
            fx_ok = 1 <= 2 * I - 1 <= nx
            fy_ok = 1 <= 2 * J - 1 <= ny
            cx_ok = 1 <= 2 * I <= nx
            cy_ok = 1 <= 2 * J <= ny
            tI, tIm = 1 <= I <= ncx, 1 <= I - 1 <= ncx
            tJ, tJm = 1 <= J <= ncy, 1 <= J - 1 <= ncy
            m[J, I, 3] = fx_ok and cy_ok and tI and tJ
            m[J, I, 4] = fx_ok and cy_ok and tIm and tJ
            m[J, I, 1] = cx_ok and fy_ok and tI and tJ
            m[J, I, 6] = cx_ok and fy_ok and tI and tJm
            m[J, I, 0] = fx_ok and fy_ok and tI and tJ
            m[J, I, 2] = fx_ok and fy_ok and tIm and tJ
            m[J, I, 5] = fx_ok and fy_ok and tI and tJm
            m[J, I, 7] = fx_ok and fy_ok and tIm and tJm
    return m


@pytest.mark.parametrize("n", [7, 31, 63])
def test_poisson_interp_is_bilinear_on_every_level(orc, n):
    """p-P1: for Poisson the operator-induced P equals bilinear exactly (all levels)."""
    h = orc.Hierarchy(P.workload("poisson", n, n))
    for l in range(h.num_levels - 1):
        nx, ny, _ = h.level_shape(l)
        _, ci = h.export_level(l)
        m = ci_interior_view(ci, nx, ny)
        assert np.array_equal(ci[m], bilinear_ci(nx // 2, ny // 2)[m]), f"level {l}"


def test_interp_1d_closed_form(orc):
    """p-P3: D varying only in x -> X weights D_{i-1/2}/(D_{i-1/2}+D_{i+1/2}) etc.;
    Y weights 1/2; Z weights are the tensor product (x weight) * 1/2."""
    n = 31
    a = np.arange(n + 1)
    D = np.tile(1.0 + 10.0 * a, (n + 1, 1))
    st = orc.expand_stencil(P.stencil5_from_D(D))
    ci = orc.setup_interp(st)
    for J in range(2, n // 2):
        for I in range(2, n // 2):
            i = 2 * I - 1  # X / Z column
            Dl, Dr = D[0, i - 1], D[0, i]
            assert ci[J, I, 4] == pytest.approx(Dl / (Dl + Dr), rel=1e-15, abs=0)  # LL
            assert ci[J, I, 3] == pytest.approx(Dr / (Dl + Dr), rel=1e-15, abs=0)  # LR
            assert ci[J, I, 1] == 0.5 and ci[J, I, 6] == 0.5  # LA, LB
            assert ci[J, I, 0] == pytest.approx(0.5 * Dr / (Dl + Dr), rel=1e-14)  # LNE
            assert ci[J, I, 5] == pytest.approx(0.5 * Dr / (Dl + Dr), rel=1e-14)  # LSE
            assert ci[J, I, 2] == pytest.approx(0.5 * Dl / (Dl + Dr), rel=1e-14)  # LNW
            assert ci[J, I, 7] == pytest.approx(0.5 * Dl / (Dl + Dr), rel=1e-14)  # LSW


@pytest.mark.parametrize("wl", ["lognormal", "checker", "poisson", "aniso"])
def test_interp_reproduces_constants(orc, wl):
    """p-P2: (P 1)(f) = 1 at every fine point whose row sum is 0 (4 eps bound)."""
    n = 63
    h = orc.Hierarchy(P.workload(wl, n, n))
    for l in range(h.num_levels - 1):
        nx, ny, _ = h.level_shape(l)
        st, ci = h.export_level(l)
        ones_c = np.zeros((ny // 2 + 2, nx // 2 + 2))
        ones_c[1:-1, 1:-1] = 1.0
        p1 = orc.interp_add(ci, ones_c, np.zeros((ny + 2, nx + 2)))
        rs = st.sum(axis=2)
        scale = np.abs(st).sum(axis=2)
        zero_row = np.abs(rs) <= 1e-13 * scale
        zero_row[0, :] = zero_row[-1, :] = zero_row[:, 0] = zero_row[:, -1] = False
        assert zero_row.sum() > 0
        err = np.abs(p1 - 1.0)[zero_row]
        assert err.max() <= 4 * np.finfo(float).eps, f"level {l}: {err.max()}"


# --------------------------------------------------------------- Galerkin RAP (c4)
def poisson_rap_closed_form(k):
    """p-RAP2: interior coarse stencil on level k of Poisson (dyadic, exact)."""
    q = 4.0 ** (-k)
    return 8.0 / 3.0 + (4.0 / 3.0) * q, -1.0 / 3.0 - (2.0 / 3.0) * q, -1.0 / 3.0 + (1.0 / 3.0) * q


def test_poisson_rap_closed_form(orc):
    n = 127
    h = orc.Hierarchy(P.workload("poisson", n, n))
    assert h.num_levels == 6
    expect = {1: (3.0, -0.5, -0.25), 2: (2.75, -0.375, -0.3125), 3: (2.6875, -0.34375, -0.328125),
              4: (2.671875, -0.3359375, -0.33203125)}
    for k in range(1, 5):
        st, _ = h.export_level(k)
        nx = st.shape[1] - 2
        O, e, c = poisson_rap_closed_form(k)
        assert (O, e, c) == expect[k]
        inner = st[2:nx, 2:nx]
        assert np.all(inner[..., 4] == O), k
        assert np.all(inner[..., [1, 3, 5, 7]] == e), k
        assert np.all(inner[..., [0, 2, 6, 8]] == c), k
        rs = st.sum(axis=2)
        # corner rows 5/3 + 4^-k/3, edge-midpoint rows 1 (p-RAP4)
        assert rs[1, 1] == 5.0 / 3.0 + (4.0 ** -k) / 3.0 or abs(rs[1, 1] - (5 / 3 + 4.0 ** -k / 3)) < 1e-15
        assert rs[1, (nx + 1) // 2] == pytest.approx(1.0, abs=1e-15)


@pytest.mark.parametrize("wl,n", [("poisson", 7), ("lognormal", 15), ("checker", 31), ("aniso", 15),
                                  ("random9", 15), ("lognormal", 14)])
def test_rap_equals_dense_galerkin(orc, wl, n):
    """p-RAP1 / p-R2 / p-I1: with P^T := the fig:restrict_kernel restriction,
    the stencil RAP equals dense P^T A P to 1e-12; interp_add equals u + P e."""
    s = P.workload(wl, n, n)
    st = orc.expand_stencil(s)
    A = dense.dense_from_planes(s)
    ci = orc.setup_interp(st)
    Pm = dense.dense_P_from_restriction(orc, ci, n, n)
    stc = orc.rap(st, ci)
    Ac = dense.dense_from_full(stc)
    ref = Pm.T @ A @ Pm
    assert np.abs(Ac - ref).max() <= 1e-12 * np.abs(ref).max()
    assert np.allclose(Ac, Ac.T, rtol=0, atol=1e-13 * np.abs(ref).max())
    # interpolation + correction is u + P e (c7 vs c5 transposes)
    rng = np.random.default_rng(1)
    e = dense.to_grid(rng.uniform(-1, 1, (n // 2) ** 2), n // 2, n // 2)
    u0 = dense.to_grid(rng.uniform(-1, 1, n * n), n, n)
    got = dense.to_vec(orc.interp_add(ci, e, u0))
    assert np.allclose(got, dense.to_vec(u0) + Pm @ dense.to_vec(e), rtol=0, atol=1e-14)
    # P has the documented sparsity: C rows are unit vectors
    for j in range(2, n + 1, 2):
        for i in range(2, n + 1, 2):
            row = Pm[(j - 1) * n + (i - 1)]
            assert row.max() == 1.0 and np.count_nonzero(row) == 1


def test_rap_row_sums_lognormal(orc):
    """p-RAP4: interior coarse row sums ~0 for zero-row-sum fine operators."""
    h = orc.Hierarchy(P.workload("lognormal", 63, 63))
    for l in range(1, h.num_levels):
        st, _ = h.export_level(l)
        nx = st.shape[1] - 2
        inner = st[2:nx, 2:nx]
        rs = inner.sum(axis=2)
        assert np.all(np.abs(rs) <= 2e-14 * np.abs(inner).sum(axis=2)), l
        # symmetry of stored entries: E(i,j) == W(i+1,j), N(i,j) == S(i,j+1), NE == SW(i+1,j+1)
        assert np.allclose(st[1:-1, 1:-2, 5], st[1:-1, 2:-1, 3], rtol=1e-13, atol=0)
        assert np.allclose(st[1:-2, 1:-1, 7], st[2:-1, 1:-1, 1], rtol=1e-13, atol=0)
        assert np.allclose(st[1:-2, 1:-2, 8], st[2:-1, 2:-1, 0], rtol=1e-13, atol=0)
