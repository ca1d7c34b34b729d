"""Pins for the oracle's cycle steps (c5-c9): relaxation, residual,
restriction, interpolation, Cholesky, norm, V-cycle and solve.

Expected values: SPEC golden fixtures (tests/golden), dense linear algebra
(tests/dense.py, numpy/scipy), closed forms, and SURVEY §8(c) p-V1/p-V2
numbers that were derived independently (dense scipy) under
the same readings.
"""
import json
import os

import numpy as np
import pytest
import scipy.sparse
import scipy.sparse.linalg

from paper_2502_05279_b200 import problems as P
from tests import dense

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def gold(name):
    with open(os.path.join(GOLD, name)) as fh:
        return json.load(fh)


# --------------------------------------------------------------- Cholesky / norm (c8)
def test_cholesky_golden(orc):
    g = gold("spec_cholesky_2x2.json")
    L = orc.chol_factor(np.array(g["A"]))
    assert np.allclose(L, np.array(g["L"]), rtol=0, atol=1e-15)
    assert np.allclose(L @ L.T, np.array(g["A"]), rtol=0, atol=1e-14)
    x = orc.chol_solve(L, np.array(g["b"]))
    assert np.allclose(x, np.array(g["x"]), rtol=0, atol=1e-15)


@pytest.mark.parametrize("n", [1, 3, 9, 16])
def test_cholesky_random_spd(orc, n):
    rng = np.random.default_rng(n)
    M = rng.standard_normal((n, n))
    A = M @ M.T + n * np.eye(n)
    b = rng.standard_normal(n)
    L = orc.chol_factor(A)
    assert np.allclose(L, np.linalg.cholesky(A), rtol=0, atol=1e-12)
    x = orc.chol_solve(L, b)
    assert np.abs(A @ x - b).max() <= 1e-10


def test_cholesky_not_spd(orc):
    with pytest.raises(np.linalg.LinAlgError):
        orc.chol_factor(np.array([[1.0, 2.0], [2.0, 1.0]]))


def test_norm_golden(orc):
    for case in gold("spec_norm2.json")["cases"]:
        v = np.array(case["v"])
        g = np.zeros((3, len(v) + 2))
        g[1, 1:-1] = v
        assert orc.norm2(g) == case["norm"]


# --------------------------------------------------------------- restriction (c5)
def test_restriction_golden_ones(orc):
    g = gold("spec_restriction_ones.json")
    n = g["n_fine"]
    ci = np.full((n // 2 + 2, n // 2 + 2, 8), g["weight"])
    q = np.full((n + 2, n + 2), g["q"])
    qc = orc.restrict(ci, q)
    assert np.all(qc[1:-1, 1:-1] == g["qc_interior"])
    assert np.all(qc[0, :] == 0) and np.all(qc[:, -1] == 0)


def test_restriction_random_weights_naive(orc):
    """p-R3: random weights vs a naive 9-term sum to 1e-13 --
    expressed with numpy slicing (a different evaluation of fig:restrict_kernel)."""
    rng = np.random.default_rng(7)
    n = 31
    nc = n // 2
    ci = rng.uniform(-1, 1, (nc + 2, nc + 2, 8))
    q = rng.uniform(-1, 1, (n + 2, n + 2))
    qc = orc.restrict(ci, q)
    I = np.arange(1, nc + 1)
    J = I[:, None]
    Ii = I[None, :]
    ref = (ci[J, Ii, 0] * q[2 * J - 1, 2 * Ii - 1] + ci[J, Ii, 1] * q[2 * J - 1, 2 * Ii]
           + ci[J, Ii + 1, 2] * q[2 * J - 1, 2 * Ii + 1] + ci[J, Ii, 3] * q[2 * J, 2 * Ii - 1]
           + q[2 * J, 2 * Ii] + ci[J, Ii + 1, 4] * q[2 * J, 2 * Ii + 1]
           + ci[J + 1, Ii, 5] * q[2 * J + 1, 2 * Ii - 1] + ci[J + 1, Ii, 6] * q[2 * J + 1, 2 * Ii]
           + ci[J + 1, Ii + 1, 7] * q[2 * J + 1, 2 * Ii + 1])
    assert np.abs(qc[1:-1, 1:-1] - ref).max() <= 1e-13


# --------------------------------------------------------------- relaxation / residual (c6)
@pytest.mark.parametrize("wl,n", [("poisson", 15), ("lognormal", 15), ("aniso", 14), ("random9", 13)])
def test_relax_equals_dense_multicolour_gs(orc, wl, n):
    """p-GS3 (+ p-GS1 via the same-colour-uncoupled assertion in dense_gs)."""
    s = P.workload(wl, n, n)
    st = orc.expand_stencil(s)
    A = dense.dense_from_planes(s)
    f = P.field_uniform(n, n, seed=3)
    u0 = P.field_uniform(n, n, seed=4)
    for kind in ([5, 9] if s.kind == 5 else [9]):  # 5-pt operators also under 4 colours
        got = orc.relax(st, kind, f, u0, nsweeps=2)
        ref = dense.dense_gs(A, dense.to_vec(f), dense.to_vec(u0), dense.colour_masks(n, n, kind), 2)
        assert np.abs(dense.to_vec(got) - ref).max() <= 1e-13 * max(1.0, np.abs(ref).max())
        assert np.all(got[0, :] == 0) and np.all(got[:, 0] == 0)


@pytest.mark.parametrize("wl", ["poisson", "checker", "aniso"])
def test_exact_solution_is_fixed_point(orc, wl):
    """p-GS2 / SPEC S:435: relaxation and the V-cycle leave A^{-1} f unchanged."""
    n = 31
    s = P.workload(wl, n, n)
    A = dense.dense_from_planes(s)
    f = P.field_uniform(n, n, seed=5)
    x = dense.to_grid(np.linalg.solve(A, dense.to_vec(f)), n, n)
    st = orc.expand_stencil(s)
    assert np.abs(orc.relax(st, s.kind, f, x, 3) - x).max() <= 1e-12 * np.abs(x).max()
    h = orc.Hierarchy(s)
    assert np.abs(h.vcycle(f, x, 1) - x).max() <= 1e-11 * np.abs(x).max()
    assert h.residual_norm(f, h.vcycle(f, x, 1)) <= 1e-12 * orc.norm2(f)


def test_residual_dense(orc):
    n = 15
    s = P.workload("random9", n, n)
    f = P.field_uniform(n, n, seed=8)
    u = P.field_uniform(n, n, seed=9)
    r = orc.residual(orc.expand_stencil(s), f, u)
    ref = dense.to_vec(f) - dense.dense_from_planes(s) @ dense.to_vec(u)
    assert np.abs(dense.to_vec(r) - ref).max() <= 1e-14 * 8


# --------------------------------------------------------------- V-cycle (c9)
@pytest.mark.parametrize("wl,n", [("poisson", 15), ("lognormal", 31), ("aniso", 15), ("checker", 31),
                                  ("random9", 15), ("lognormal", 30)])
def test_vcycle_equals_dense_vcycle(orc, wl, n):
    """The recursive cycle (c9) equals the dense V(2,1) built from dense A_l,
    P_l (from the restriction), dense coloured GS and np.linalg.solve."""
    s = P.workload(wl, n, n)
    h = orc.Hierarchy(s)
    As, Ps, kinds, dims = [], [], [], []
    A = dense.dense_from_planes(s)
    for l in range(h.num_levels):
        nx, ny, kind = h.level_shape(l)
        st, ci = h.export_level(l)
        As.append(A)
        kinds.append(kind)
        dims.append((nx, ny))
        if ci is not None:
            Pm = dense.dense_P_from_restriction(orc, ci, nx, ny)
            Ps.append(Pm)
            A = Pm.T @ A @ Pm  # dense Galerkin (not the oracle's stencil RAP)
    f = P.field_uniform(n, n, seed=11)
    u0 = P.field_uniform(n, n, seed=12)
    got = dense.to_vec(h.vcycle(f, u0, 1))
    ref = dense.dense_vcycle(As, Ps, kinds, dims, dense.to_vec(f), dense.to_vec(u0), 2, 1)
    assert np.abs(got - ref).max() <= 1e-11 * np.abs(ref).max()


def test_config1_history(orc):
    """p-V1 (config 1): 31^2 Poisson, f = h^2, x0 = 0, V(2,1) -> 7 cycles to 1e-10,
    relative history as derived independently in SURVEY §8(c) p-V1."""
    n = 31
    s = P.workload("poisson", n, n)
    f = P.rhs_const(n, n)
    h = orc.Hierarchy(s)
    assert orc.norm2(f) == 0.0302734375
    u, it, hist, rc = h.solve(f, np.zeros_like(f), 1e-10, 50)
    assert rc == orc.OK and it == 7
    rel = hist / hist[0]
    expect = [1, 3.170619e-2, 6.781695e-4, 1.594269e-5, 4.010287e-7, 9.972273e-9, 2.500688e-10]
    assert np.allclose(rel[:7], expect, rtol=2e-6, atol=2e-14)  # atol: residual rounding floor ~1e-14
    assert rel[7] == pytest.approx(6.349e-12, rel=1e-3)  # roundoff-level digits differ
    assert np.all(np.diff(hist) < 0)  # p-V3 / SPEC S:461
    A = scipy.sparse.csr_matrix(dense.dense_from_planes(s))
    x = scipy.sparse.linalg.spsolve(A, dense.to_vec(f))
    assert np.abs(dense.to_vec(u) - x).max() <= 1e-12  # p-V4 (2.4e-14 observed in SURVEY)
    assert u[16, 16] == pytest.approx(0.0736147373545, abs=1e-12)


def test_spec_convergence_bounds(orc):
    """SPEC S:436 (one V(1,1) reduction <= 0.2) and S:445 (<= 12 cycles to 1e-8)."""
    g = gold("spec_convergence.json")
    n = 63
    s = P.workload("poisson", n, n)
    f = P.rhs_const(n, n)
    h = orc.Hierarchy(s, nu1=1, nu2=1)
    u1 = h.vcycle(f, np.zeros_like(f), 1)
    assert h.residual_norm(f, u1) / orc.norm2(f) <= g["vcycle11_n63_first_reduction_max"]
    u, it, hist, rc = h.solve(f, np.zeros_like(f), g["poisson_n63_tol"], 50)
    assert rc == orc.OK and it <= g["poisson_n63_max_cycles"]
    assert np.all(np.diff(hist) < 0)


def test_zero_rhs_returns_immediately(orc):
    """b = 0 -> x = 0, no cycles."""
    n = 15
    h = orc.Hierarchy(P.workload("poisson", n, n))
    f = np.zeros((n + 2, n + 2))
    u, it, hist, rc = h.solve(f, P.field_uniform(n, n), 1e-8, 10)
    assert rc == orc.OK and it == 0 and np.all(u == 0)


def test_not_converged(orc):
    """anisotropy with point smoothing -> ENOTCONV, history valid."""
    n = 31
    h = orc.Hierarchy(P.workload("aniso", n, n))
    f = P.rhs_const(n, n)
    u, it, hist, rc = h.solve(f, np.zeros_like(f), 1e-14, 5)
    assert rc == orc.ENOTCONV and it == 5 and len(hist) == 6


def asymptotic_factor(orc, s, ncyc=12, seed=0):
    n = s.nx
    h = orc.Hierarchy(s)
    f = np.zeros((s.ny + 2, n + 2))
    u = P.field_uniform(n, s.ny, seed=seed)
    prev = None
    for _ in range(ncyc):
        u = h.vcycle(f, u, 1)
        rn = h.residual_norm(f, u)
        fac = rn / prev if prev else None
        prev = rn
    return fac


@pytest.mark.parametrize("wl,n,lo,hi", [
    ("poisson", 31, 0.020, 0.034),   # p-V2: 0.0268
    ("poisson", 63, 0.022, 0.035),   # 0.0283
    ("checker", 31, 0.30, 0.45),     # 8x8 coarse-aligned 1e6 checkerboard: 0.372
    ("checker_off3", 63, 0.12, 0.19),  # offset-by-3 checkerboard: 0.155
    ("lognormal", 63, 0.33, 0.46),   # 0.397
])
def test_convergence_factors(orc, wl, n, lo, hi):
    fac = asymptotic_factor(orc, P.workload(wl, n, n), ncyc=14)
    assert lo <= fac <= hi, fac


def test_operator_induced_beats_bilinear_at_jump(orc):
    """p-P4: a 1e6 jump at an odd node (x=21, n=63): OI factor ~0.035 (bilinear 0.37)."""
    n = 63
    s = P.stencil5_from_D(P.d_node_jump(n, n, 21))
    fac = asymptotic_factor(orc, s, ncyc=12)
    assert fac < 0.08, fac


@pytest.mark.parametrize("wl,kind,n", [("lognormal", 5, 31), ("checker", 5, 31), ("random9", 9, 30), ("aniso", 9, 31)])
def test_last_colour_residual_vanishes(orc, wl, kind, n):
    """The identity behind DESIGN §3 c5a: after a multicolour GS sweep the residual is
    zero (to rounding) at every point of the colour relaxed last -- 5-point: black
    ((i+j) odd), 9-point: colour 3 (i, j odd) -- and not at the others."""
    stc = P.workload(wl, n, n)
    st = orc.expand_stencil(stc)
    f = P.field_uniform(n, n, seed=11)
    u = orc.relax(st, kind, f, P.field_uniform(n, n, seed=12), 1)
    r = orc.residual(st, f, u)
    J, I = np.meshgrid(np.arange(n + 2), np.arange(n + 2), indexing="ij")
    inside = (I >= 1) & (I <= n) & (J >= 1) & (J <= n)
    last = inside & (((I + J) % 2 == 1) if kind == 5 else ((I % 2 == 1) & (J % 2 == 1)))
    scale = np.abs(f).max() + np.abs(u).max() * np.abs(st).sum(-1).max()
    assert np.abs(r[last]).max() <= 1e-15 * scale
    assert np.abs(r[inside & ~last]).max() > 1e-6 * np.abs(r).max()
