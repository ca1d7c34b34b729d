"""Pins of the 3-D oracle (oracle/bmg3_oracle.c, readings
c16-c24 in DESIGN.md §3) against what the mathematics fixes: closed forms of the
generators, the trilinear weights and the Kronecker-product Galerkin operator of
the 7-point Laplacian, constant reproduction and A-harmonic cell weights, dense
P^T A P, dense colour-ordered Gauss-Seidel and V-cycle, exact zebra block
Gauss-Seidel when the plane solve is exact, the exact solution as a fixed point
of plane relaxation, and a direct solve."""
from __future__ import annotations

import itertools

import numpy as np
import pytest

from oracle import oracle3d as o3
from paper_2502_05279_b200 import problems3d as p3
from tests import dense3 as d3


def _ent(dx, dy, dz):
    return (dz + 1) * 9 + (dy + 1) * 3 + (dx + 1)


# ----------------------------------------------------------------- c18 inputs
def test_poisson7_closed_form():
    s = p3.poisson7(5)
    st = o3.expand_stencil(s)
    a = st[3, 3, 3]
    assert a[13] == 6.0
    for o in [(-1, 0, 0), (1, 0, 0), (0, -1, 0), (0, 1, 0), (0, 0, -1), (0, 0, 1)]:
        assert a[_ent(*o)] == -1.0
    assert np.count_nonzero(a) == 7
    # Dirichlet elimination: the corner node keeps O = 6 and loses 3 couplings
    assert st[1, 1, 1, 13] == 6.0 and np.count_nonzero(st[1, 1, 1]) == 4


def test_q1_isotropic_closed_form_and_brute_force():
    s = p3.q1_27(p3.d3_constant(5, 5, 5))
    a = o3.expand_stencil(s)[3, 3, 3]
    for e in range(27):
        o = (e % 3 - 1, (e // 3) % 3 - 1, e // 9 - 1)
        nz = sum(1 for c in o if c)
        want = {0: 8.0 / 3.0, 1: 0.0, 2: -1.0 / 6.0, 3: -1.0 / 12.0}[nz]
        assert abs(a[e] - want) < 1e-15
    # cell-by-cell FE assembly with a lognormal D, done densely here
    n = 3
    D = p3.d3_lognormal(n, n, n, seed=7)
    A = o3.assemble_dense(o3.expand_stencil(p3.q1_27(D, 1.0, 0.5, 2.0)))
    K1 = np.array([[1.0, -1.0], [-1.0, 1.0]])
    M1 = np.array([[1.0 / 3, 1.0 / 6], [1.0 / 6, 1.0 / 3]])
    Ke = (1.0 * np.kron(np.kron(M1, M1), K1) + 0.5 * np.kron(np.kron(M1, K1), M1)
          + 2.0 * np.kron(np.kron(K1, M1), M1))
    N = n + 2
    G = np.zeros((N ** 3, N ** 3))
    for c, b, a_ in itertools.product(range(n + 1), repeat=3):
        nodes = [((c + dz) * N + (b + dy)) * N + (a_ + dx) for dz in (0, 1) for dy in (0, 1) for dx in (0, 1)]
        G[np.ix_(nodes, nodes)] += D[c, b, a_] * Ke
    idx = [(k * N + j) * N + i for k in range(1, n + 1) for j in range(1, n + 1) for i in range(1, n + 1)]
    np.testing.assert_allclose(A, G[np.ix_(idx, idx)], rtol=0, atol=1e-13)


@pytest.mark.parametrize("name", ["lognormal7", "checker27"])
def test_expand_matches_dense_planes_symmetric_zero_rowsum(name):
    n = 7
    s = p3.WORKLOADS3[name][0](n)
    st = o3.expand_stencil(s)
    A = o3.assemble_dense(st)
    np.testing.assert_array_equal(A, d3.dense_from_planes3(s))
    np.testing.assert_array_equal(A, A.T)
    # rows of nodes whose whole neighbourhood is interior sum to zero
    inner = st[2:-2, 2:-2, 2:-2].sum(axis=-1)
    assert np.abs(inner).max() < 1e-10 * np.abs(st[..., 13]).max()


def test_expand_rejects_nonpositive_diagonal():
    s = p3.poisson7(3)
    s.planes["O"][2, 2, 2] = 0.0
    with pytest.raises(ValueError):
        o3.expand_stencil(s)


# ----------------------------------------------------------------- c19 interpolation
def test_poisson7_weights_trilinear():
    n = 15
    st = o3.expand_stencil(p3.poisson7(n))
    ci = o3.setup_interp(st)
    # interior coarse indices whose fine points are two away from the boundary
    blk = ci[2:-2, 2:-2, 2:-2]
    want = np.array([0.5] * 6 + [0.25] * 12 + [0.125] * 8)
    np.testing.assert_array_equal(blk, np.broadcast_to(want, blk.shape))


@pytest.mark.parametrize("name", ["lognormal7", "checker27"])
def test_interpolation_reproduces_constants(name):
    n = 15
    s = p3.WORKLOADS3[name][0](n)
    st = o3.expand_stencil(s)
    ci = o3.setup_interp(st)
    P = d3.dense_P3(ci, n, n, n)
    ones = P @ np.ones(P.shape[1])
    g = d3.to_grid3(ones, n, n, n)
    # zero-row-sum rows (the row-sum switch is off) whose lower-phase neighbours are too
    np.testing.assert_allclose(g[3:-3, 3:-3, 3:-3], 1.0, rtol=0, atol=1e-13)


def test_cell_weights_are_A_harmonic():
    """At a cell point whose row sums to zero, den = sig and (A P e_C)(p) = 0 for
    every coarse C: the cell value is the operator-weighted mean of its neighbours."""
    n = 15
    s = p3.WORKLOADS3["lognormal7"][0](n)
    st = o3.expand_stencil(s)
    ci = o3.setup_interp(st)
    AP = d3.dense_from_planes3(s) @ d3.dense_P3(ci, n, n, n)
    idx = d3.index3(n, n, n)
    for k, j, i in itertools.product(range(3, n - 1, 2), repeat=3):
        np.testing.assert_allclose(AP[idx[k, j, i]], 0.0, rtol=0, atol=1e-13)


def test_interp_rejects_nonpositive_denominator():
    st = o3.expand_stencil(p3.poisson7(7))
    st[..., :] *= 0.0
    st[..., 13] = 1.0  # no couplings: every collapsed side is 0, den = R switch only at R > 0
    st[1:-1, 1:-1, 1:-1, 13] = 0.0
    with pytest.raises(ValueError):
        o3.setup_interp(st)


# ----------------------------------------------------------------- c20 Galerkin
@pytest.mark.parametrize("name", ["lognormal7", "checker27", "aniso7"])
def test_rap_equals_dense_PtAP(name):
    n = 7
    s = p3.WORKLOADS3[name][0](n)
    st = o3.expand_stencil(s)
    ci = o3.setup_interp(st)
    stc = o3.rap(st, ci)
    A = d3.dense_from_planes3(s)
    P = d3.dense_P3(ci, n, n, n)
    Ac = P.T @ A @ P
    np.testing.assert_allclose(o3.assemble_dense(stc), Ac, rtol=0, atol=1e-12 * np.abs(Ac).max())


def test_rap_poisson7_kronecker_closed_form():
    """With trilinear P = P1 (x) P1 (x) P1 and A = T(x)I(x)I + I(x)T(x)I + I(x)I(x)T, the
    Galerkin operator is sum over axes of (P1'TP1) (x) (P1'P1) (x) (P1'P1) -- at the coarse
    points whose support sees only trilinear weights."""
    n = 15
    m = n // 2
    st = o3.expand_stencil(p3.poisson7(n))
    stc = o3.rap(st, o3.setup_interp(st))
    T = 2 * np.eye(n) - np.eye(n, k=1) - np.eye(n, k=-1)
    P1 = np.zeros((n, m))
    for I in range(1, m + 1):
        P1[2 * I - 1, I - 1] = 1.0
        P1[2 * I - 2, I - 1] = 0.5
        P1[2 * I, I - 1] = 0.5
    Tc, Mc = P1.T @ T @ P1, P1.T @ P1
    Ac = np.kron(np.kron(Mc, Mc), Tc) + np.kron(np.kron(Mc, Tc), Mc) + np.kron(np.kron(Tc, Mc), Mc)
    idx = d3.index3(m, m, m)
    for K, J, I in itertools.product(range(2, m), repeat=3):
        for e in range(27):
            dx, dy, dz = e % 3 - 1, (e // 3) % 3 - 1, e // 9 - 1
            assert abs(stc[K, J, I, e] - Ac[idx[K, J, I], idx[K + dz, J + dy, I + dx]]) < 1e-14


# ----------------------------------------------------------------- c21/c22 cycle steps
@pytest.mark.parametrize("name,kind", [("lognormal7", 7), ("checker27", 27)])
def test_relax_residual_restrict_interp_dense(name, kind):
    n = 7
    s = p3.WORKLOADS3[name][0](n)
    st = o3.expand_stencil(s)
    A = d3.dense_from_planes3(s)
    f = p3.random_interior(n, n, n, seed=1)
    u = p3.random_interior(n, n, n, seed=2)
    fv, uv = d3.to_vec3(f), d3.to_vec3(u)
    got = o3.relax(st, kind, f, u, 2)
    want = d3.dense_gs3(A, fv, uv, d3.colour_masks3(n, n, n, kind), 2)
    np.testing.assert_allclose(d3.to_vec3(got), want, rtol=0, atol=1e-12 * np.abs(want).max())
    r = o3.residual(st, f, u)
    rv = fv - A @ uv
    tol = 1e-14 * np.abs(A).max() * np.abs(uv).max() * 27
    np.testing.assert_allclose(d3.to_vec3(r), rv, rtol=0, atol=tol)
    ci = o3.setup_interp(st)
    P = d3.dense_P3(ci, n, n, n)
    np.testing.assert_allclose(d3.to_vec3(o3.restrict(ci, r)), P.T @ rv, rtol=0, atol=30 * tol)
    e = p3.random_interior(n // 2, n // 2, n // 2, seed=3)
    np.testing.assert_allclose(d3.to_vec3(o3.interp_add(ci, e, u)), uv + P @ d3.to_vec3(e), rtol=0, atol=1e-13)


def _dense_vcycle3(As, Ps, kinds, dims, f, u, nu1, nu2):
    def rec(l, f, u):
        A = As[l]
        if l == len(As) - 1:
            return np.linalg.solve(A, f)
        masks = d3.colour_masks3(*dims[l], kinds[l])
        u = d3.dense_gs3(A, f, u, masks, nu1)
        fc = Ps[l].T @ (f - A @ u)
        u = u + Ps[l] @ rec(l + 1, fc, np.zeros_like(fc))
        return d3.dense_gs3(A, f, u, masks, nu2)
    return rec(0, f, u)


@pytest.mark.parametrize("name", ["lognormal7", "checker27"])
def test_vcycle_point_equals_dense(name):
    n = 15
    s = p3.WORKLOADS3[name][0](n)
    H = o3.Hierarchy3(s)
    assert H.num_levels == 3
    As, Ps, kinds, dims = [], [], [], []
    for l in range(H.num_levels):
        nx, ny, nz, kind = H.level_shape(l)
        st, ci = H.export_level(l)
        As.append(d3.dense_from_full3(st))
        kinds.append(kind)
        dims.append((nx, ny, nz))
        if ci is not None:
            Ps.append(d3.dense_P3(ci, nx, ny, nz))
    f = p3.random_interior(n, n, n, seed=5)
    u = p3.random_interior(n, n, n, seed=6)
    got = H.vcycle(f, u, 1)
    want = _dense_vcycle3(As, Ps, kinds, dims, d3.to_vec3(f), d3.to_vec3(u), 2, 1)
    np.testing.assert_allclose(d3.to_vec3(got), want, rtol=0, atol=1e-11 * np.abs(want).max())


# ----------------------------------------------------------------- c23 plane relaxation
@pytest.mark.parametrize("nz", [2, 5, 7])
@pytest.mark.parametrize("name", ["lognormal7", "checker27", "aniso7"])
def test_planes_exact_zebra_when_planes_are_3x3(name, nz):
    """On 3x3 planes the plane hierarchy is one level (c1), its V-cycle a Cholesky
    solve: a plane sweep is exact zebra block Gauss-Seidel (k even first)."""
    nx = ny = 3
    D = p3.d3_lognormal(nx, ny, nz, seed=11)
    s = {"lognormal7": p3.fv7(D), "aniso7": p3.fv7(D, az=1e-3), "checker27": p3.q1_27(D)}[name]
    # a hierarchy needs >= 2 levels for the fine level to relax by planes: embed in a 7x7 plane? No --
    # coarsest=1 keeps 3x3xnz as a relaxed fine level (min(3,3,nz) > 1 for nz >= 2).
    H = o3.Hierarchy3(s, relax="planes", coarsest=1)
    assert H.num_levels >= 2
    f = p3.random_interior(nx, ny, nz, seed=12)
    u = p3.random_interior(nx, ny, nz, seed=13)
    got = H.relax_fine(f, u, 2)
    A = d3.dense_from_planes3(s)
    want = d3.dense_zebra_exact(A, d3.to_vec3(f), d3.to_vec3(u), nx, ny, nz, 2)
    np.testing.assert_allclose(d3.to_vec3(got), want, rtol=0, atol=1e-12 * np.abs(want).max())


@pytest.mark.parametrize("name", ["aniso7", "checker27", "lognormal7"])
def test_planes_fixed_point_exact_solution(name):
    n = 15
    s = p3.WORKLOADS3[name][0](n)
    H = o3.Hierarchy3(s, relax="planes")
    A = d3.dense_from_planes3(s)
    f = p3.random_interior(n, n, n, seed=21)
    x = np.linalg.solve(A, d3.to_vec3(f))
    got = H.relax_fine(f, d3.to_grid3(x, n, n, n), 1)
    np.testing.assert_allclose(d3.to_vec3(got), x, rtol=0, atol=1e-11 * np.abs(x).max())


def test_planes_one_sweep_equals_dense_block_gs_with_2d_cycle():
    """7x7 planes (a 2-level plane hierarchy): one plane sweep = for each plane (k even,
    then odd) g = f_k - A_{k,other} u, then the pinned 2-D oracle's V(1,1) cycle on the
    plane's in-plane operator, built here from the dense matrix."""
    from oracle import Hierarchy as H2
    from paper_2502_05279_b200.problems import Stencil

    n, nz = 7, 5
    s = p3.q1_27(p3.d3_lognormal(n, n, nz, seed=31))
    H = o3.Hierarchy3(s, relax="planes", coarsest=1)
    f = p3.random_interior(n, n, nz, seed=32)
    u = p3.random_interior(n, n, nz, seed=33)
    got = H.relax_fine(f, u, 1)
    A = d3.dense_from_planes3(s)
    idx = d3.index3(n, n, nz)
    fv, uv = d3.to_vec3(f), d3.to_vec3(u)
    kk = d3.plane_masks(n, n, nz)
    for c in (0, 1):
        for k in range(1, nz + 1):
            if k % 2 != c:
                continue
            m = kk == k
            g = fv[m] - A[np.ix_(m, ~m)] @ uv[~m]
            # the plane operator as 2-D ABI planes, read off the dense block
            planes = {nm: np.zeros((n + 2, n + 2)) for nm in ("O", "W", "S", "SW", "NW")}
            for j, i in itertools.product(range(1, n + 1), repeat=2):
                p = idx[k, j, i]
                planes["O"][j, i] = A[p, p]
                for nm, (dx, dy) in {"W": (-1, 0), "S": (0, -1), "SW": (-1, -1), "NW": (-1, 1)}.items():
                    q = idx[k, j + dy, i + dx]
                    planes[nm][j, i] = A[p, q] if q >= 0 else 0.0
            h2 = H2(Stencil(9, n, n, planes), nu1=1, nu2=1)
            g2 = np.zeros((n + 2, n + 2))
            g2[1:-1, 1:-1] = g.reshape(n, n)
            u2 = np.zeros((n + 2, n + 2))
            u2[1:-1, 1:-1] = uv[m].reshape(n, n)
            uv[m] = h2.vcycle(g2, u2, 1)[1:-1, 1:-1].reshape(-1)
    np.testing.assert_allclose(d3.to_vec3(got), uv, rtol=0, atol=1e-13 * np.abs(uv).max())


# ----------------------------------------------------------------- solve
@pytest.mark.parametrize("name,relax,factor", [("poisson7", "point", 0.1), ("lognormal7", "point", 0.3),
                                               ("checker27", "point", 0.35), ("aniso7", "planes", 0.01),
                                               ("checker27", "planes", 0.35)])
def test_solve_converges_to_direct_solution(name, relax, factor):
    n = 15
    s = p3.WORKLOADS3[name][0](n)
    H = o3.Hierarchy3(s, relax=relax)
    f = p3.rhs_const(n, n, n)
    x, it, hist, rc = H.solve(f, np.zeros_like(f), 1e-11, 60)
    assert rc == o3.OK
    assert np.all(np.diff(hist) < 0)
    assert (hist[-1] / hist[0]) ** (1.0 / it) < factor
    A = d3.dense_from_planes3(s)
    xd = np.linalg.solve(A, d3.to_vec3(f))
    np.testing.assert_allclose(d3.to_vec3(x), xd, rtol=0, atol=1e-9 * np.abs(xd).max())


def test_point_relaxation_stalls_on_weak_z_coupling():
    """Why c23 exists: with z-coupling 1e-3, point GS smoothing leaves a V-cycle factor near 1."""
    n = 15
    s = p3.WORKLOADS3["aniso7"][0](n)
    f = p3.rhs_const(n, n, n)
    _, it, hist, _ = o3.Hierarchy3(s, relax="point").solve(f, np.zeros_like(f), 1e-11, 10)
    assert (hist[-1] / hist[0]) ** (1.0 / it) > 0.5


def test_zero_rhs_and_levels():
    s = p3.poisson7(7)
    H = o3.Hierarchy3(s)
    f = np.zeros((9, 9, 9))
    x, it, hist, rc = H.solve(f, p3.random_interior(7, 7, 7), 1e-8, 5)
    assert rc == o3.OK and it == 0 and not x.any()
    assert o3.count_levels(255, 255, 255) == 7 and o3.count_levels(63, 63, 15) == 3
    assert o3.count_levels(7, 7, 7, max_levels=1) == 1


def test_poisson7_boundary_weights_row_sum_switch():
    """c19's row-sum switch at the Dirichlet boundary (7-point Laplacian, n = 14 so the
    last interior index 14 is even and line points can touch the boundary across their
    line).  ci[K, J, I, slot]; an x-line point (2I-1, 2J, 2K) uses slots 0 (toward I-1), 1.
    * (3, 2, 2): interior row, R = 0 -> den = sig_b = 2 -> 1/2, 1/2 (trilinear);
    * (1, 2, 2): the x = 0 ghost drops cW: eps = 0, R = 1 > 0 -> den = 0 + 1 + 1 -> 0, 1/2;
    * (3, 14, 2): one ghost neighbour across the line: sig = 5, R = 1 > sig/6 -> den = 3;
    * (3, 14, 14): two ghost neighbours: sig = 4, R = 2 > 4/6 -> den = 4."""
    ci = o3.setup_interp(o3.expand_stencil(p3.poisson7(14)))
    assert list(ci[1, 1, 2, 0:2]) == [0.5, 0.5]
    assert list(ci[1, 1, 1, 0:2]) == [0.0, 0.5]
    assert ci[1, 7, 2, 0] == pytest.approx(1 / 3, abs=1e-16) and ci[1, 7, 2, 1] == pytest.approx(1 / 3, abs=1e-16)
    assert list(ci[7, 7, 2, 0:2]) == [0.25, 0.25]
    # the same switch reaches the face points: XY face (3, 3, 14) (top z face): collapse over z
    # drops nothing in-plane (b = 4-neighbour Laplacian, b_O = 6 - 1), sig = 5, R = 1 > 5/6
    # -> den = sig_b + R = 4 + 1 = 5; its four line neighbours sit on the same face (1/3
    # each, as above), so each corner weight = (1/3 + 1/3) / 5 = 2/15
    assert ci[7, 2, 2, 6:10] == pytest.approx([2 / 15] * 4, abs=1e-16)
