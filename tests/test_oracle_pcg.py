"""Pins for the symmetric cycle (reading c12) and V-cycle-preconditioned CG
(reading c13), SURVEY §8(f) row 3 ("BoxMG-faithful variants + Krylov wrapper").

What fixes them independently of the oracle's own formulas:
* p-S1 the adjoint smoother: with the colours (and line directions) in reverse
  order, one sweep's error propagator E* is the A-adjoint of the forward
  sweep's E: A E* = E^T A (a property of Gauss-Seidel on symmetric A, checked
  on dense matrices built by applying the sweeps to unit vectors);
* p-S2 the V(nu,nu) cycle with the adjoint post-smoother, applied to a right-
  hand side from a zero guess, is a symmetric positive definite operator B
  (dense, from unit vectors); V(2,1) and V(1,1) without it are not symmetric;
* p-C1 CG's defining optimality: the k-th PCG iterate minimises the A-norm of
  the error over x0 + span{z0, (BA) z0, ..., (BA)^{k-1} z0}, z0 = B r0 --
  computed here by a dense Galerkin solve in that Krylov space, not by the CG
  recurrences;
* p-C2 convergence to the direct solve; zero right-hand side; EINVAL without a
  symmetric preconditioner; fewer iterations than the plain cycle where the
  V-cycle factor is poor (the 1e6 checkerboard of config 2).
"""
import numpy as np
import pytest

from paper_2502_05279_b200 import problems as P
from tests import dense


def propagator(fn, n_int, nx, ny):
    """Dense matrix of the linear map e -> fn(e) on interior vectors."""
    E = np.zeros((n_int, n_int))
    for k in range(n_int):
        e = np.zeros(n_int)
        e[k] = 1.0
        E[:, k] = dense.to_vec(fn(dense.to_grid(e, nx, ny)))
    return E


@pytest.mark.parametrize("wl,nx,ny", [("lognormal", 7, 6), ("random9", 6, 7), ("aniso", 5, 6)])
@pytest.mark.parametrize("mode", ["point", "xline", "yline", "altline"])
def test_adjoint_smoother(orc, wl, nx, ny, mode):
    """p-S1: A E_adj = E_fwd^T A."""
    stc = P.workload(wl, nx, ny)
    st = orc.expand_stencil(stc)
    A = dense.dense_from_planes(stc)
    z = np.zeros((ny + 2, nx + 2))
    if mode == "point":
        fwd = lambda e: orc.relax(st, stc.kind, z, e, 1)  # noqa: E731
        adj = lambda e: orc.relax_adjoint(st, stc.kind, z, e, 1)  # noqa: E731
    else:
        fwd = lambda e: orc.relax_lines(st, z, e, 1, mode)  # noqa: E731
        adj = lambda e: orc.relax_lines_adjoint(st, z, e, 1, mode)  # noqa: E731
    Ef = propagator(fwd, nx * ny, nx, ny)
    Ea = propagator(adj, nx * ny, nx, ny)
    lhs, rhs = A @ Ea, Ef.T @ A
    assert np.abs(lhs - rhs).max() <= 1e-13 * np.abs(A).max()
    assert np.abs(Ef - Ea).max() > 1e-3  # the reversal changes the sweep


def vcycle_operator(orc, H, nx, ny):
    return propagator(lambda r: H.vcycle(r, np.zeros_like(r), 1), nx * ny, nx, ny)


@pytest.mark.parametrize("wl,n", [("lognormal", 15), ("random9", 15), ("checker", 15)])
@pytest.mark.parametrize("mode", ["point", "yline", "altline"])
def test_symmetric_cycle_is_spd(orc, wl, n, mode):
    """p-S2"""
    stc = P.workload(wl, n, n)
    B = vcycle_operator(orc, orc.Hierarchy(stc, nu1=1, nu2=1, relax=mode, cycle_sym=1), n, n)
    assert np.abs(B - B.T).max() <= 1e-12 * np.abs(B).max()
    assert np.linalg.eigvalsh(0.5 * (B + B.T)).min() > 0
    B21 = vcycle_operator(orc, orc.Hierarchy(stc, nu1=2, nu2=1, relax=mode, cycle_sym=1), n, n)
    B11 = vcycle_operator(orc, orc.Hierarchy(stc, nu1=1, nu2=1, relax=mode, cycle_sym=0), n, n)
    assert np.abs(B21 - B21.T).max() > 1e-8 * np.abs(B21).max()
    assert np.abs(B11 - B11.T).max() > 1e-8 * np.abs(B11).max()


@pytest.mark.parametrize("wl,n,mode", [("lognormal", 15, "point"), ("checker", 15, "point"), ("aniso", 15, "yline")])
def test_pcg_krylov_optimality(orc, wl, n, mode):
    """p-C1: x_k = argmin ||x - x*||_A over x0 + K_k(BA, B r0), k = 1, 2, 3."""
    stc = P.workload(wl, n, n)
    H = orc.Hierarchy(stc, nu1=1, nu2=1, relax=mode, cycle_sym=1)
    A = dense.dense_from_planes(stc)
    B = vcycle_operator(orc, H, n, n)
    f = P.field_uniform(n, n, seed=3)
    x0 = P.field_uniform(n, n, seed=4, scale=0.1)
    fv, xv0 = dense.to_vec(f), dense.to_vec(x0)
    xs = np.linalg.solve(A, fv)
    z = B @ (fv - A @ xv0)
    V = [z]
    for k in range(1, 4):
        got, it, hist, rc = H.pcg(f, x0, 1e-300, k)
        assert it == k and rc == orc.ENOTCONV and len(hist) == k + 1
        K = np.stack(V, axis=1)
        y = np.linalg.solve(K.T @ A @ K, K.T @ A @ (xs - xv0))
        want = xv0 + K @ y
        err0 = np.sqrt((xs - xv0) @ A @ (xs - xv0))
        d = dense.to_vec(got) - want
        assert np.sqrt(d @ A @ d) <= 1e-9 * err0, k
        V.append(B @ (A @ V[-1]))


def test_pcg_solves(orc):
    """p-C2: converged PCG equals the direct solve; history starts at ||f - A x0||
    and is recorded per iteration."""
    n = 31
    stc = P.workload("lognormal", n, n)
    H = orc.Hierarchy(stc, nu1=1, nu2=1, cycle_sym=1)
    A = dense.dense_from_planes(stc)
    f = P.rhs_const(n, n)
    x, it, hist, rc = H.pcg(f, np.zeros_like(f), 1e-12, 50)
    assert rc == orc.OK and 0 < it < 30
    assert hist[0] == pytest.approx(orc.norm2(f), rel=1e-15)
    assert hist[-1] <= 1e-12 * orc.norm2(f)
    xs = np.linalg.solve(A, dense.to_vec(f))
    assert np.abs(dense.to_vec(x) - xs).max() <= 1e-9 * np.abs(xs).max()
    x0, it0, h0, rc0 = H.pcg(np.zeros_like(f), P.field_uniform(n, n), 1e-8, 10)
    assert it0 == 0 and rc0 == orc.OK and np.all(x0 == 0)
    _, _, _, rcv = orc.Hierarchy(stc, nu1=2, nu2=1, cycle_sym=1).pcg(f, np.zeros_like(f), 1e-8, 10)
    assert rcv == orc.EINVAL


def test_pcg_beats_plain_cycle_on_checkerboard(orc):
    """p-C2 (behaviour): 1e6 checkerboard, n = 127 (config 2's operator at 1/8 size):
    the plain V(1,1) cycle needs markedly more iterations than PCG to 1e-10."""
    n = 127
    stc = P.workload("checker", n, n)
    f = P.rhs_const(n, n)
    _, it_v, _, rc_v = orc.Hierarchy(stc, nu1=1, nu2=1, cycle_sym=1).solve(f, np.zeros_like(f), 1e-10, 400)
    _, it_c, _, rc_c = orc.Hierarchy(stc, nu1=1, nu2=1, cycle_sym=1).pcg(f, np.zeros_like(f), 1e-10, 400)
    assert rc_v == orc.OK and rc_c == orc.OK
    assert it_c < 0.5 * it_v, (it_c, it_v)
