"""Pins for BoxMG's affine interpolation-correction (reading c14, SURVEY §8(f)
row 3): u(F) += (P e)(F) + r(F)/a_O(F) at the non-coarse points, u(C) += e(C).

* p-A1 the dense form u + P e + D_F^{-1} r_F, with P assembled from the
  oracle's restriction (R = P^T, tests/dense.py) and D_F the diagonal of A at
  the F points -- a wrong index, a missing F type or a C point wrongly
  included fails it;
* p-A2 what the extra term does (a property, not the formula): on a 5-point
  level right after a red-black sweep the black (X, Y) residual is zero, so
  with a zero coarse correction the affine term is one Jacobi step on the Z
  points alone -- it must zero the residual at every Z point and leave the C
  points' residual unchanged; a sign error doubles it, a misplaced term
  leaves it;
* p-A3 behaviour: on the offset 1e6 checkerboard the cycle converges faster
  with the affine term (measured 0.124 vs 0.151 per cycle at n = 63).
"""
import numpy as np
import pytest

from paper_2502_05279_b200 import problems as P
from tests import dense
from tests.test_oracle_lines import _factor


@pytest.mark.parametrize("wl,nx,ny", [("lognormal", 15, 11), ("random9", 13, 14), ("checker_off3", 23, 23)])
def test_affine_dense_form(orc, wl, nx, ny):
    """p-A1"""
    stc = P.workload(wl, nx, ny)
    st = orc.expand_stencil(stc)
    ci = orc.setup_interp(st)
    Pm = dense.dense_P_from_restriction(orc, ci, nx, ny)
    A = dense.dense_from_planes(stc)
    u0 = P.field_uniform(nx, ny, seed=1)
    r = P.field_uniform(nx, ny, seed=2)
    e = P.field_uniform(nx // 2, ny // 2, seed=3)
    J, I = np.meshgrid(np.arange(1, ny + 1), np.arange(1, nx + 1), indexing="ij")
    fpt = ((I % 2) | (J % 2)).reshape(-1).astype(bool)
    want = dense.to_vec(u0) + Pm @ dense.to_vec(e) + np.where(fpt, dense.to_vec(r) / np.diag(A), 0.0)
    got = dense.to_vec(orc.interp_add_affine(ci, e, st, r, u0))
    assert np.abs(got - want).max() <= 1e-14 * np.abs(want).max()


@pytest.mark.parametrize("wl,n", [("lognormal", 31), ("checker", 31), ("poisson", 15)])
def test_affine_term_is_a_z_point_jacobi_step(orc, wl, n):
    """p-A2"""
    stc = P.workload(wl, n, n)
    st = orc.expand_stencil(stc)
    ci = orc.setup_interp(st)
    f = P.field_uniform(n, n, seed=4)
    u = orc.relax(st, 5, f, P.field_uniform(n, n, seed=5), 1)
    r = orc.residual(st, f, u)
    J, I = np.meshgrid(np.arange(n + 2), np.arange(n + 2), indexing="ij")
    inside = (I >= 1) & (I <= n) & (J >= 1) & (J <= n)
    black = inside & ((I + J) % 2 == 1)
    zpt = inside & (I % 2 == 1) & (J % 2 == 1)
    cpt = inside & (I % 2 == 0) & (J % 2 == 0)
    scale = np.abs(r).max()
    # after red-black GS (rounding of the black update, scaled by the coefficients)
    assert np.abs(r[black]).max() <= 1e-13 * (np.abs(f).max() + np.abs(u).max() * 2 * np.abs(st).max())
    u2 = orc.interp_add_affine(ci, np.zeros((n // 2 + 2, n // 2 + 2)), st, r, u)
    r2 = orc.residual(st, f, u2)
    assert np.abs(r2[zpt]).max() <= 1e-12 * scale
    assert np.abs(r2[cpt] - r[cpt]).max() <= 1e-12 * scale
    assert np.abs(r[zpt]).max() > 1e-3 * scale  # the Z residual was not trivially zero


def test_affine_cycle_behaviour(orc):
    """p-A3"""
    n = 63
    stc = P.workload("checker_off3", n, n)
    plain = _factor(orc.Hierarchy(stc), n, 5, 10)[0]
    affine = _factor(orc.Hierarchy(stc, affine=1), n, 5, 10)[0]
    assert affine < 0.9 * plain, (affine, plain)
