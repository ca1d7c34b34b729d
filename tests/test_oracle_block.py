"""Pins for the oracle's block multi-RHS solve (c15; SURVEY §8(f) row 2,
PAPER P:512-513 §5 "solve several initial vectors in block fashion").

Expected values: the p-V1 history of config 1 (derived
independently with dense scipy) for every column of a block, the exact
homogeneity of the cycle from a zero start (x(2f) = 2 x(f), x(-f) = -x(f):
scaling by a power of two or by -1 is exact in binary floating point, and a
V-cycle from x0 = 0 is linear in f), the sparse direct solve per column, and
SPEC S:444 (b = 0 -> x = 0) for a zero column.  A column mix-up, a stopping
rule that stops at the first converged column, or a column that is not
cycled fails one of them.
"""
import numpy as np
import scipy.sparse
import scipy.sparse.linalg

from paper_2502_05279_b200 import problems as P
from tests import dense

P_V1 = [1, 3.170619e-2, 6.781695e-4, 1.594269e-5, 4.010287e-7, 9.972273e-9, 2.500688e-10]


def test_block_config1_columns(orc):
    """Config 1 (31^2 Poisson, f = h^2) in three columns f, 2f, -f: 7 block steps
    to 1e-10; every column's relative history is p-V1; the iterates are exactly
    x, 2x, -x; x matches the direct solve (p-V4)."""
    n = 31
    s = P.workload("poisson", n, n)
    f = P.rhs_const(n, n)
    h = orc.Hierarchy(s)
    F = np.stack([f, 2 * f, -f])
    U, it, hist, rc = h.solve_block(F, np.zeros_like(F), 1e-10, 50)
    assert rc == orc.OK and it == 7 and hist.shape == (8, 3)
    for c in range(3):
        rel = hist[:, c] / hist[0, c]
        assert np.allclose(rel[:7], P_V1, rtol=2e-6, atol=2e-14)
    assert np.array_equal(U[1], 2 * U[0]) and np.array_equal(U[2], -U[0])
    assert np.array_equal(hist[:, 1], 2 * hist[:, 0]) and np.array_equal(hist[:, 2], hist[:, 0])
    A = scipy.sparse.csr_matrix(dense.dense_from_planes(s))
    x = scipy.sparse.linalg.spsolve(A, dense.to_vec(f))
    assert np.abs(dense.to_vec(U[0]) - x).max() <= 1e-12


def test_block_runs_until_every_column_converges(orc):
    """Columns of different difficulty (a lognormal-D rhs and a random one, random
    x0): the block takes as many steps as the slowest column needs, and every
    column -- including one that met its test earlier -- received every step."""
    n = 63
    s = P.workload("lognormal", n, n)
    h = orc.Hierarchy(s)
    F = np.stack([P.rhs_const(n, n), P.field_uniform(n, n, seed=3), P.field_uniform(n, n, seed=4)])
    U0 = np.stack([np.zeros((n + 2, n + 2)), P.field_uniform(n, n, seed=5), np.zeros((n + 2, n + 2))])
    tol = 1e-9
    U, it, hist, rc = h.solve_block(F, U0, tol, 60)
    assert rc == orc.OK
    single = [h.solve(F[c], U0[c], tol, 60)[1] for c in range(3)]
    assert it == max(single) and min(single) < it  # the columns differ; the block waits for the slowest
    for c in range(3):
        fn = orc.norm2(F[c])
        assert hist[-1, c] <= tol * fn
        # every column was cycled `it` times (also after it met its own test)
        assert np.array_equal(U[c], h.vcycle(F[c], U0[c], it))
        assert hist[0, c] == h.residual_norm(F[c], U0[c])


def test_block_zero_column(orc):
    """SPEC S:444 per column: f_c = 0 -> x_c = 0 (whatever x0 was), norm 0, converged."""
    n = 15
    h = orc.Hierarchy(P.workload("poisson", n, n))
    F = np.stack([P.rhs_const(n, n), np.zeros((n + 2, n + 2))])
    U0 = np.stack([np.zeros((n + 2, n + 2)), P.field_uniform(n, n, seed=9)])
    U, it, hist, rc = h.solve_block(F, U0, 1e-8, 30)
    assert rc == orc.OK and it > 0
    assert np.all(U[1] == 0.0) and np.all(hist[:, 1] == 0.0)


def test_block_not_converged(orc):
    """maxiter reached with one column unconverged -> ENOTCONV, maxiter steps."""
    n = 31
    h = orc.Hierarchy(P.workload("checker", n, n))
    F = np.stack([P.rhs_const(n, n), P.field_uniform(n, n, seed=1)])
    U, it, hist, rc = h.solve_block(F, np.zeros_like(F), 1e-14, 3)
    assert rc == orc.ENOTCONV and it == 3 and hist.shape == (4, 2)


def test_block_pcg_columns(orc):
    """c13 x c15: block PCG = independent PCG per column.  Pinned by exact
    homogeneity (CG from x0 = 0 on 2f / -f runs the same alpha, beta on scaled
    vectors: x(2f) = 2 x(f), x(-f) = -x(f), same iteration counts) and the zero
    column (x = 0, 0 iterations)."""
    n = 63
    st = P.workload("checker", n, n)
    h = orc.Hierarchy(st, nu1=1, nu2=1, cycle_sym=1)
    f = P.rhs_const(n, n)
    F = np.stack([f, 2 * f, -f, np.zeros_like(f)])
    U, its, hists, rcs = h.pcg_block(F, np.zeros_like(F), 1e-10, 100)
    assert rcs == [orc.OK] * 4 and its[0] == its[1] == its[2] > 0 and its[3] == 0
    assert np.array_equal(U[1], 2 * U[0]) and np.array_equal(U[2], -U[0]) and np.all(U[3] == 0)
    assert np.array_equal(hists[1], 2 * hists[0]) and np.array_equal(hists[2], hists[0])
