"""Block multi-RHS V-cycle (c15) through the
C ABI (bmg_vcycle_block, bmg_residual_norm_block, bmg_solve_block).

Each column of a block cycle is checked (i) against the single-RHS per-step
cycle of the same handle parameters on that column -- the same per-point
operations, but nvcc may contract a*b + c*d to either FMA in the single
kernels, while the block kernels fix the source order with __fma_rn; so the
two agree to rounding (each is within the DESIGN §7 1e-12 of the oracle, so
2e-12 of each other), not bit for bit -- and
(ii) against the oracle at the DESIGN §7 tolerance; the block solve against
the oracle's block solve (same step count, per-column histories at the §7
norm tolerance).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from paper_2502_05279_b200 import bmg, problems as P  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__ as ge

    ge.build_lib()


def params(fused=1, **kw):
    prm = bmg.bmg_params_default()
    prm.fused = fused
    for k, v in kw.items():
        setattr(prm, k, v)
    return prm


def columns(nx, ny, K, seed):
    F = [P.field_uniform(nx, ny, seed=seed + 2 * c) for c in range(K)]
    X = [P.field_uniform(nx, ny, seed=seed + 2 * c + 1) for c in range(K)]
    return F, X


def assert_iterate_close(g, o, rtol=1e-12):
    tol = rtol * np.maximum(np.abs(o), np.abs(o).max())
    err = np.abs(g - o)
    assert np.all(err <= tol), (err.max(), np.abs(o).max())


CASES = [("poisson", 31, 31, 1), ("lognormal", 63, 63, 2), ("random9", 47, 33, 3), ("checker", 127, 127, 4),
         ("checker_off3", 95, 47, 8), ("lognormal", 300, 257, 4), ("random9", 200, 131, 5), ("aniso", 64, 30, 2),
         ("lognormal", 9, 8, 6), ("poisson", 1, 1, 2)]


@pytest.mark.parametrize("wl,nx,ny,K", CASES)
def test_block_vcycle_vs_single(wl, nx, ny, K):
    st = P.workload(wl, nx, ny)
    s = bmg.Solver(st, params(fused=0))
    F, X = columns(nx, ny, K, 100)
    Fb, Xb = s.block_grid(K, F), s.block_grid(K, X)
    s.vcycle_block(Fb, Xb, 2)
    torch.cuda.synchronize()
    got = bmg.from_device_block(Xb, nx)
    for c in range(K):
        x = s.grid(X[c])
        s.vcycle(s.grid(F[c]), x, 2)
        torch.cuda.synchronize()
        assert_iterate_close(got[c], bmg.from_device(x, nx), rtol=2e-12)
    assert torch.equal(Fb, s.block_grid(K, F))  # rhs untouched
    s.close()


@pytest.mark.parametrize("wl,nx,ny,K", CASES[:7])
def test_block_vcycle_oracle(orc, wl, nx, ny, K):
    st = P.workload(wl, nx, ny)
    s = bmg.Solver(st)  # default handle (fused single-RHS path elsewhere; the block path is its own)
    h = orc.Hierarchy(st)
    F, X = columns(nx, ny, K, 200)
    Xb = s.block_grid(K, X)
    s.vcycle_block(s.block_grid(K, F), Xb, 1)
    torch.cuda.synchronize()
    got = bmg.from_device_block(Xb, nx)
    for c in range(K):
        assert_iterate_close(got[c], h.vcycle(F[c], X[c], 1))
    s.close()


@pytest.mark.parametrize("opt", [dict(cycle_sym=1, nu1=1, nu2=1), dict(affine=1), dict(nu1=0, nu2=2),
                                 dict(cycle_sym=1, nu1=2, nu2=2),
                                 # the one-pass sweeps' ping-pong for every parity of nu1 / nu2
                                 dict(nu1=1, nu2=2), dict(nu1=3, nu2=1), dict(nu1=2, nu2=0), dict(nu1=1, nu2=1)])
@pytest.mark.parametrize("wl,nx,ny", [("lognormal", 63, 63), ("random9", 65, 47)])
def test_block_variants_vs_single(orc, wl, nx, ny, opt):
    """c12 reversed post-smoother, c14 affine correction, nu1 = 0 (no vanishing
    restriction): column for column the per-step single cycle and the oracle."""
    st = P.workload(wl, nx, ny)
    s = bmg.Solver(st, params(fused=0, **opt))
    K = 3
    F, X = columns(nx, ny, K, 300)
    Xb = s.block_grid(K, X)
    s.vcycle_block(s.block_grid(K, F), Xb, 2)
    torch.cuda.synchronize()
    got = bmg.from_device_block(Xb, nx)
    for c in range(K):
        x = s.grid(X[c])
        s.vcycle(s.grid(F[c]), x, 2)
        torch.cuda.synchronize()
        assert_iterate_close(got[c], bmg.from_device(x, nx), rtol=2e-12)
    h = orc.Hierarchy(st, nu1=opt.get("nu1", 2), nu2=opt.get("nu2", 1), cycle_sym=opt.get("cycle_sym", 0),
                      affine=opt.get("affine", 0))
    for c in range(K):
        assert_iterate_close(got[c], h.vcycle(F[c], X[c], 2))
    s.close()


@pytest.mark.parametrize("wl,n,K,tol", [("poisson", 31, 3, 1e-10), ("lognormal", 63, 4, 1e-9),
                                        ("checker", 127, 2, 1e-8), ("random9", 65, 5, 1e-9)])
def test_block_solve_parity(orc, wl, n, K, tol):
    st = P.workload(wl, n, n)
    s = bmg.Solver(st)
    h = orc.Hierarchy(st)
    F = [P.rhs_const(n, n)] + [P.field_uniform(n, n, seed=400 + c) for c in range(K - 1)]
    X = [np.zeros((n + 2, n + 2))] + [P.field_uniform(n, n, seed=500 + c) for c in range(K - 1)]
    Xb = s.block_grid(K, X)
    it, hist, rc = s.solve_block(s.block_grid(K, F), Xb, tol, 100)
    Uo, ito, histo, rco = h.solve_block(np.stack(F), np.stack(X), tol, 100)
    assert rc == rco == 0 and it == ito and hist.shape == histo.shape
    floor = 1e-12 * histo[0]
    assert np.all(np.abs(hist - histo) <= 1e-10 * histo + floor), np.abs(hist / histo - 1).max()
    got = bmg.from_device_block(Xb, n)
    for c in range(K):
        assert_iterate_close(got[c], Uo[c], rtol=1e-10)
    # per-column norms through the ABI agree with the last history row
    nb = bmg.bmg_residual_norm_block(s.h, K, s.block_grid(K, F), Xb)
    assert np.array_equal(nb, hist[-1])
    s.close()


def test_block_solve_zero_column_and_realloc(orc):
    """SPEC S:444 per column; switching nrhs reallocates the workspace and re-captures."""
    n = 63
    st = P.workload("lognormal", n, n)
    s = bmg.Solver(st)
    h = orc.Hierarchy(st)
    F = [P.rhs_const(n, n), np.zeros((n + 2, n + 2))]
    X = [np.zeros((n + 2, n + 2)), P.field_uniform(n, n, seed=7)]
    Xb = s.block_grid(2, X)
    it, hist, rc = s.solve_block(s.block_grid(2, F), Xb, 1e-8, 50)
    assert rc == 0 and it > 0
    got = bmg.from_device_block(Xb, n)
    assert np.all(got[1] == 0.0) and np.all(hist[:, 1] == 0.0)
    for K in (4, 1, 2):  # other block widths on the same handle
        Fk, Xk = columns(n, n, K, 600)
        Xkb = s.block_grid(K, Xk)
        s.vcycle_block(s.block_grid(K, Fk), Xkb, 1)
        torch.cuda.synchronize()
        gk = bmg.from_device_block(Xkb, n)
        for c in range(K):
            assert_iterate_close(gk[c], h.vcycle(Fk[c], Xk[c], 1))
    s.close()


def test_block_errors():
    n = 31
    st = P.workload("poisson", n, n)
    s = bmg.Solver(st)
    for K in (0, bmg.BMG_MAX_NRHS + 1):
        with pytest.raises(bmg.BmgError) as e:
            bmg.bmg_vcycle_block(s.h, K, s.block_grid(2), s.block_grid(2))
        assert e.value.status == bmg.BMG_EINVAL
    # even nrhs needs 16-byte aligned rhs/x
    buf = torch.zeros((n + 2) * s.pitch * 2 + 1, dtype=torch.float64, device="cuda")
    with pytest.raises(bmg.BmgError) as e:
        bmg.bmg_vcycle_block(s.h, 2, buf[1:], s.block_grid(2))
    assert e.value.status == bmg.BMG_EINVAL
    s.close()
    prm = params(relax=bmg.BMG_RELAX_YLINES)
    s = bmg.Solver(st, prm)
    with pytest.raises(bmg.BmgError) as e:
        bmg.bmg_vcycle_block(s.h, 2, s.block_grid(2), s.block_grid(2))
    assert e.value.status == bmg.BMG_EINVAL
    s.close()



def test_block_fullsize_vs_single():
    """At the bench size (8191^2, BASELINE config 4) and the bench's K: every
    column of one block cycle against the fused single-RHS cycle on that column
    (each within DESIGN §7 of the oracle, hence 2e-12 of each other), all points."""
    n, K = 8191, 8
    # lognormal D with sigma = 1 (sigma = 2 is EINVAL from 1023^2 up, test_gpu_fullsize.py)
    st = P.stencil5_from_D(P.d_lognormal(n, n, sigma=1.0))
    s = bmg.Solver(st)
    gen = torch.Generator(device="cuda").manual_seed(11)
    fb = s.block_grid(K)
    fb[1:-1, 1:n + 1, :] = 2 * torch.rand((n, n, K), generator=gen, device="cuda", dtype=torch.float64) - 1
    xb = s.block_grid(K)
    s.vcycle_block(fb, xb, 1)
    for c in (0, 5, 7):
        f = s.grid()
        f[:, :] = fb[:, :, c]
        x = s.grid()
        s.vcycle(f, x, 1)
        torch.cuda.synchronize()
        g, o = xb[:, :, c], x
        tol = 2e-12 * torch.maximum(o.abs(), o.abs().max())
        assert bool(((g - o).abs() <= tol).all()), float((g - o).abs().max())
    s.close()


@pytest.mark.parametrize("wl,n,K,tol", [("checker", 127, 3, 1e-10), ("lognormal", 63, 4, 1e-10),
                                        ("random9", 65, 2, 1e-10), ("checker", 511, 8, 1e-9)])
def test_block_pcg_parity(orc, wl, n, K, tol):
    """bmg_pcg_block: every column against its own oracle PCG (c13) -- its
    iteration count (the first step whose norm meets the test), its history up
    to there (DESIGN §7 norms) and its iterate (1e-10, as tests/test_gpu_pcg.py);
    the block takes the slowest column's count; frozen columns repeat their norm."""
    st = P.workload(wl, n, n)
    prm = bmg.bmg_params_default()
    prm.nu1, prm.nu2, prm.cycle_sym = 1, 1, 1
    s = bmg.Solver(st, prm)
    h = orc.Hierarchy(st, nu1=1, nu2=1, cycle_sym=1)
    F = [P.rhs_const(n, n)] + [P.field_uniform(n, n, seed=700 + c) for c in range(K - 1)]
    X = [np.zeros((n + 2, n + 2))] + [P.field_uniform(n, n, seed=800 + c) for c in range(K - 1)]
    xb = s.block_grid(K, X)
    it, hist, rc = s.pcg_block(s.block_grid(K, F), xb, tol, 200)
    Uo, its, hists, rcs = h.pcg_block(np.stack(F), np.stack(X), tol, 200)
    assert rc == 0 and all(r == 0 for r in rcs) and it == max(its)
    got = bmg.from_device_block(xb, n)
    for c in range(K):
        fn = np.linalg.norm(F[c][1:-1, 1:-1])
        kc = int(np.argmax(hist[:, c] <= tol * fn))
        assert kc == its[c], (c, kc, its[c])
        ho = hists[c]
        assert np.all(np.abs(hist[: kc + 1, c] - ho) <= 1e-10 * ho + 1e-12 * ho[0])
        assert np.all(hist[kc:, c] == hist[kc, c])  # frozen after convergence
        assert_iterate_close(got[c], Uo[c], rtol=1e-10)
    s.close()
