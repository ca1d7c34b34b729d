"""Parity at the BASELINE bench size (8191^2 interior, the launch configuration
bench.py times: fused level-0 legs), on sampled outputs the oracle computes
window by window (DESIGN §7 tolerances).

The down leg's smoothed iterate at a point depends only on inputs within 4
points (two red-black sweeps), its residual within 5, and a coarse right-hand
side within 6 fine points; the up leg's result within 2 fine / 1 coarse point.
So the oracle's own steps (relax, residual, setup_interp, restrict,
interp_add) run on a window of the global problem -- the window's ring holding
the true input values and its stencil keeping the couplings into that ring --
reproduce the global result exactly on the window's central block (margin 8).
Windows sit at the four corners (the true Dirichlet boundary inside them) and
in the interior.  The stencil is the lognormal-D operator (non-trivial
coefficients and interpolation weights everywhere; sigma = 1), f and u random.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from paper_2502_05279_b200 import bmg, problems as P  # noqa: E402

N = 8191
WN = 48  # window interior size (even)
MARGIN = 8


@pytest.fixture(scope="module")
def big():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__ as ge

    ge.build_lib()
    # lognormal D with sigma = 1 (the sigma = 2 parity field of DESIGN §4 makes some coarse
    # Galerkin rows lose the collapse's positive denominator at these sizes -- reading
    # c3 (iii) EINVAL, on the oracle as on the GPU, from 1023^2 up)
    st = P.stencil5_from_D(P.d_lognormal(N, N, sigma=1.0))
    s = bmg.Solver(st)
    yield st, s
    s.close()


def window_stencil(st, j0, i0):
    """Full 9-entry stencil (fig:stencil_operator order) of the window whose local
    (0,0) is global (i0, j0); couplings into the GLOBAL ring dropped, couplings
    into the window's own ring kept."""
    w = WN + 2
    O, W, S = st.planes["O"], st.planes["W"], st.planes["S"]
    J, I = np.meshgrid(np.arange(j0, j0 + w), np.arange(i0, i0 + w), indexing="ij")
    out = np.zeros((w, w, 9))
    inside = (I >= 1) & (I <= N) & (J >= 1) & (J <= N)

    def g(plane, jj, ii):
        ok = (ii >= 0) & (ii <= N + 1) & (jj >= 0) & (jj <= N + 1)
        return np.where(ok, plane[np.clip(jj, 0, N + 1), np.clip(ii, 0, N + 1)], 0.0)

    def keep(di, dj):  # coupling target inside the global interior
        return (I + di >= 1) & (I + di <= N) & (J + dj >= 1) & (J + dj <= N)

    out[..., 1] = np.where(keep(0, -1), g(S, J, I), 0.0)          # S
    out[..., 3] = np.where(keep(-1, 0), g(W, J, I), 0.0)          # W
    out[..., 4] = g(O, J, I)                                       # O
    out[..., 5] = np.where(keep(1, 0), g(W, J, I + 1), 0.0)       # E = W(i+1, j)
    out[..., 7] = np.where(keep(0, 1), g(S, J + 1, I), 0.0)       # N = S(i, j+1)
    out[~inside] = 0.0
    return out


WINDOWS = [(0, 0), (0, N + 1 - WN - 2 + 1), (N + 1 - WN - 2 + 1, 0), (4000, 5200), (N + 1 - WN - 2 + 1,) * 2]


def central(a, m=MARGIN):
    return a[m:-m, m:-m]


def test_down_leg_fullsize_windows(orc, big):
    st, s = big
    rng = np.random.default_rng(7)
    f = np.zeros((N + 2, N + 2))
    u0 = np.zeros((N + 2, N + 2))
    f[1:-1, 1:-1] = rng.uniform(-1, 1, (N, N))
    u0[1:-1, 1:-1] = rng.uniform(-1, 1, (N, N))
    fd, ud, uo = s.grid(f), s.grid(u0), s.grid()
    fc, uc = s.level_grid(1), s.level_grid(1)
    bmg.bmg_smooth_restrict(s.h, 0, fd, ud, uo, fc, uc)
    torch.cuda.synchronize()
    uo_h = uo[:, : N + 2].cpu().numpy()
    fc_h = fc[:, : N // 2 + 2].cpu().numpy()
    for (j0, i0) in WINDOWS:
        j0 -= j0 & 1  # window origin on even global indices: coarse (I,J) <-> fine (2I,2J)
        i0 -= i0 & 1
        sw = window_stencil(st, j0, i0)
        fw = f[j0:j0 + WN + 2, i0:i0 + WN + 2].copy()
        uw = u0[j0:j0 + WN + 2, i0:i0 + WN + 2].copy()
        ur = orc.relax(sw, 5, fw, uw, 2)
        got = uo_h[j0:j0 + WN + 2, i0:i0 + WN + 2]
        ref = central(ur)
        tol = 1e-12 * np.maximum(np.abs(ref), np.abs(ref).max())
        assert np.all(np.abs(central(got) - ref) <= tol), ((j0, i0), np.abs(central(got) - ref).max())
        ci = orc.setup_interp(sw)
        fcw = orc.restrict(ci, orc.residual(sw, fw, ur))
        J0, I0 = j0 // 2, i0 // 2
        gotc = fc_h[J0:J0 + WN // 2 + 2, I0:I0 + WN // 2 + 2]
        refc = central(fcw, MARGIN // 2)
        tolc = 1e-12 * np.maximum(np.abs(refc), np.abs(refc).max())
        assert np.all(np.abs(central(gotc, MARGIN // 2) - refc) <= tolc), ((j0, i0), "fc")


def test_up_leg_fullsize_windows(orc, big):
    st, s = big
    rng = np.random.default_rng(8)
    f = np.zeros((N + 2, N + 2))
    u0 = np.zeros((N + 2, N + 2))
    e = np.zeros((N // 2 + 2, N // 2 + 2))
    f[1:-1, 1:-1] = rng.uniform(-1, 1, (N, N))
    u0[1:-1, 1:-1] = rng.uniform(-1, 1, (N, N))
    e[1:-1, 1:-1] = rng.uniform(-1, 1, (N // 2, N // 2))
    uo = s.grid()
    bmg.bmg_correct_smooth(s.h, 0, s.grid(f), s.grid(u0), s.level_grid(1, e), uo)
    torch.cuda.synchronize()
    uo_h = uo[:, : N + 2].cpu().numpy()
    for (j0, i0) in WINDOWS:
        j0 -= j0 & 1
        i0 -= i0 & 1
        sw = window_stencil(st, j0, i0)
        ci = orc.setup_interp(sw)
        ew = e[j0 // 2:j0 // 2 + WN // 2 + 2, i0 // 2:i0 // 2 + WN // 2 + 2].copy()
        uw = orc.interp_add(ci, ew, u0[j0:j0 + WN + 2, i0:i0 + WN + 2].copy())
        ur = orc.relax(sw, 5, f[j0:j0 + WN + 2, i0:i0 + WN + 2].copy(), uw, 1)
        got = uo_h[j0:j0 + WN + 2, i0:i0 + WN + 2]
        ref = central(ur)
        tol = 1e-12 * np.maximum(np.abs(ref), np.abs(ref).max())
        assert np.all(np.abs(central(got) - ref) <= tol), ((j0, i0), np.abs(central(got) - ref).max())
