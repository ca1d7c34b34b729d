"""Race evidence for the fused streaming legs (kernels_fused.cu), whose shared-memory
ring is ordered by raw-PTX mbarrier arrive / try_wait -- synchronisation that
compute-sanitizer racecheck does not model (tools/mb_racecheck.cu: a race-free
producer/consumer pair through one mbarrier is reported as a hazard;
profiles/r02_sanitizer.txt).  A real race in the pipeline would make the legs
nondeterministic or differ from the per-step kernels, which share the per-point
arithmetic (DESIGN §3 c10) and are synchronised by kernel boundaries: both are
checked bitwise here, over many launches, for the 5- and 9-point legs in the
shapes that exercise several CTAs, row chunks, a ragged strip and the REV order."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from paper_2502_05279_b200 import bmg, problems as P  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__ as ge

    ge.build_lib()


def _legs(wl, nx, ny, fused, sym, reps):
    prm = bmg.bmg_params_default()
    prm.fused = fused
    prm.cycle_sym = sym
    if sym:
        prm.nu1 = prm.nu2 = 1
    s = bmg.Solver(P.workload(wl, nx, ny), prm)
    f = s.grid(P.field_uniform(nx, ny, seed=1))
    u0 = s.grid(P.field_uniform(nx, ny, seed=2))
    ec = s.level_grid(1, P.field_uniform(nx // 2, ny // 2, seed=3))
    outs = []
    for _ in range(reps):
        uo, fc, uc, u2 = s.grid(), s.level_grid(1), s.level_grid(1), s.grid()
        bmg.bmg_smooth_restrict(s.h, 0, f, u0, uo, fc, uc)
        bmg.bmg_correct_smooth(s.h, 0, f, u0, ec, u2)
        torch.cuda.synchronize()
        outs.append((uo.cpu().numpy(), fc.cpu().numpy(), u2.cpu().numpy()))
    s.close()
    return outs


@pytest.mark.parametrize("wl,nx,ny,sym", [("checker", 1023, 1021, 0), ("random9", 1021, 1023, 0),
                                          ("lognormal", 300, 257, 0), ("lognormal", 299, 250, 1),
                                          ("aniso", 1023, 777, 0)])
def test_fused_legs_deterministic_and_equal_to_per_step(wl, nx, ny, sym):
    fused = _legs(wl, nx, ny, 1, sym, 25)
    ref = _legs(wl, nx, ny, 0, sym, 1)[0]
    for run in fused[1:]:  # every launch bitwise the first (a race would scatter the bits)
        for a, b in zip(run, fused[0]):
            assert np.array_equal(a, b)
    uo, fc, u2 = fused[0]
    # the down-leg iterate is bitwise the per-step kernels'; the restricted residual and
    # the up leg's interpolation sum the same terms in another order (FMA contraction
    # of the fused legs' row-ring expressions), so those agree to rounding
    assert np.array_equal(uo, ref[0])
    assert np.abs(fc - ref[1]).max() <= 1e-13 * np.abs(ref[1]).max()
    assert np.abs(u2 - ref[2]).max() <= 1e-13 * np.abs(ref[2]).max()
