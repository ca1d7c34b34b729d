"""CPU-side checks of the boundary: libbmg.so loads (no GPU needed) and
exports every entry point include/bmg.h declares; the binding covers them."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    with open(os.path.join(ROOT, "include", "bmg.h")) as fh:
        txt = fh.read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(bmg_[a-z_0-9]+)\s*\(", txt)))


@pytest.fixture(scope="module")
def libbmg():
    import __graft_entry__ as ge

    ge.build_lib()
    from paper_2502_05279_b200 import bmg

    return bmg.lib()


def test_header_declares_expected(libbmg):
    syms = header_symbols()
    assert "bmg_setup" in syms and "bmg_vcycle" in syms and "bmg_solve" in syms
    from paper_2502_05279_b200 import bmg

    assert set(syms) == set(bmg.EXPORTS)


def test_library_exports_every_header_symbol(libbmg):
    for s in header_symbols():
        assert getattr(libbmg, s) is not None


def test_nm_exports_are_unmangled(libbmg):
    import subprocess

    from paper_2502_05279_b200 import bmg

    out = subprocess.run(["nm", "-D", "--defined-only", bmg.LIB_PATH], capture_output=True, text=True).stdout
    defined = {ln.split()[-1] for ln in out.splitlines() if ln.strip()}
    for s in header_symbols():
        assert s in defined, s


def test_host_only_calls_without_gpu(libbmg):
    from paper_2502_05279_b200 import bmg

    p = bmg.bmg_params_default()
    assert (p.nu1, p.nu2, p.coarsest, p.fused) == (2, 1, 3, 1)
    assert libbmg.bmg_strerror(bmg.BMG_ENOTSPD).startswith(b"coarsest")
    # argument validation happens before any device work
    st = bmg.bmg_stencil_t()
    st.kind, st.nx, st.ny, st.pitch = 7, 3, 3, 5
    h = ctypes.c_void_p()
    assert libbmg.bmg_setup(ctypes.byref(st), None, None, ctypes.byref(h)) == bmg.BMG_EINVAL
    assert b"kind" in libbmg.bmg_last_error_detail()
    assert libbmg.bmg_destroy(None) == bmg.BMG_OK
    # the newer entry points reject a null handle / bad sizes before any device work
    d = ctypes.c_double()
    it = ctypes.c_int()
    assert libbmg.bmg_pcg(None, None, None, 1e-8, 10, ctypes.byref(it), None, None) == bmg.BMG_EINVAL
    for K in (1, 0, bmg.BMG_MAX_NRHS + 1):
        assert libbmg.bmg_vcycle_block(None, K, None, None, 1, None) == bmg.BMG_EINVAL
        assert libbmg.bmg_residual_norm_block(None, K, None, None, ctypes.byref(d), None) == bmg.BMG_EINVAL
        assert libbmg.bmg_solve_block(None, K, None, None, 1e-8, 10, ctypes.byref(it), None, None) == bmg.BMG_EINVAL
    assert b"nrhs" in libbmg.bmg_last_error_detail()


def test_product_package_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2502_05279_b200")
    for dirpath, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                with open(os.path.join(dirpath, fn)) as fh:
                    src = fh.read()
                assert "import oracle" not in src and "from oracle" not in src and "bmg_oracle" not in src, fn


def test_missing_library_fails_loudly(tmp_path, monkeypatch):
    from paper_2502_05279_b200 import bmg

    monkeypatch.setattr(bmg, "_lib", None)
    monkeypatch.setattr(bmg, "LIB_PATH", str(tmp_path / "nope.so"))
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        bmg.lib()


def header3_symbols():
    with open(os.path.join(ROOT, "include", "bmg3.h")) as fh:
        txt = fh.read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(bmg3_[a-z_0-9]+)\s*\(", txt)))


def test_3d_header_exports_and_binding(libbmg):
    """include/bmg3.h: every declared entry point is exported
    unmangled and bound by paper_2502_05279_b200/bmg3.py."""
    import subprocess

    from paper_2502_05279_b200 import bmg, bmg3

    syms = header3_symbols()
    assert set(syms) == set(bmg3.EXPORTS3)
    out = subprocess.run(["nm", "-D", "--defined-only", bmg.LIB_PATH], capture_output=True, text=True).stdout
    defined = {ln.split()[-1] for ln in out.splitlines() if ln.strip()}
    for s in syms:
        assert s in defined, s
    bmg3.lib()


def test_3d_host_only_validation(libbmg):
    from paper_2502_05279_b200 import bmg, bmg3

    p = bmg3.bmg3_params_default()
    assert (p.nu1, p.nu2, p.coarsest, p.max_levels, p.relax) == (2, 1, 3, 0, 0)
    L = bmg3.lib()
    st = bmg3.bmg3_stencil_t()
    st.kind, st.nx, st.ny, st.nz, st.pitch, st.plane_stride = 9, 3, 3, 3, 5, 25
    h = ctypes.c_void_p()
    assert L.bmg3_setup(ctypes.byref(st), None, None, ctypes.byref(h)) == bmg.BMG_EINVAL
    st.kind, st.plane_stride = 7, 20  # plane_stride < pitch*(ny+2)
    assert L.bmg3_setup(ctypes.byref(st), None, None, ctypes.byref(h)) == bmg.BMG_EINVAL
    st.plane_stride = 25  # planes NULL
    assert L.bmg3_setup(ctypes.byref(st), None, None, ctypes.byref(h)) == bmg.BMG_EINVAL
    assert b"NULL" in L.bmg_last_error_detail()
    d = ctypes.c_double()
    assert L.bmg3_vcycle(None, None, None, 1, None) == bmg.BMG_EINVAL
    assert L.bmg3_residual_norm(None, None, None, ctypes.byref(d), None) == bmg.BMG_EINVAL
    assert L.bmg3_destroy(None) == bmg.BMG_OK
