"""Thin ctypes binding of the 3-D entry points of libbmg.so (include/bmg3.h),
same names as the C ABI.  Argument marshalling only (every step runs in the
CUDA kernels behind the ABI); device arrays are torch CUDA float64 tensors of
shape (nz+2, ny+2, pitch); no CPU fallback (libbmg.so missing -> RuntimeError).
"""
from __future__ import annotations

import ctypes

import numpy as np

from .bmg import BMG_OK, BMG_ENOTCONV, _check, _ptr, _stream, lib as _lib2

EXPORTS3 = (
    "bmg3_params_default", "bmg3_setup", "bmg3_vcycle", "bmg3_solve", "bmg3_residual_norm", "bmg3_relax",
    "bmg3_num_levels", "bmg3_level_shape", "bmg3_cycle_kernel_count", "bmg3_export_level", "bmg3_destroy",
)

BMG3_RELAX_POINT, BMG3_RELAX_PLANES = 0, 1
RELAX3 = {"point": BMG3_RELAX_POINT, "planes": BMG3_RELAX_PLANES}


class bmg3_stencil_t(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int), ("nx", ctypes.c_int), ("ny", ctypes.c_int), ("nz", ctypes.c_int),
                ("pitch", ctypes.c_longlong), ("plane_stride", ctypes.c_longlong), ("plane", ctypes.c_void_p * 14)]


class bmg3_params_t(ctypes.Structure):
    _fields_ = [("nu1", ctypes.c_int), ("nu2", ctypes.c_int), ("coarsest", ctypes.c_int),
                ("max_levels", ctypes.c_int), ("relax", ctypes.c_int)]


_done = False


def lib():
    global _done
    L = _lib2()
    if not _done:
        vp, i, d = ctypes.c_void_p, ctypes.c_int, ctypes.c_double
        ip, dp = ctypes.POINTER(i), ctypes.POINTER(d)
        sig = {
            "bmg3_params_default": (None, [ctypes.POINTER(bmg3_params_t)]),
            "bmg3_setup": (i, [ctypes.POINTER(bmg3_stencil_t), ctypes.POINTER(bmg3_params_t), vp, ctypes.POINTER(vp)]),
            "bmg3_vcycle": (i, [vp, vp, vp, i, vp]),
            "bmg3_solve": (i, [vp, vp, vp, d, i, ip, dp, vp]),
            "bmg3_residual_norm": (i, [vp, vp, vp, dp, vp]),
            "bmg3_relax": (i, [vp, vp, vp, i, vp]),
            "bmg3_num_levels": (i, [vp, ip]),
            "bmg3_level_shape": (i, [vp, i, ip, ip, ip, ip]),
            "bmg3_cycle_kernel_count": (i, [vp, ip]),
            "bmg3_export_level": (i, [vp, i, dp, dp]),
            "bmg3_destroy": (i, [vp]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _done = True
    return L


def bmg3_params_default(**kw) -> bmg3_params_t:
    p = bmg3_params_t()
    lib().bmg3_params_default(ctypes.byref(p))
    for k, v in kw.items():
        setattr(p, k, RELAX3.get(v, v) if k == "relax" else v)
    return p


def bmg3_setup(planes, kind, nx, ny, nz, pitch, plane_stride, params=None, stream=None):
    st = bmg3_stencil_t()
    st.kind, st.nx, st.ny, st.nz, st.pitch, st.plane_stride = kind, nx, ny, nz, pitch, plane_stride
    for q, p in enumerate(planes):
        st.plane[q] = p.data_ptr()
    h = ctypes.c_void_p()
    _check(lib().bmg3_setup(ctypes.byref(st), ctypes.byref(params) if params is not None else None, _stream(stream),
                            ctypes.byref(h)), "bmg3_setup")
    return h


def bmg3_vcycle(h, rhs, x, ncycles=1, stream=None):
    _check(lib().bmg3_vcycle(h, _ptr(rhs), _ptr(x), ncycles, _stream(stream)), "bmg3_vcycle")


def bmg3_solve(h, rhs, x, tol, maxiter, stream=None):
    it = ctypes.c_int()
    hist = np.zeros(maxiter + 1)
    rc = lib().bmg3_solve(h, _ptr(rhs), _ptr(x), tol, maxiter, ctypes.byref(it),
                          hist.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), _stream(stream))
    _check(rc, "bmg3_solve", ok=(BMG_OK, BMG_ENOTCONV))
    return it.value, hist[: it.value + 1], rc


def bmg3_residual_norm(h, rhs, x, stream=None) -> float:
    out = ctypes.c_double()
    _check(lib().bmg3_residual_norm(h, _ptr(rhs), _ptr(x), ctypes.byref(out), _stream(stream)), "bmg3_residual_norm")
    return out.value


def bmg3_relax(h, rhs, x, nsweeps=1, stream=None):
    _check(lib().bmg3_relax(h, _ptr(rhs), _ptr(x), nsweeps, _stream(stream)), "bmg3_relax")


def bmg3_num_levels(h) -> int:
    L = ctypes.c_int()
    _check(lib().bmg3_num_levels(h, ctypes.byref(L)), "bmg3_num_levels")
    return L.value


def bmg3_level_shape(h, level):
    a = [ctypes.c_int() for _ in range(4)]
    _check(lib().bmg3_level_shape(h, level, *[ctypes.byref(x) for x in a]), "bmg3_level_shape")
    return tuple(x.value for x in a)


def bmg3_cycle_kernel_count(h) -> int:
    c = ctypes.c_int()
    _check(lib().bmg3_cycle_kernel_count(h, ctypes.byref(c)), "bmg3_cycle_kernel_count")
    return c.value


def bmg3_export_level(h, level):
    """(stencil (14, nz+2, ny+2, nx+2), ci (26, ncz+2, ncy+2, ncx+2) or None) as host arrays."""
    nx, ny, nz, _ = bmg3_level_shape(h, level)
    st = np.zeros((14, nz + 2, ny + 2, nx + 2))
    L = bmg3_num_levels(h)
    ci = np.zeros((26, nz // 2 + 2, ny // 2 + 2, nx // 2 + 2)) if level + 1 < L else None
    dp = ctypes.POINTER(ctypes.c_double)
    _check(lib().bmg3_export_level(h, level, st.ctypes.data_as(dp), ci.ctypes.data_as(dp) if ci is not None else None),
           "bmg3_export_level")
    return st, ci


def bmg3_destroy(h):
    if h is not None and h.value:
        _check(lib().bmg3_destroy(h), "bmg3_destroy")


# --------------------------------------------------------------------------- helpers
def default_pitch3(nx: int) -> int:
    return (nx + 2 + 31) // 32 * 32


def to_device3(a: np.ndarray, pitch: int, device="cuda"):
    """(nz+2, ny+2, nx+2) host array -> (nz+2, ny+2, pitch) device float64 tensor (pad zero)."""
    import torch

    t = torch.zeros((a.shape[0], a.shape[1], pitch), dtype=torch.float64, device=device)
    t[:, :, : a.shape[2]] = torch.from_numpy(np.ascontiguousarray(a)).to(device)
    return t


def from_device3(t, nx: int) -> np.ndarray:
    return t[:, :, : nx + 2].cpu().numpy().copy()


class Solver3:
    """Owner of a bmg3_solver_t for a problems3d.Stencil3 (device copies kept)."""

    def __init__(self, stencil, relax="point", nu1=2, nu2=1, coarsest=3, max_levels=0, pitch=None, device="cuda"):
        self.nx, self.ny, self.nz, self.kind = stencil.nx, stencil.ny, stencil.nz, stencil.kind
        self.pitch = pitch or default_pitch3(self.nx)
        self.stride = self.pitch * (self.ny + 2)
        self.device = device
        planes = [to_device3(p, self.pitch, device) for p in stencil.plane_list()]
        prm = bmg3_params_default(nu1=nu1, nu2=nu2, coarsest=coarsest, max_levels=max_levels, relax=relax)
        import time

        import torch

        torch.cuda.synchronize()
        t0 = time.perf_counter()
        self.h = bmg3_setup(planes, self.kind, self.nx, self.ny, self.nz, self.pitch, self.stride, prm)  # synchronises
        self.setup_ms = (time.perf_counter() - t0) * 1e3
        self.L = bmg3_num_levels(self.h)

    def grid(self, a: np.ndarray | None = None):
        import torch

        if a is None:
            return torch.zeros((self.nz + 2, self.ny + 2, self.pitch), dtype=torch.float64, device=self.device)
        return to_device3(a, self.pitch, self.device)

    def vcycle(self, rhs, x, ncycles=1):
        bmg3_vcycle(self.h, rhs, x, ncycles)

    def solve(self, rhs, x, tol, maxiter):
        return bmg3_solve(self.h, rhs, x, tol, maxiter)

    def relax(self, rhs, x, nsweeps=1):
        bmg3_relax(self.h, rhs, x, nsweeps)

    def residual_norm(self, rhs, x):
        return bmg3_residual_norm(self.h, rhs, x)

    def close(self):
        if getattr(self, "h", None) is not None:
            bmg3_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
