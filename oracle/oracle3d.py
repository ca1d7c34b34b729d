"""ctypes wrapper of the 3-D CPU oracle (oracle/bmg3_oracle.c, linked with the
2-D oracle bmg_oracle.c whose V-cycle is its plane solver).

TEST INFRASTRUCTURE ONLY (same rule as oracle/__init__.py): imported by tests/
and bench.py's cpu_baseline / --impl reference legs, never by the product
package.  Marshalling only; every arithmetic step is in bmg3_oracle.c.

Grid functions: float64 (nz+2, ny+2, nx+2); full stencils (nz+2, ny+2, nx+2, 27)
with entry e = (dz+1)*9+(dy+1)*3+(dx+1); interpolation weights
(ncz+2, ncy+2, ncx+2, 26) in the c19 slot order (X 0-1, Y 2-3, Z 4-5, XY 6-9,
XZ 10-13, YZ 14-17, XYZ 18-25; corner bit b = 1 -> upper coarse coordinate on
the b-th odd axis).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRCS = [os.path.join(_HERE, "bmg3_oracle.c"), os.path.join(_HERE, "bmg_oracle.c")]
_LIB = os.path.join(_HERE, "liboracle3.so")

OK, EINVAL, ENOMEM, ENOTSPD, ENOTCONV = 0, 1, 2, 5, 6
POINT, PLANES = 0, 1
RELAX3 = {"point": POINT, "planes": PLANES}
SLOT = {1: 0, 2: 2, 4: 4, 3: 6, 5: 10, 6: 14, 7: 18}


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(os.path.getmtime(s) for s in _SRCS):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
                               "-std=c11", "-o", tmp, *_SRCS, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None
_dp = ctypes.POINTER(ctypes.c_double)
_ip = ctypes.POINTER(ctypes.c_int)


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        i, d, v = ctypes.c_int, ctypes.c_double, ctypes.c_void_p
        sig = {
            "o3_coarsen": (i, [i]),
            "o3_count_levels": (i, [i, i, i, i, i]),
            "o3_expand_stencil": (i, [i, i, i, i, _dp, _dp]),
            "o3_setup_interp": (i, [i, i, i, _dp, _dp]),
            "o3_rap": (i, [i, i, i, _dp, _dp, _dp]),
            "o3_relax": (None, [i, i, i, i, _dp, _dp, _dp, i]),
            "o3_residual": (None, [i, i, i, _dp, _dp, _dp, _dp]),
            "o3_restrict": (None, [i, i, i, _dp, _dp, _dp]),
            "o3_interp_add": (None, [i, i, i, _dp, _dp, _dp]),
            "o3_assemble_dense": (None, [i, i, i, _dp, _dp]),
            "o3_norm2": (d, [i, i, i, _dp]),
            "o3_setup": (i, [i, i, i, i, _dp, i, i, i, i, i, ctypes.POINTER(v)]),
            "o3_destroy": (None, [v]),
            "o3_num_levels": (i, [v]),
            "o3_level_shape": (None, [v, i, _ip, _ip, _ip, _ip]),
            "o3_export_level": (None, [v, i, _dp, _dp]),
            "o3_vcycle": (None, [v, _dp, _dp, i]),
            "o3_relax_level": (None, [v, _dp, _dp, i]),
            "o3_residual_norm": (d, [v, _dp, _dp]),
            "o3_solve": (i, [v, _dp, _dp, d, i, _ip, _dp]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _p(a):
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


def _c(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _dims(g):
    return g.shape[2] - 2, g.shape[1] - 2, g.shape[0] - 2


def count_levels(nx, ny, nz, coarsest=3, max_levels=0) -> int:
    return lib().o3_count_levels(nx, ny, nz, coarsest, max_levels)


def expand_stencil(stencil) -> np.ndarray:
    nx, ny, nz = stencil.nx, stencil.ny, stencil.nz
    st = np.zeros((nz + 2, ny + 2, nx + 2, 27))
    rc = lib().o3_expand_stencil(nx, ny, nz, stencil.kind, _p(stencil.stacked()), _p(st))
    if rc != OK:
        raise ValueError(f"o3_expand_stencil: status {rc}")
    return st


def setup_interp(st) -> np.ndarray:
    nx, ny, nz = _dims(st)
    ci = np.zeros((nz // 2 + 2, ny // 2 + 2, nx // 2 + 2, 26))
    rc = lib().o3_setup_interp(nx, ny, nz, _p(_c(st)), _p(ci))
    if rc != OK:
        raise ValueError(f"o3_setup_interp: status {rc}")
    return ci


def rap(st, ci) -> np.ndarray:
    nx, ny, nz = _dims(st)
    stc = np.zeros((nz // 2 + 2, ny // 2 + 2, nx // 2 + 2, 27))
    rc = lib().o3_rap(nx, ny, nz, _p(_c(st)), _p(_c(ci)), _p(stc))
    if rc != OK:
        raise ValueError(f"o3_rap: status {rc}")
    return stc


def relax(st, kind, f, u, nsweeps=1) -> np.ndarray:
    nx, ny, nz = _dims(st)
    u = np.array(u, dtype=np.float64, copy=True, order="C")
    lib().o3_relax(nx, ny, nz, kind, _p(_c(st)), _p(_c(f)), _p(u), nsweeps)
    return u


def residual(st, f, u) -> np.ndarray:
    nx, ny, nz = _dims(st)
    r = np.zeros((nz + 2, ny + 2, nx + 2))
    lib().o3_residual(nx, ny, nz, _p(_c(st)), _p(_c(f)), _p(_c(u)), _p(r))
    return r


def restrict(ci, q) -> np.ndarray:
    nx, ny, nz = _dims(q)
    qc = np.zeros((nz // 2 + 2, ny // 2 + 2, nx // 2 + 2))
    lib().o3_restrict(nx, ny, nz, _p(_c(ci)), _p(_c(q)), _p(qc))
    return qc


def interp_add(ci, e, u) -> np.ndarray:
    nx, ny, nz = _dims(u)
    u = np.array(u, dtype=np.float64, copy=True, order="C")
    lib().o3_interp_add(nx, ny, nz, _p(_c(ci)), _p(_c(e)), _p(u))
    return u


def assemble_dense(st) -> np.ndarray:
    nx, ny, nz = _dims(st)
    n = nx * ny * nz
    A = np.zeros((n, n))
    lib().o3_assemble_dense(nx, ny, nz, _p(_c(st)), _p(A))
    return A


def norm2(g) -> float:
    nx, ny, nz = _dims(g)
    return lib().o3_norm2(nx, ny, nz, _p(_c(g)))


class Hierarchy3:
    """Oracle 3-D BoxMG hierarchy (c16-c24) with V-cycle / solve."""

    def __init__(self, stencil, nu1=2, nu2=1, coarsest=3, max_levels=0, relax="point"):
        self.nx, self.ny, self.nz = stencil.nx, stencil.ny, stencil.nz
        self._pl = stencil.stacked()
        h = ctypes.c_void_p()
        rc = lib().o3_setup(self.nx, self.ny, self.nz, stencil.kind, _p(self._pl), nu1, nu2, coarsest, max_levels,
                            RELAX3.get(relax, relax), ctypes.byref(h))
        if rc != OK:
            raise ValueError(f"o3_setup: status {rc}")
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and _lib is not None:
            _lib.o3_destroy(h)
            self._h = None

    @property
    def num_levels(self) -> int:
        return lib().o3_num_levels(self._h)

    def level_shape(self, l):
        a = [ctypes.c_int() for _ in range(4)]
        lib().o3_level_shape(self._h, l, *[ctypes.byref(x) for x in a])
        return tuple(x.value for x in a)

    def export_level(self, l):
        nx, ny, nz, _ = self.level_shape(l)
        st = np.zeros((nz + 2, ny + 2, nx + 2, 27))
        ci = np.zeros((nz // 2 + 2, ny // 2 + 2, nx // 2 + 2, 26)) if l + 1 < self.num_levels else None
        lib().o3_export_level(self._h, l, _p(st), _p(ci))
        return st, ci

    def vcycle(self, f, u, ncycles=1) -> np.ndarray:
        u = np.array(u, dtype=np.float64, copy=True, order="C")
        lib().o3_vcycle(self._h, _p(_c(f)), _p(u), ncycles)
        return u

    def relax_fine(self, f, u, nsweeps=1) -> np.ndarray:
        """The hierarchy's relaxation (point or planes) on the fine level alone."""
        u = np.array(u, dtype=np.float64, copy=True, order="C")
        lib().o3_relax_level(self._h, _p(_c(f)), _p(u), nsweeps)
        return u

    def residual_norm(self, f, u) -> float:
        return lib().o3_residual_norm(self._h, _p(_c(f)), _p(_c(u)))

    def solve(self, f, u, tol, maxiter):
        u = np.array(u, dtype=np.float64, copy=True, order="C")
        hist = np.zeros(maxiter + 1)
        it = ctypes.c_int()
        rc = lib().o3_solve(self._h, _p(_c(f)), _p(u), tol, maxiter, ctypes.byref(it), _p(hist))
        return u, it.value, hist[: it.value + 1], rc
