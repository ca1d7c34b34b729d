"""ctypes wrapper of the extended-precision build of the oracle (bmg_oracle_ext.c).

TEST INFRASTRUCTURE ONLY (same rule as oracle/__init__.py).  The library is the
unchanged oracle source compiled with every fp64 value as an x87 80-bit
``long double``; arrays cross the boundary as ``numpy.longdouble`` (the same
16-byte C type on x86-64 Linux).  Inputs given as float64 convert exactly, so
the fp64 oracle, the GPU path and this build all start from identical numbers;
only the rounding unit of the arithmetic differs (2^-64 against 2^-53).
Marshalling only -- no arithmetic here.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "bmg_oracle_ext.c")
_DEP = os.path.join(_HERE, "bmg_oracle.c")
_LIB = os.path.join(_HERE, "liboracle_ext.so")

assert np.finfo(np.longdouble).nmant >= 63, "x87 extended long double required"


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(os.path.getmtime(_SRC),
                                                                           os.path.getmtime(_DEP)):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
                               "-std=c11", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None
_lp = ctypes.POINTER(ctypes.c_longdouble)
_ip = ctypes.POINTER(ctypes.c_int)


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        c_int, c_long, c_ld, c_void_p = ctypes.c_int, ctypes.c_long, ctypes.c_longdouble, ctypes.c_void_p
        sig = {
            "orc_setup": (c_int, [c_int, c_int, c_int, c_long, _lp, _lp, _lp, _lp, _lp, c_int, c_int, c_int,
                                  c_int, c_int, c_int, ctypes.POINTER(c_void_p)]),
            "orc_destroy": (None, [c_void_p]),
            "orc_num_levels": (c_int, [c_void_p]),
            "orc_level_shape": (None, [c_void_p, c_int, _ip, _ip, _ip]),
            "orc_export_level": (None, [c_void_p, c_int, _lp, _lp]),
            "orc_vcycle": (None, [c_void_p, _lp, _lp, c_int]),
            "orc_residual_norm": (c_ld, [c_void_p, _lp, _lp]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _ld(a):
    return np.ascontiguousarray(a, dtype=np.longdouble)


def _p(a):
    if a is None:
        return None
    assert a.dtype == np.longdouble and a.flags.c_contiguous
    return a.ctypes.data_as(_lp)


class HierarchyExt:
    """oracle.Hierarchy in extended precision (setup c0-c4, c8; V-cycle c9)."""

    def __init__(self, stencil, nu1=2, nu2=1, coarsest=3, max_levels=0, relax=0, cycle_sym=0):
        nx, ny = stencil.nx, stencil.ny
        self.nx, self.ny = nx, ny
        self._planes = [_ld(p) for p in stencil.plane_list()]
        planes = self._planes + [None] * (5 - len(self._planes))
        h = ctypes.c_void_p()
        rc = lib().orc_setup(nx, ny, stencil.kind, nx + 2, *[_p(p) for p in planes], nu1, nu2, coarsest,
                             max_levels, relax, cycle_sym, ctypes.byref(h))
        if rc != 0:
            raise ValueError(f"orc_setup (extended): status {rc}")
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and _lib is not None:
            _lib.orc_destroy(h)
            self._h = None

    @property
    def num_levels(self) -> int:
        return lib().orc_num_levels(self._h)

    def level_shape(self, l):
        nx, ny, kind = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        lib().orc_level_shape(self._h, l, ctypes.byref(nx), ctypes.byref(ny), ctypes.byref(kind))
        return nx.value, ny.value, kind.value

    def export_level(self, l):
        nx, ny, _ = self.level_shape(l)
        st = np.zeros((ny + 2, nx + 2, 9), dtype=np.longdouble)
        ci = np.zeros((ny // 2 + 2, nx // 2 + 2, 8), dtype=np.longdouble) if l + 1 < self.num_levels else None
        lib().orc_export_level(self._h, l, _p(st), _p(ci))
        return st, ci

    def vcycle(self, f, u, ncycles=1) -> np.ndarray:
        """Returns the iterate as numpy.longdouble (call .astype(float) to round once)."""
        u = np.array(u, dtype=np.longdouble, copy=True, order="C")
        f = _ld(f)
        lib().orc_vcycle(self._h, _p(f), _p(u), ncycles)
        return u

    def residual_norm(self, f, u):
        return lib().orc_residual_norm(self._h, _p(_ld(f)), _p(_ld(u)))
