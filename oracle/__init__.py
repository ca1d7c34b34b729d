"""ctypes wrapper of the CPU oracle (oracle/bmg_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs, never by the product package
``paper_2502_05279_b200``.  This file is argument marshalling only; every
arithmetic step is in bmg_oracle.c (see its header for the paper citations).

Grid functions are float64 arrays of shape (ny+2, nx+2) (ghost ring
included); full stencils are (ny+2, nx+2, 9) in fig:stencil_operator order
SW,S,SE,W,O,E,NW,N,NE; interpolation weights are (ncy+2, ncx+2, 8) in order
LNE,LA,LNW,LR,LL,LSE,LB,LSW.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "bmg_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

STENCIL_ORDER = ("SW", "S", "SE", "W", "O", "E", "NW", "N", "NE")
CI_ORDER = ("LNE", "LA", "LNW", "LR", "LL", "LSE", "LB", "LSW")

OK, EINVAL, ENOMEM, ENOTSPD, ENOTCONV = 0, 1, 2, 5, 6


def build(force: bool = False) -> str:
    """Compile the oracle with gcc -O2 -ffp-contract=off (no contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
                               "-std=c11", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None
_dp = ctypes.POINTER(ctypes.c_double)
_ip = ctypes.POINTER(ctypes.c_int)


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        c_int, c_long, c_double, c_void_p = ctypes.c_int, ctypes.c_long, ctypes.c_double, ctypes.c_void_p
        sig = {
            "orc_coarsen": (c_int, [c_int]),
            "orc_count_levels": (c_int, [c_int, c_int, c_int, c_int]),
            "orc_expand_stencil": (c_int, [c_int, c_int, c_int, c_long, _dp, _dp, _dp, _dp, _dp, _dp]),
            "orc_setup_interp": (c_int, [c_int, c_int, _dp, _dp]),
            "orc_rap": (c_int, [c_int, c_int, _dp, _dp, _dp]),
            "orc_relax": (None, [c_int, c_int, c_int, _dp, _dp, _dp, c_int]),
            "orc_relax_lines": (c_int, [c_int, c_int, _dp, _dp, _dp, c_int, c_int]),
            "orc_relax_adjoint": (None, [c_int, c_int, c_int, _dp, _dp, _dp, c_int]),
            "orc_relax_lines_adjoint": (c_int, [c_int, c_int, _dp, _dp, _dp, c_int, c_int]),
            "orc_pcg": (c_int, [c_void_p, _dp, _dp, c_double, c_int, _ip, _dp]),
            "orc_residual": (None, [c_int, c_int, _dp, _dp, _dp, _dp]),
            "orc_restrict": (None, [c_int, c_int, _dp, _dp, _dp]),
            "orc_interp_add": (None, [c_int, c_int, _dp, _dp, _dp]),
            "orc_interp_add_affine": (None, [c_int, c_int, _dp, _dp, _dp, _dp, _dp]),
            "orc_set_affine": (None, [c_void_p, c_int]),
            "orc_chol_factor": (c_int, [c_int, _dp]),
            "orc_chol_solve": (None, [c_int, _dp, _dp]),
            "orc_assemble_dense": (None, [c_int, c_int, _dp, _dp]),
            "orc_norm2": (c_double, [c_int, c_int, _dp]),
            "orc_setup": (c_int, [c_int, c_int, c_int, c_long, _dp, _dp, _dp, _dp, _dp, c_int, c_int, c_int,
                                  c_int, c_int, c_int, ctypes.POINTER(c_void_p)]),
            "orc_destroy": (None, [c_void_p]),
            "orc_num_levels": (c_int, [c_void_p]),
            "orc_level_shape": (None, [c_void_p, c_int, _ip, _ip, _ip]),
            "orc_export_level": (None, [c_void_p, c_int, _dp, _dp]),
            "orc_vcycle": (None, [c_void_p, _dp, _dp, c_int]),
            "orc_residual_norm": (c_double, [c_void_p, _dp, _dp]),
            "orc_solve": (c_int, [c_void_p, _dp, _dp, c_double, c_int, _ip, _dp]),
            "orc_solve_block": (c_int, [c_void_p, c_int, _dp, _dp, c_double, c_int, _ip, _dp]),
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


def _grid(nx, ny):
    return np.zeros((ny + 2, nx + 2))


def coarsen(n: int) -> int:
    return lib().orc_coarsen(n)


def count_levels(nx, ny, coarsest=3, max_levels=0) -> int:
    return lib().orc_count_levels(nx, ny, coarsest, max_levels)


def expand_stencil(stencil) -> np.ndarray:
    """Full 9-entry stencil with ghost couplings dropped (c0, c2)."""
    nx, ny = stencil.nx, stencil.ny
    planes = [np.ascontiguousarray(p, dtype=np.float64) for p in stencil.plane_list()]
    while len(planes) < 5:
        planes.append(None)
    st = np.zeros((ny + 2, nx + 2, 9))
    rc = lib().orc_expand_stencil(nx, ny, stencil.kind, nx + 2, *[_p(p) for p in planes], _p(st))
    if rc != OK:
        raise ValueError(f"orc_expand_stencil: status {rc}")
    return st


def setup_interp(st: np.ndarray) -> np.ndarray:
    ny, nx = st.shape[0] - 2, st.shape[1] - 2
    ci = np.zeros((ny // 2 + 2, nx // 2 + 2, 8))
    rc = lib().orc_setup_interp(nx, ny, _p(st), _p(ci))
    if rc != OK:
        raise ValueError(f"orc_setup_interp: status {rc}")
    return ci


def rap(st: np.ndarray, ci: np.ndarray) -> np.ndarray:
    ny, nx = st.shape[0] - 2, st.shape[1] - 2
    stc = np.zeros((ny // 2 + 2, nx // 2 + 2, 9))
    rc = lib().orc_rap(nx, ny, _p(st), _p(ci), _p(stc))
    if rc != OK:
        raise ValueError(f"orc_rap: status {rc}")
    return stc


def relax(st, kind, f, u, nsweeps=1) -> np.ndarray:
    ny, nx = st.shape[0] - 2, st.shape[1] - 2
    u = np.array(u, dtype=np.float64, copy=True, order="C")
    lib().orc_relax(nx, ny, kind, _p(st), _p(np.ascontiguousarray(f)), _p(u), nsweeps)
    return u


POINT, XLINES, YLINES, ALTLINES = 0, 1, 2, 3
RELAX_MODES = {"point": POINT, "xline": XLINES, "yline": YLINES, "altline": ALTLINES}


def relax_lines(st, f, u, nsweeps=1, mode=XLINES) -> np.ndarray:
    """c11 zebra line GS (x-lines, y-lines or alternating), nsweeps sweeps."""
    ny, nx = st.shape[0] - 2, st.shape[1] - 2
    u = np.array(u, dtype=np.float64, copy=True, order="C")
    rc = lib().orc_relax_lines(nx, ny, _p(np.ascontiguousarray(st)), _p(np.ascontiguousarray(f)), _p(u), nsweeps,
                               RELAX_MODES.get(mode, mode))
    if rc != OK:
        raise np.linalg.LinAlgError(f"orc_relax_lines: status {rc} (line block not SPD)")
    return u


def relax_adjoint(st, kind, f, u, nsweeps=1) -> np.ndarray:
    """c12: multicolour point GS with the colours in descending order."""
    ny, nx = st.shape[0] - 2, st.shape[1] - 2
    u = np.array(u, dtype=np.float64, copy=True, order="C")
    lib().orc_relax_adjoint(nx, ny, kind, _p(st), _p(np.ascontiguousarray(f)), _p(u), nsweeps)
    return u


def relax_lines_adjoint(st, f, u, nsweeps=1, mode=XLINES) -> np.ndarray:
    """c12: line GS with every sweep's (direction, colour) passes reversed."""
    ny, nx = st.shape[0] - 2, st.shape[1] - 2
    u = np.array(u, dtype=np.float64, copy=True, order="C")
    rc = lib().orc_relax_lines_adjoint(nx, ny, _p(np.ascontiguousarray(st)), _p(np.ascontiguousarray(f)), _p(u),
                                       nsweeps, RELAX_MODES.get(mode, mode))
    if rc != OK:
        raise np.linalg.LinAlgError(f"orc_relax_lines_adjoint: status {rc}")
    return u


def residual(st, f, u) -> np.ndarray:
    ny, nx = st.shape[0] - 2, st.shape[1] - 2
    r = _grid(nx, ny)
    lib().orc_residual(nx, ny, _p(st), _p(np.ascontiguousarray(f)), _p(np.ascontiguousarray(u)), _p(r))
    return r


def restrict(ci, q) -> np.ndarray:
    ny, nx = q.shape[0] - 2, q.shape[1] - 2
    qc = _grid(nx // 2, ny // 2)
    lib().orc_restrict(nx, ny, _p(np.ascontiguousarray(ci)), _p(np.ascontiguousarray(q)), _p(qc))
    return qc


def interp_add(ci, e, u) -> np.ndarray:
    ny, nx = u.shape[0] - 2, u.shape[1] - 2
    u = np.array(u, dtype=np.float64, copy=True, order="C")
    lib().orc_interp_add(nx, ny, _p(np.ascontiguousarray(ci)), _p(np.ascontiguousarray(e)), _p(u))
    return u


def interp_add_affine(ci, e, st, r, u) -> np.ndarray:
    """c14: u += P e + r/a_O at the non-coarse fine points."""
    ny, nx = u.shape[0] - 2, u.shape[1] - 2
    u = np.array(u, dtype=np.float64, copy=True, order="C")
    lib().orc_interp_add_affine(nx, ny, _p(np.ascontiguousarray(ci)), _p(np.ascontiguousarray(e)),
                                _p(np.ascontiguousarray(st)), _p(np.ascontiguousarray(r)), _p(u))
    return u


def chol_factor(A) -> np.ndarray:
    A = np.array(A, dtype=np.float64, copy=True, order="C")
    rc = lib().orc_chol_factor(A.shape[0], _p(A))
    if rc != OK:
        raise np.linalg.LinAlgError(f"orc_chol_factor: status {rc} (not SPD)")
    return A


def chol_solve(L, b) -> np.ndarray:
    b = np.array(b, dtype=np.float64, copy=True)
    lib().orc_chol_solve(L.shape[0], _p(np.ascontiguousarray(L)), _p(b))
    return b


def assemble_dense(st) -> np.ndarray:
    ny, nx = st.shape[0] - 2, st.shape[1] - 2
    A = np.zeros((nx * ny, nx * ny))
    lib().orc_assemble_dense(nx, ny, _p(st), _p(A))
    return A


def norm2(g) -> float:
    ny, nx = g.shape[0] - 2, g.shape[1] - 2
    return lib().orc_norm2(nx, ny, _p(np.ascontiguousarray(g)))


class Hierarchy:
    """Oracle BoxMG hierarchy (setup c0-c4, c8) with V-cycle / solve (c9)."""

    def __init__(self, stencil, nu1=2, nu2=1, coarsest=3, max_levels=0, relax="point", cycle_sym=0, affine=0):
        nx, ny = stencil.nx, stencil.ny
        self.nx, self.ny = nx, ny
        planes = [np.ascontiguousarray(p, dtype=np.float64) for p in stencil.plane_list()]
        while len(planes) < 5:
            planes.append(None)
        h = ctypes.c_void_p()
        rc = lib().orc_setup(nx, ny, stencil.kind, nx + 2, *[_p(p) for p in planes], nu1, nu2, coarsest,
                             max_levels, RELAX_MODES.get(relax, relax), cycle_sym, ctypes.byref(h))
        if rc != OK:
            raise ValueError(f"orc_setup: status {rc}")
        self._h = h
        if affine:
            lib().orc_set_affine(h, 1)

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
        st = np.zeros((ny + 2, nx + 2, 9))
        ci = np.zeros((ny // 2 + 2, nx // 2 + 2, 8)) if l + 1 < self.num_levels else None
        lib().orc_export_level(self._h, l, _p(st), _p(ci))
        return st, ci

    def vcycle(self, f, u, ncycles=1) -> np.ndarray:
        u = np.array(u, dtype=np.float64, copy=True, order="C")
        lib().orc_vcycle(self._h, _p(np.ascontiguousarray(f)), _p(u), ncycles)
        return u

    def residual_norm(self, f, u) -> float:
        return lib().orc_residual_norm(self._h, _p(np.ascontiguousarray(f)), _p(np.ascontiguousarray(u)))

    def pcg(self, f, u, tol, maxiter):
        """c13: V-cycle-preconditioned CG (needs nu1 == nu2, cycle_sym=1)."""
        u = np.array(u, dtype=np.float64, copy=True, order="C")
        hist = np.zeros(maxiter + 1)
        it = ctypes.c_int()
        rc = lib().orc_pcg(self._h, _p(np.ascontiguousarray(f)), _p(u), tol, maxiter, ctypes.byref(it), _p(hist))
        return u, it.value, hist[: it.value + 1], rc

    def solve(self, f, u, tol, maxiter):
        u = np.array(u, dtype=np.float64, copy=True, order="C")
        hist = np.zeros(maxiter + 1)
        it = ctypes.c_int()
        rc = lib().orc_solve(self._h, _p(np.ascontiguousarray(f)), _p(u), tol, maxiter, ctypes.byref(it), _p(hist))
        return u, it.value, hist[: it.value + 1], rc

    def solve_block(self, F, U, tol, maxiter):
        """c15 block multi-RHS solve: F, U of shape (nrhs, ny+2, nx+2).  Returns
        (U, block steps, hist (steps+1, nrhs) absolute norms, status)."""
        F = np.ascontiguousarray(F, dtype=np.float64)
        U = np.array(U, dtype=np.float64, copy=True, order="C")
        K = F.shape[0]
        hist = np.zeros((maxiter + 1, K))
        it = ctypes.c_int()
        rc = lib().orc_solve_block(self._h, K, _p(F), _p(U), tol, maxiter, ctypes.byref(it), _p(hist))
        return U, it.value, hist[: it.value + 1], rc

    def pcg_block(self, F, U, tol, maxiter):
        """c13 on each column of a c15 block (bmg_pcg_block's reading): the columns
        are independent PCG runs (orc_pcg), each stopping at its own test.
        Returns (U, per-column iterations, per-column histories, per-column status)."""
        outs = [self.pcg(F[c], U[c], tol, maxiter) for c in range(len(F))]
        return (np.stack([o[0] for o in outs]), [o[1] for o in outs], [o[2] for o in outs], [o[3] for o in outs])
