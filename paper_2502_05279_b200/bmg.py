"""Thin ctypes binding of libbmg.so (include/bmg.h), same names as the C ABI.

Argument marshalling only: every step of the method runs in the CUDA kernels
behind the ABI.  Device arrays are torch CUDA tensors (float64) passed by
``data_ptr()``; the stream is ``torch.cuda.current_stream().cuda_stream``
unless given.  There is no CPU fallback: if libbmg.so is missing the first
call raises ``RuntimeError``.
"""
from __future__ import annotations

import ctypes
import time
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BMG_LIB") or os.path.join(_HERE, "libbmg.so")

BMG_OK, BMG_EINVAL, BMG_ENOMEM, BMG_ECUDA, BMG_ENCCL, BMG_ENOTSPD, BMG_ENOTCONV = range(7)

# Every symbol include/bmg.h declares (checked by tests/test_abi.py).
EXPORTS = (
    "bmg_params_default", "bmg_setup", "bmg_vcycle", "bmg_vcycle_host", "bmg_vcycle_host_batch", "bmg_solve", "bmg_pcg", "bmg_residual_norm",
    "bmg_num_levels", "bmg_level_shape", "bmg_level_pitch", "bmg_export_level", "bmg_relax", "bmg_residual",
    "bmg_restrict", "bmg_interp_add", "bmg_smooth_restrict", "bmg_correct_smooth", "bmg_cycle_kernel_count", "bmg_timing",
    "bmg_timing_read", "bmg_profile_legs", "bmg_setup_time", "bmg_destroy", "bmg_strerror",
    "bmg_last_error_detail", "bmg_partition", "bmg_setup_dist", "bmg_local_rows", "bmg_vcycle_block",
    "bmg_residual_norm_block", "bmg_solve_block", "bmg_pcg_block",
)

BMG_MAX_NRHS = 8

BMG_HALO = 6

# bmg_params_t.relax (include/bmg.h)
BMG_RELAX_POINT, BMG_RELAX_XLINES, BMG_RELAX_YLINES, BMG_RELAX_ALTLINES = range(4)


class bmg_stencil_t(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int), ("nx", ctypes.c_int), ("ny", ctypes.c_int), ("pitch", ctypes.c_longlong),
                ("plane", ctypes.c_void_p * 5)]


class bmg_params_t(ctypes.Structure):
    _fields_ = [("nu1", ctypes.c_int), ("nu2", ctypes.c_int), ("coarsest", ctypes.c_int),
                ("max_levels", ctypes.c_int), ("agglom_rows", ctypes.c_int), ("cycle_sym", ctypes.c_int),
                ("fused", ctypes.c_int), ("relax", ctypes.c_int), ("affine", ctypes.c_int)]


class bmg_comm_t(ctypes.Structure):
    _fields_ = [("nranks", ctypes.c_int), ("rank", ctypes.c_int), ("nccl_comm", ctypes.c_void_p),
                ("nccl_lib", ctypes.c_char_p), ("loopback", ctypes.c_int), ("peer", ctypes.c_int)]


class BmgError(RuntimeError):
    def __init__(self, status: int, where: str, detail: str):
        super().__init__(f"{where}: status {status} ({detail})")
        self.status = status


_lib = None


def lib():
    """Load libbmg.so (built by __graft_entry__.build()); fail loudly if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"libbmg.so not built ({LIB_PATH}); run __graft_entry__.build() -- "
                               "there is no CPU fallback")
        L = ctypes.CDLL(LIB_PATH)
        vp, i, ll, d = ctypes.c_void_p, ctypes.c_int, ctypes.c_longlong, ctypes.c_double
        ip, dp, lp = ctypes.POINTER(i), ctypes.POINTER(d), ctypes.POINTER(ll)
        sig = {
            "bmg_params_default": (None, [ctypes.POINTER(bmg_params_t)]),
            "bmg_setup": (i, [ctypes.POINTER(bmg_stencil_t), ctypes.POINTER(bmg_params_t), vp,
                              ctypes.POINTER(vp)]),
            "bmg_vcycle": (i, [vp, vp, vp, i, vp]),
            "bmg_vcycle_host": (i, [vp, vp, vp, i, vp]),
            "bmg_vcycle_host_batch": (i, [vp, i, vp, vp, i, vp]),
            "bmg_solve": (i, [vp, vp, vp, d, i, ip, dp, vp]),
            "bmg_pcg": (i, [vp, vp, vp, d, i, ip, dp, vp]),
            "bmg_vcycle_block": (i, [vp, i, vp, vp, i, vp]),
            "bmg_residual_norm_block": (i, [vp, i, vp, vp, dp, vp]),
            "bmg_solve_block": (i, [vp, i, vp, vp, d, i, ip, dp, vp]),
            "bmg_pcg_block": (i, [vp, i, vp, vp, d, i, ip, dp, vp]),
            "bmg_residual_norm": (i, [vp, vp, vp, vp, dp, vp]),
            "bmg_num_levels": (i, [vp, ip]),
            "bmg_level_shape": (i, [vp, i, ip, ip, ip]),
            "bmg_level_pitch": (i, [vp, i, lp]),
            "bmg_export_level": (i, [vp, i, dp, dp]),
            "bmg_relax": (i, [vp, i, vp, vp, i, vp]),
            "bmg_residual": (i, [vp, i, vp, vp, vp, vp]),
            "bmg_restrict": (i, [vp, i, vp, vp, vp]),
            "bmg_interp_add": (i, [vp, i, vp, vp, vp]),
            "bmg_smooth_restrict": (i, [vp, i, vp, vp, vp, vp, vp, vp]),
            "bmg_correct_smooth": (i, [vp, i, vp, vp, vp, vp, vp]),
            "bmg_cycle_kernel_count": (i, [vp, ip]),
            "bmg_profile_legs": (i, [vp, vp, vp, i, dp, i, ip, vp]),
            "bmg_setup_time": (i, [vp, dp]),
            "bmg_destroy": (i, [vp]),
            "bmg_strerror": (ctypes.c_char_p, [i]),
            "bmg_last_error_detail": (ctypes.c_char_p, []),
            "bmg_partition": (i, [i, i, i, ctypes.POINTER(bmg_params_t), ip, ip]),
            "bmg_setup_dist": (i, [ctypes.POINTER(bmg_stencil_t), ctypes.POINTER(bmg_comm_t),
                                   ctypes.POINTER(bmg_params_t), vp, ctypes.POINTER(vp)]),
            "bmg_local_rows": (i, [vp, ip, ip, ip, ip, ip]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _check(rc: int, where: str, ok=(BMG_OK,)):
    if rc not in ok:
        detail = lib().bmg_last_error_detail().decode(errors="replace")
        raise BmgError(rc, where, detail)
    return rc


def _stream(stream):
    if stream is not None:
        return ctypes.c_void_p(int(stream))
    import torch

    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _ptr(t):
    if t is None:
        return None
    return ctypes.c_void_p(t.data_ptr())


def bmg_params_default() -> bmg_params_t:
    p = bmg_params_t()
    lib().bmg_params_default(ctypes.byref(p))
    return p


def bmg_setup(planes, kind: int, nx: int, ny: int, pitch: int, params: bmg_params_t | None = None,
              stream=None) -> ctypes.c_void_p:
    """planes: list of 3 (kind 5) or 5 (kind 9) device float64 tensors, (ny+2)*pitch each."""
    st = bmg_stencil_t()
    st.kind, st.nx, st.ny, st.pitch = kind, nx, ny, pitch
    for k, p in enumerate(planes):
        st.plane[k] = p.data_ptr()
    h = ctypes.c_void_p()
    _check(lib().bmg_setup(ctypes.byref(st), ctypes.byref(params) if params is not None else None, _stream(stream),
                           ctypes.byref(h)), "bmg_setup")
    return h


def bmg_vcycle(h, rhs, x, ncycles: int = 1, stream=None):
    _check(lib().bmg_vcycle(h, _ptr(rhs), _ptr(x), ncycles, _stream(stream)), "bmg_vcycle")


def bmg_vcycle_host_batch(h, rhs_hosts, x_hosts, ncycles: int = 1, stream=None):
    """bmg_vcycle_host_batch: lists of host tensors/arrays (pinned for overlap), one problem each."""
    n = len(rhs_hosts)
    assert len(x_hosts) == n
    ra = (ctypes.c_void_p * max(n, 1))(*[_ptr(a).value for a in rhs_hosts])
    xa = (ctypes.c_void_p * max(n, 1))(*[_ptr(a).value for a in x_hosts])
    _check(lib().bmg_vcycle_host_batch(h, n, ra, xa, ncycles, _stream(stream)), "bmg_vcycle_host_batch")


def bmg_vcycle_host(h, rhs_host, x_host, ncycles: int = 1, stream=None):
    """rhs_host / x_host: CPU float64 torch tensors (pinned for full speed), setup pitch."""
    _check(lib().bmg_vcycle_host(h, _ptr(rhs_host), _ptr(x_host), ncycles, _stream(stream)), "bmg_vcycle_host")


def bmg_solve(h, rhs, x, tol: float, maxiter: int, stream=None):
    """Returns (iters, hist ndarray of iters+1 absolute norms, status)."""
    it = ctypes.c_int()
    hist = np.zeros(maxiter + 1)
    rc = lib().bmg_solve(h, _ptr(rhs), _ptr(x), tol, maxiter, ctypes.byref(it),
                         hist.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), _stream(stream))
    _check(rc, "bmg_solve", ok=(BMG_OK, BMG_ENOTCONV))
    return it.value, hist[: it.value + 1], rc


def bmg_pcg(h, rhs, x, tol: float, maxiter: int, stream=None):
    """V-cycle-preconditioned CG.  Returns (iters, hist of iters+1 absolute norms, status)."""
    it = ctypes.c_int()
    hist = np.zeros(maxiter + 1)
    rc = lib().bmg_pcg(h, _ptr(rhs), _ptr(x), tol, maxiter, ctypes.byref(it),
                       hist.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), _stream(stream))
    _check(rc, "bmg_pcg", ok=(BMG_OK, BMG_ENOTCONV))
    return it.value, hist[: it.value + 1], rc


def bmg_vcycle_block(h, nrhs: int, rhs, x, ncycles: int = 1, stream=None):
    """rhs, x: device tensors (ny+2, pitch, nrhs) -- the interleaved block layout."""
    _check(lib().bmg_vcycle_block(h, nrhs, _ptr(rhs), _ptr(x), ncycles, _stream(stream)), "bmg_vcycle_block")


def bmg_residual_norm_block(h, nrhs: int, rhs, x, stream=None) -> np.ndarray:
    out = np.zeros(nrhs)
    _check(lib().bmg_residual_norm_block(h, nrhs, _ptr(rhs), _ptr(x), out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                         _stream(stream)), "bmg_residual_norm_block")
    return out


def bmg_solve_block(h, nrhs: int, rhs, x, tol: float, maxiter: int, stream=None):
    """Returns (block steps, hist (steps+1, nrhs) absolute norms, status)."""
    it = ctypes.c_int()
    hist = np.zeros((maxiter + 1, nrhs))
    rc = lib().bmg_solve_block(h, nrhs, _ptr(rhs), _ptr(x), tol, maxiter, ctypes.byref(it),
                               hist.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), _stream(stream))
    _check(rc, "bmg_solve_block", ok=(BMG_OK, BMG_ENOTCONV))
    return it.value, hist[: it.value + 1], rc


def bmg_pcg_block(h, nrhs: int, rhs, x, tol: float, maxiter: int, stream=None):
    """Block PCG.  Returns (steps, hist (steps+1, nrhs) recursive residual norms, status)."""
    it = ctypes.c_int()
    hist = np.zeros((maxiter + 1, nrhs))
    rc = lib().bmg_pcg_block(h, nrhs, _ptr(rhs), _ptr(x), tol, maxiter, ctypes.byref(it),
                             hist.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), _stream(stream))
    _check(rc, "bmg_pcg_block", ok=(BMG_OK, BMG_ENOTCONV))
    return it.value, hist[: it.value + 1], rc


def bmg_residual_norm(h, rhs, x, r_out=None, stream=None) -> float:
    out = ctypes.c_double()
    _check(lib().bmg_residual_norm(h, _ptr(rhs), _ptr(x), _ptr(r_out), ctypes.byref(out), _stream(stream)),
           "bmg_residual_norm")
    return out.value


def bmg_num_levels(h) -> int:
    L = ctypes.c_int()
    _check(lib().bmg_num_levels(h, ctypes.byref(L)), "bmg_num_levels")
    return L.value


def bmg_level_shape(h, level: int):
    nx, ny, kind = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    _check(lib().bmg_level_shape(h, level, ctypes.byref(nx), ctypes.byref(ny), ctypes.byref(kind)),
           "bmg_level_shape")
    return nx.value, ny.value, kind.value


def bmg_level_pitch(h, level: int) -> int:
    p = ctypes.c_longlong()
    _check(lib().bmg_level_pitch(h, level, ctypes.byref(p)), "bmg_level_pitch")
    return p.value


def bmg_export_level(h, level: int):
    """Returns (planes (5, ny+2, nx+2) O,W,S,SW,NW; ci (8, ncy+2, ncx+2) or None)."""
    nx, ny, _ = bmg_level_shape(h, level)
    st = np.zeros((5, ny + 2, nx + 2))
    L = bmg_num_levels(h)
    ci = np.zeros((8, ny // 2 + 2, nx // 2 + 2)) if level + 1 < L else None
    dp = ctypes.POINTER(ctypes.c_double)
    _check(lib().bmg_export_level(h, level, st.ctypes.data_as(dp), ci.ctypes.data_as(dp) if ci is not None else None),
           "bmg_export_level")
    return st, ci


def bmg_relax(h, level, f, u, nsweeps=1, stream=None):
    _check(lib().bmg_relax(h, level, _ptr(f), _ptr(u), nsweeps, _stream(stream)), "bmg_relax")


def bmg_residual(h, level, f, u, r, stream=None):
    _check(lib().bmg_residual(h, level, _ptr(f), _ptr(u), _ptr(r), _stream(stream)), "bmg_residual")


def bmg_restrict(h, level, r, fc, stream=None):
    _check(lib().bmg_restrict(h, level, _ptr(r), _ptr(fc), _stream(stream)), "bmg_restrict")


def bmg_interp_add(h, level, ec, u, stream=None):
    _check(lib().bmg_interp_add(h, level, _ptr(ec), _ptr(u), _stream(stream)), "bmg_interp_add")


def bmg_smooth_restrict(h, level, f, u_in, u_out, fc, uc=None, stream=None):
    _check(lib().bmg_smooth_restrict(h, level, _ptr(f), _ptr(u_in), _ptr(u_out), _ptr(fc), _ptr(uc), _stream(stream)),
           "bmg_smooth_restrict")


def bmg_correct_smooth(h, level, f, u_in, ec, u_out, stream=None):
    _check(lib().bmg_correct_smooth(h, level, _ptr(f), _ptr(u_in), _ptr(ec), _ptr(u_out), _stream(stream)),
           "bmg_correct_smooth")


def bmg_cycle_kernel_count(h) -> int:
    c = ctypes.c_int()
    _check(lib().bmg_cycle_kernel_count(h, ctypes.byref(c)), "bmg_cycle_kernel_count")
    return c.value


def bmg_timing(h, enable: bool) -> None:
    _check(lib().bmg_timing(h, 1 if enable else 0), "bmg_timing")


def bmg_timing_read(h):
    """(summed ms, launches) of the level-0 down legs recorded since the last clear."""
    ms = ctypes.c_double()
    n = ctypes.c_int()
    _check(lib().bmg_timing_read(h, ctypes.byref(ms), ctypes.byref(n)), "bmg_timing_read")
    return ms.value, n.value


def bmg_profile_legs(h, rhs, x, ncycles: int = 5, stream=None):
    """Mean device time (ms) of every leg of one cycle: (down[0..lt-1], tail, up[lt-1..0])."""
    L = bmg_num_levels(h)
    out = (ctypes.c_double * (2 * L + 1))()
    n = ctypes.c_int()
    _check(lib().bmg_profile_legs(h, _ptr(rhs), _ptr(x), ncycles, out, 2 * L + 1, ctypes.byref(n), _stream(stream)),
           "bmg_profile_legs")
    v = list(out[: n.value])
    lt = (n.value - 1) // 2
    return v[:lt], v[lt], v[lt + 1:][::-1]


def bmg_setup_time(h) -> float:
    """Device time (ms) of the setup kernels S0-S3 of a single-GPU handle."""
    ms = ctypes.c_double()
    _check(lib().bmg_setup_time(h, ctypes.byref(ms)), "bmg_setup_time")
    return ms.value


def bmg_partition(nx: int, ny: int, nranks: int, params: bmg_params_t | None = None):
    """Host-only: (slab boundaries y_0..y_nranks, number of distributed levels)."""
    yb = (ctypes.c_int * (nranks + 1))()
    k = ctypes.c_int()
    _check(lib().bmg_partition(nx, ny, nranks, ctypes.byref(params) if params is not None else None, yb,
                               ctypes.byref(k)), "bmg_partition")
    return list(yb), k.value


def bmg_setup_dist(planes, kind: int, nx: int, ny: int, pitch: int, comm: bmg_comm_t,
                   params: bmg_params_t | None = None, stream=None) -> ctypes.c_void_p:
    """planes: device tensors (local arrays in NCCL mode, global arrays in loopback mode)."""
    st = bmg_stencil_t()
    st.kind, st.nx, st.ny, st.pitch = kind, nx, ny, pitch
    for k, p in enumerate(planes):
        st.plane[k] = p.data_ptr()
    h = ctypes.c_void_p()
    _check(lib().bmg_setup_dist(ctypes.byref(st), ctypes.byref(comm),
                                ctypes.byref(params) if params is not None else None, _stream(stream),
                                ctypes.byref(h)), "bmg_setup_dist")
    return h


def bmg_local_rows(h):
    """(row0, nrows, ylo, yhi, kdist) of this handle's level-0 local arrays."""
    v = [ctypes.c_int() for _ in range(5)]
    _check(lib().bmg_local_rows(h, *[ctypes.byref(x) for x in v]), "bmg_local_rows")
    return tuple(x.value for x in v)


def bmg_destroy(h):
    if h is not None and h.value:
        _check(lib().bmg_destroy(h), "bmg_destroy")


# --------------------------------------------------------------------------- helpers
def default_pitch(nx: int) -> int:
    """Row pitch used for rhs/x/planes: nx+2 rounded up to 32 doubles (256 B rows)."""
    return (nx + 2 + 31) // 32 * 32


def to_device(a: np.ndarray, pitch: int, device="cuda"):
    """(ny+2, nx+2) host array -> (ny+2, pitch) device float64 tensor (pad zero)."""
    import torch

    t = torch.zeros((a.shape[0], pitch), dtype=torch.float64, device=device)
    t[:, : a.shape[1]] = torch.from_numpy(np.ascontiguousarray(a)).to(device)
    return t


def from_device(t, nx: int) -> np.ndarray:
    return t[:, : nx + 2].cpu().numpy().copy()


def to_device_block(arrays, pitch: int, device="cuda"):
    """nrhs (ny+2, nx+2) host arrays -> (ny+2, pitch, nrhs) device tensor (block layout)."""
    import torch

    a = np.stack([np.asarray(x, dtype=np.float64) for x in arrays], axis=-1)
    t = torch.zeros((a.shape[0], pitch, a.shape[2]), dtype=torch.float64, device=device)
    t[:, : a.shape[1], :] = torch.from_numpy(np.ascontiguousarray(a)).to(device)
    return t


def from_device_block(t, nx: int) -> np.ndarray:
    """(ny+2, pitch, nrhs) device tensor -> (nrhs, ny+2, nx+2) host array."""
    return np.ascontiguousarray(np.moveaxis(t[:, : nx + 2, :].cpu().numpy(), -1, 0))


class Solver:
    """Convenience owner of a bmg_solver_t for a problems.Stencil (device copies kept)."""

    def __init__(self, stencil, params: bmg_params_t | None = None, pitch: int | None = None, device="cuda"):
        self.nx, self.ny, self.kind = stencil.nx, stencil.ny, stencil.kind
        self.pitch = pitch or default_pitch(self.nx)
        self.device = device
        planes = [to_device(p, self.pitch, device) for p in stencil.plane_list()]
        t0 = time.perf_counter()
        self.h = bmg_setup(planes, self.kind, self.nx, self.ny, self.pitch, params)  # synchronises
        self.setup_ms = (time.perf_counter() - t0) * 1e3
        self.L = bmg_num_levels(self.h)

    def grid(self, a: np.ndarray | None = None):
        import torch

        if a is None:
            return torch.zeros((self.ny + 2, self.pitch), dtype=torch.float64, device=self.device)
        return to_device(a, self.pitch, self.device)

    def level_grid(self, level: int, a: np.ndarray | None = None):
        import torch

        nx, ny, _ = bmg_level_shape(self.h, level)
        p = bmg_level_pitch(self.h, level)
        if a is None:
            return torch.zeros((ny + 2, p), dtype=torch.float64, device=self.device)
        return to_device(a, p, self.device)

    def block_grid(self, nrhs: int, arrays=None):
        """(ny+2, pitch, nrhs) device tensor in the block layout (zeros or the given arrays)."""
        import torch

        if arrays is None:
            return torch.zeros((self.ny + 2, self.pitch, nrhs), dtype=torch.float64, device=self.device)
        assert len(arrays) == nrhs
        return to_device_block(arrays, self.pitch, self.device)

    def vcycle(self, rhs, x, ncycles=1):
        bmg_vcycle(self.h, rhs, x, ncycles)

    def vcycle_block(self, rhs, x, ncycles=1):
        bmg_vcycle_block(self.h, rhs.shape[-1], rhs, x, ncycles)

    def solve_block(self, rhs, x, tol, maxiter):
        return bmg_solve_block(self.h, rhs.shape[-1], rhs, x, tol, maxiter)

    def pcg_block(self, rhs, x, tol, maxiter):
        return bmg_pcg_block(self.h, rhs.shape[-1], rhs, x, tol, maxiter)

    def solve(self, rhs, x, tol, maxiter):
        return bmg_solve(self.h, rhs, x, tol, maxiter)

    def pcg(self, rhs, x, tol, maxiter):
        return bmg_pcg(self.h, rhs, x, tol, maxiter)

    def residual_norm(self, rhs, x):
        return bmg_residual_norm(self.h, rhs, x)

    def close(self):
        if getattr(self, "h", None) is not None:
            bmg_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
