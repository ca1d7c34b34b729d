"""Multi-GPU plumbing for the row-slab solver (bmg_setup_dist), argument
marshalling only: an NCCL communicator over the torch.distributed ranks and
the rank-local slab arrays in the layout include/bmg.h defines (global rows
[row0, row0+nrows) = owned rows + BMG_HALO ghost rows).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from . import bmg

_nccl = None


class ncclUniqueId(ctypes.Structure):  # passed BY VALUE to ncclCommInitRank
    _fields_ = [("internal", ctypes.c_char * 128)]


def nccl_lib_path() -> str:
    """The libnccl.so.2 that torch bundles (the one its NCCL process group uses)."""
    import importlib.util

    spec = importlib.util.find_spec("nvidia.nccl")
    for base in (spec.submodule_search_locations or []) if spec else []:
        p = os.path.join(base, "lib", "libnccl.so.2")
        if os.path.exists(p):
            return p
    return "libnccl.so.2"


def _lib():
    global _nccl
    if _nccl is None:
        _nccl = ctypes.CDLL(nccl_lib_path(), mode=ctypes.RTLD_GLOBAL)
        _nccl.ncclGetUniqueId.argtypes = [ctypes.POINTER(ncclUniqueId)]
        _nccl.ncclCommInitRank.argtypes = [ctypes.POINTER(ctypes.c_void_p), ctypes.c_int, ncclUniqueId,
                                           ctypes.c_int]
        _nccl.ncclGetErrorString.restype = ctypes.c_char_p
    return _nccl


def nccl_comm(world: int, rank: int):
    """Create an NCCL communicator over the torch.distributed group (unique id
    broadcast through torch.distributed).  Call with the CUDA device set."""
    import torch.distributed as dist

    L = _lib()
    uid = ncclUniqueId()
    if rank == 0:
        rc = L.ncclGetUniqueId(ctypes.byref(uid))
        if rc != 0:
            raise RuntimeError(f"ncclGetUniqueId: {L.ncclGetErrorString(rc).decode()}")
    obj = [bytes(ctypes.string_at(ctypes.addressof(uid), 128))]
    if world > 1:
        dist.broadcast_object_list(obj, src=0)
    uid = ncclUniqueId.from_buffer_copy(obj[0])
    comm = ctypes.c_void_p()
    rc = L.ncclCommInitRank(ctypes.byref(comm), world, uid, rank)
    if rc != 0:
        raise RuntimeError(f"ncclCommInitRank: {L.ncclGetErrorString(rc).decode()}")
    return comm


def local_layout(nx: int, ny: int, world: int, rank: int, params=None):
    """(row0, nrows, ylo, yhi, kdist) of this rank's level-0 local arrays."""
    yb, k = bmg.bmg_partition(nx, ny, world, params)
    ylo, yhi = yb[rank], yb[rank + 1]
    row0 = max(ylo - bmg.BMG_HALO, 0)
    row1 = min(yhi + bmg.BMG_HALO, ny + 2)
    return row0, row1 - row0, ylo, yhi, k


class DistSolver:
    """One rank of the slab-partitioned solver for a problems.Stencil (global)."""

    def __init__(self, stencil, world: int, rank: int, comm, params=None, pitch: int | None = None,
                 device="cuda", loopback: bool = False, nccl_lib: str | None = None, peer: bool = False):
        self.nx, self.ny, self.kind = stencil.nx, stencil.ny, stencil.kind
        self.pitch = pitch or bmg.default_pitch(self.nx)
        self.device = device
        self.loopback = loopback
        c = bmg.bmg_comm_t()
        c.nranks, c.rank, c.loopback = world, rank, 1 if loopback else 0
        c.peer = 1 if peer else 0
        c.nccl_comm = comm.value if comm is not None else None
        # nccl_lib: another libnccl ABI implementation to dlopen (tests: the one-GPU CUDA-IPC shim)
        c.nccl_lib = (nccl_lib or nccl_lib_path()).encode() if not loopback else None
        self._comm = c
        if loopback:
            self.row0, self.nrows = 0, self.ny + 2
            planes = [bmg.to_device(p, self.pitch, device) for p in stencil.plane_list()]
        else:
            self.row0, self.nrows, self.ylo, self.yhi, self.kdist = local_layout(self.nx, self.ny, world, rank,
                                                                                 params)
            planes = [self.local(p) for p in stencil.plane_list()]
        self.h = bmg.bmg_setup_dist(planes, self.kind, self.nx, self.ny, self.pitch, c, params)
        del planes

    def local(self, a: np.ndarray | None = None):
        """Rank-local device array (rows [row0, row0+nrows)) of a global (ny+2, nx+2) array."""
        import torch

        t = torch.zeros((self.nrows, self.pitch), dtype=torch.float64, device=self.device)
        if a is not None:
            t[:, : a.shape[1]] = torch.from_numpy(np.ascontiguousarray(a[self.row0: self.row0 + self.nrows])).to(
                self.device)
        return t

    def vcycle(self, rhs, x, ncycles=1):
        bmg.bmg_vcycle(self.h, rhs, x, ncycles)

    def residual_norm(self, rhs, x):
        return bmg.bmg_residual_norm(self.h, rhs, x)

    def close(self):
        if getattr(self, "h", None) is not None:
            bmg.bmg_destroy(self.h)
            self.h = None
