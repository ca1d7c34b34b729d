"""T0 dense-matrix definitions, written independently of oracle/.

These helpers assemble the operator straight from the symmetric-half planes
the ABI defines (include/bmg.h), build P from the oracle's fig:restrict_kernel
restriction applied to unit vectors (R = P^T), and evaluate the
method's steps as dense linear algebra so that a dropped term, wrong sign,
wrong index or transposed operand in the oracle fails a comparison.
"""
from __future__ import annotations

import numpy as np


def interior_index(nx, ny):
    """Map (j, i) interior -> lexicographic row (x fastest)."""
    idx = -np.ones((ny + 2, nx + 2), dtype=np.int64)
    idx[1:ny + 1, 1:nx + 1] = np.arange(nx * ny).reshape(ny, nx)
    return idx


def dense_from_planes(stencil) -> np.ndarray:
    """A from the ABI planes: A[p, p+off_d] = plane_d(p) and, by symmetry,
    A[p+off_d, p] = plane_d(p); couplings to ghost points dropped."""
    nx, ny = stencil.nx, stencil.ny
    idx = interior_index(nx, ny)
    n = nx * ny
    A = np.zeros((n, n))
    offs = {"W": (-1, 0), "S": (0, -1), "SW": (-1, -1), "NW": (-1, 1)}
    for j in range(1, ny + 1):
        for i in range(1, nx + 1):
            p = idx[j, i]
            A[p, p] = stencil.planes["O"][j, i]
            for name, (dx, dy) in offs.items():
                if name not in stencil.planes:
                    continue
                q = idx[j + dy, i + dx]
                if q < 0:
                    continue
                A[p, q] = stencil.planes[name][j, i]
                A[q, p] = stencil.planes[name][j, i]
    return A


def dense_from_full(st) -> np.ndarray:
    """A from a full 9-entry stencil (ny+2, nx+2, 9) (rows only; no symmetry assumed)."""
    ny, nx = st.shape[0] - 2, st.shape[1] - 2
    idx = interior_index(nx, ny)
    A = np.zeros((nx * ny, nx * ny))
    dxy = [(-1, -1), (0, -1), (1, -1), (-1, 0), (0, 0), (1, 0), (-1, 1), (0, 1), (1, 1)]
    for j in range(1, ny + 1):
        for i in range(1, nx + 1):
            for d, (dx, dy) in enumerate(dxy):
                q = idx[j + dy, i + dx]
                if q >= 0:
                    A[idx[j, i], q] = st[j, i, d]
    return A


def to_vec(g):
    return g[1:-1, 1:-1].reshape(-1).copy()


def to_grid(v, nx, ny):
    g = np.zeros((ny + 2, nx + 2))
    g[1:ny + 1, 1:nx + 1] = v.reshape(ny, nx)
    return g


def dense_P_from_restriction(orc, ci, nx, ny) -> np.ndarray:
    """P (fine x coarse) with P^T = the oracle's restriction (fig:restrict_kernel)."""
    ncx, ncy = nx // 2, ny // 2
    P = np.zeros((nx * ny, ncx * ncy))
    for p in range(nx * ny):
        e = np.zeros(nx * ny)
        e[p] = 1.0
        P[p, :] = to_vec(orc.restrict(ci, to_grid(e, nx, ny)))
    return P


def colour_masks(nx, ny, kind):
    J, I = np.meshgrid(np.arange(1, ny + 1), np.arange(1, nx + 1), indexing="ij")
    col = ((I + J) % 2) if kind == 5 else ((I % 2) + 2 * (J % 2))
    ncol = 2 if kind == 5 else 4
    return [col.reshape(-1) == c for c in range(ncol)]


def dense_gs(A, f, u, masks, nsweeps):
    """Multicolour GS as dense block updates: within a colour the points are
    uncoupled (asserted), so u_c <- u_c + D_c^{-1}(f - A u)_c is exact GS."""
    u = u.copy()
    d = np.diag(A)
    for m in masks:
        blk = A[np.ix_(m, m)]
        assert np.count_nonzero(blk - np.diag(np.diag(blk))) == 0, "same-colour coupling"
    for _ in range(nsweeps):
        for m in masks:
            r = f - A @ u
            u[m] = u[m] + r[m] / d[m]
    return u


def dense_vcycle(As, Ps, kinds, dims, f, u, nu1, nu2):
    """Recursive V(nu1,nu2) on dense matrices, coarsest exact solve (c9)."""

    def rec(l, f, u):
        if l == len(As) - 1:
            return np.linalg.solve(As[l], f)
        nx, ny = dims[l]
        masks = colour_masks(nx, ny, kinds[l])
        u = dense_gs(As[l], f, u, masks, nu1)
        r = f - As[l] @ u
        fc = Ps[l].T @ r
        ec = rec(l + 1, fc, np.zeros_like(fc))
        u = u + Ps[l] @ ec
        return dense_gs(As[l], f, u, masks, nu2)

    return rec(0, f, u)
