"""Dense-matrix definitions for the 3-D pins (tests/test_oracle3d.py), written
independently of oracle/bmg3_oracle.c: the operator straight from the ABI's
symmetric-half planes, P from the documented c19 slot layout, and the method's
steps (colour-ordered Gauss-Seidel, residual, P^T, P, the V-cycle, zebra plane
Gauss-Seidel) as dense linear algebra."""
from __future__ import annotations

import itertools

import numpy as np

from paper_2502_05279_b200.problems3d import LOWER13, NAMES13

SLOT = {1: 0, 2: 2, 4: 4, 3: 6, 5: 10, 6: 14, 7: 18}


def index3(nx, ny, nz):
    idx = -np.ones((nz + 2, ny + 2, nx + 2), dtype=np.int64)
    idx[1:-1, 1:-1, 1:-1] = np.arange(nx * ny * nz).reshape(nz, ny, nx)
    return idx


def dense_from_planes3(s) -> np.ndarray:
    """A[p, p+o] = plane_o(p) = A[p+o, p]; ghost couplings dropped."""
    idx = index3(s.nx, s.ny, s.nz)
    n = s.nx * s.ny * s.nz
    A = np.zeros((n, n))
    offs = {"W": (-1, 0, 0), "S": (0, -1, 0), "B": (0, 0, -1)} if s.kind == 7 else dict(zip(NAMES13, LOWER13))
    for k, j, i in itertools.product(range(1, s.nz + 1), range(1, s.ny + 1), range(1, s.nx + 1)):
        p = idx[k, j, i]
        A[p, p] = s.planes["O"][k, j, i]
        for name, (dx, dy, dz) in offs.items():
            q = idx[k + dz, j + dy, i + dx]
            if q < 0:
                continue
            A[p, q] = s.planes[name][k, j, i]
            A[q, p] = s.planes[name][k, j, i]
    return A


def dense_from_full3(st) -> np.ndarray:
    nz, ny, nx = st.shape[0] - 2, st.shape[1] - 2, st.shape[2] - 2
    idx = index3(nx, ny, nz)
    A = np.zeros((nx * ny * nz, nx * ny * nz))
    for k, j, i in itertools.product(range(1, nz + 1), range(1, ny + 1), range(1, nx + 1)):
        for e in range(27):
            dx, dy, dz = e % 3 - 1, (e // 3) % 3 - 1, e // 9 - 1
            q = idx[k + dz, j + dy, i + dx]
            if q >= 0:
                A[idx[k, j, i], q] = st[k, j, i, e]
    return A


def parents(i, j, k, ci):
    """[(I, J, K, w)] of fine point (i,j,k) read from the c19 slot layout."""
    q = (i, j, k)
    m = (i & 1) | (j & 1) << 1 | (k & 1) << 2
    if m == 0:
        return [(i // 2, j // 2, k // 2, 1.0)]
    Q = [(c + 1) // 2 if c & 1 else c // 2 for c in q]
    odd = [d for d in range(3) if q[d] & 1]
    out = []
    for corner in range(1 << len(odd)):
        C = list(Q)
        for b, d in enumerate(odd):
            if not (corner >> b) & 1:
                C[d] -= 1
        out.append((C[0], C[1], C[2], ci[Q[2], Q[1], Q[0], SLOT[m] + corner]))
    return out


def dense_P3(ci, nx, ny, nz) -> np.ndarray:
    ncx, ncy, ncz = nx // 2, ny // 2, nz // 2
    fi, ci_idx = index3(nx, ny, nz), index3(ncx, ncy, ncz)
    P = np.zeros((nx * ny * nz, ncx * ncy * ncz))
    for k, j, i in itertools.product(range(1, nz + 1), range(1, ny + 1), range(1, nx + 1)):
        for I, J, K, w in parents(i, j, k, ci):
            c = ci_idx[K, J, I]
            if c >= 0:
                P[fi[k, j, i], c] += w
    return P


def to_vec3(g):
    return g[1:-1, 1:-1, 1:-1].reshape(-1).copy()


def to_grid3(v, nx, ny, nz):
    g = np.zeros((nz + 2, ny + 2, nx + 2))
    g[1:-1, 1:-1, 1:-1] = v.reshape(nz, ny, nx)
    return g


def colour_masks3(nx, ny, nz, kind):
    k, j, i = np.meshgrid(np.arange(1, nz + 1), np.arange(1, ny + 1), np.arange(1, nx + 1), indexing="ij")
    k, j, i = k.reshape(-1), j.reshape(-1), i.reshape(-1)
    if kind == 7:
        col = (i + j + k) % 2
        return [col == c for c in range(2)]
    col = (i % 2) + 2 * (j % 2) + 4 * (k % 2)
    return [col == c for c in range(8)]


def dense_gs3(A, f, u, masks, nsweeps):
    """Multicolour GS: within a colour the points do not couple, so the colour's
    update is one Jacobi step on its rows."""
    u = u.copy()
    d = np.diag(A)
    for _ in range(nsweeps):
        for m in masks:
            r = f - A @ u
            u[m] = u[m] + r[m] / d[m]
    return u


def plane_masks(nx, ny, nz):
    k = np.repeat(np.arange(1, nz + 1), nx * ny)
    return k


def dense_zebra_exact(A, f, u, nx, ny, nz, nsweeps):
    """Zebra xy-plane block GS with EXACT plane solves: planes k mod 2 = 0, then 1."""
    u = u.copy()
    k = plane_masks(nx, ny, nz)
    for _ in range(nsweeps):
        for c in (0, 1):
            for kk in range(1, nz + 1):
                if kk % 2 != c:
                    continue
                m = k == kk
                g = f[m] - A[np.ix_(m, ~m)] @ u[~m]
                u[m] = np.linalg.solve(A[np.ix_(m, m)], g)
    return u
