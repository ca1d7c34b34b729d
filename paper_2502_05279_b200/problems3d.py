"""Seeded synthetic 3-D inputs (c18).

Shared by the oracle tests, the GPU parity tests and bench.py; it holds NO
multigrid arithmetic -- it discretises -div(D grad u) = f (Eq. (1), in
three dimensions) into the stencil planes the C ABI takes (``include/bmg3.h``).

* vertex-centred unknowns on an nx*ny*nz interior with a homogeneous
  Dirichlet ghost ring, h = 1/(n+1); D is cell-wise constant on the
  (nx+1)(ny+1)(nz+1) cells, cell (a,b,c) spanning nodes [a,a+1]x[b,b+1]x[c,c+1];
  per-axis anisotropy factors (ax, ay, az) multiply the x-, y-, z-flux terms;
* 7-point: each face coupling is the mean of the four cells sharing the dual
  face, times the axis factor: W(i,j,k) = -ax*mean(D(i-1, j-1..j, k-1..k)),
  likewise S, B; O = -(sum of the six couplings) before Dirichlet
  elimination.  D == 1 gives O = 6, W = S = B = -1;
* 27-point: the Q1 (trilinear) finite-element stiffness matrix, assembled
  cell by cell from K_cell = D(cell) (ax Kx My Mz + ay Mx Ky Mz + az Mx My Kz)
  with the 1-D stiffness K = [[1,-1],[-1,1]] and mass M = [[1/3,1/6],[1/6,1/3]].
  D == 1 gives O = 8/3, face 0, edge -1/6, corner -1/12.
* rhs = h^2 f; random fields use numpy PCG64 (seed 42 default).

Arrays have shape (nz+2, ny+2, nx+2) (x fastest) with the ghost ring.  Plane
entries are matrix entries: plane_e(p) = A[p, p+off_e] for the 13 offsets
that precede the centre in e = (dz+1)*9+(dy+1)*3+(dx+1) order (LOWER13).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

# the 13 stored offsets (dx, dy, dz), e = 0..12, and their names
LOWER13 = [(dx, dy, dz) for dz in (-1, 0, 1) for dy in (-1, 0, 1) for dx in (-1, 0, 1)][:13]
NAMES13 = ["BSW", "BS", "BSE", "BW", "B", "BE", "BNW", "BN", "BNE", "SW", "S", "SE", "W"]


@dataclass
class Stencil3:
    """Symmetric-half stencil planes of an nx*ny*nz interior (ghost ring included)."""

    kind: int  # 7 -> planes O, W, S, B ; 27 -> O + the 13 lower entries (NAMES13 order)
    nx: int
    ny: int
    nz: int
    planes: dict  # name -> (nz+2, ny+2, nx+2) float64

    def plane_names(self):
        return ["O", "W", "S", "B"] if self.kind == 7 else ["O"] + NAMES13

    def plane_list(self):
        return [self.planes[n] for n in self.plane_names()]

    def stacked(self) -> np.ndarray:
        """(nplanes, nz+2, ny+2, nx+2) contiguous, ABI plane order."""
        return np.ascontiguousarray(np.stack(self.plane_list()), dtype=np.float64)


def h_of(n: int) -> float:
    return 1.0 / (n + 1)


# ----------------------------------------------------------------- D fields
def d3_constant(nx, ny, nz, value=1.0) -> np.ndarray:
    """Cell field of shape (nz+1, ny+1, nx+1): D[c, b, a] is cell (a, b, c)."""
    return np.full((nz + 1, ny + 1, nx + 1), float(value))


def d3_checkerboard(nx, ny, nz, block, jump=1e4, offset=0) -> np.ndarray:
    """D = jump on cells with (floor(a/block)+floor(b/block)+floor(c/block)) odd, else 1."""
    a = (np.arange(nx + 1) + offset) // block
    b = (np.arange(ny + 1) + offset) // block
    c = (np.arange(nz + 1) + offset) // block
    odd = (c[:, None, None] + b[None, :, None] + a[None, None, :]) % 2 == 1
    return np.where(odd, float(jump), 1.0)


def d3_lognormal(nx, ny, nz, sigma=1.0, seed=42) -> np.ndarray:
    rng = np.random.Generator(np.random.PCG64(seed))
    return np.exp(sigma * rng.standard_normal((nz + 1, ny + 1, nx + 1)))


# ----------------------------------------------------------------- operators
def fv7(D: np.ndarray, ax=1.0, ay=1.0, az=1.0) -> Stencil3:
    """7-point finite-volume stencil (c18) from a cell field D (nz+1, ny+1, nx+1)."""
    nz, ny, nx = D.shape[0] - 1, D.shape[1] - 1, D.shape[2] - 1
    sh = (nz + 2, ny + 2, nx + 2)
    W, S, B = np.zeros(sh), np.zeros(sh), np.zeros(sh)
    # W(i,j,k): cells a = i-1, b in {j-1, j}, c in {k-1, k}; i in 1..nx+1, j, k in 1..n
    Dw = D[:-1, :-1, :] + D[1:, :-1, :] + D[:-1, 1:, :] + D[1:, 1:, :]  # (nz, ny, nx+1): over b, c
    W[1:nz + 1, 1:ny + 1, 1:nx + 2] = -ax * Dw / 4.0
    Ds = D[:-1, :, :-1] + D[1:, :, :-1] + D[:-1, :, 1:] + D[1:, :, 1:]  # (nz, ny+1, nx): over a, c
    S[1:nz + 1, 1:ny + 2, 1:nx + 1] = -ay * Ds / 4.0
    Db = D[:, :-1, :-1] + D[:, 1:, :-1] + D[:, :-1, 1:] + D[:, 1:, 1:]  # (nz+1, ny, nx): over a, b
    B[1:nz + 2, 1:ny + 1, 1:nx + 1] = -az * Db / 4.0
    O = np.zeros(sh)
    I = (slice(1, nz + 1), slice(1, ny + 1), slice(1, nx + 1))
    O[I] = -(W[1:nz + 1, 1:ny + 1, 1:nx + 1] + W[1:nz + 1, 1:ny + 1, 2:nx + 2] + S[1:nz + 1, 1:ny + 1, 1:nx + 1]
             + S[1:nz + 1, 2:ny + 2, 1:nx + 1] + B[1:nz + 1, 1:ny + 1, 1:nx + 1] + B[2:nz + 2, 1:ny + 1, 1:nx + 1])
    return Stencil3(7, nx, ny, nz, {"O": O, "W": W, "S": S, "B": B})


def _kref(ox, oy, oz, ax, ay, az):
    """Q1 element stiffness between two vertices of one cell whose coordinates
    differ on the axes where o != 0 (K same/diff = 1/-1, M same/diff = 1/3, 1/6)."""
    K = lambda o: -1.0 if o else 1.0  # noqa: E731
    M = lambda o: 1.0 / 6.0 if o else 1.0 / 3.0  # noqa: E731
    return ax * K(ox) * M(oy) * M(oz) + ay * M(ox) * K(oy) * M(oz) + az * M(ox) * M(oy) * K(oz)


def q1_27(D: np.ndarray, ax=1.0, ay=1.0, az=1.0) -> Stencil3:
    """27-point Q1 FE stiffness stencil (c18), assembled over the cells."""
    nz, ny, nx = D.shape[0] - 1, D.shape[1] - 1, D.shape[2] - 1
    sh = (nz + 2, ny + 2, nx + 2)
    planes = {}
    # entry (o) at node p = sum over cells containing p and p+o; per axis, cell index
    # choices: o=0 -> {p-1, p}; o=-1 -> {p-1}; o=+1 -> {p}; cell index range [0, n].
    ch = {0: (-1, 0), -1: (-1,), 1: (0,)}
    def cell_sum(ox, oy, oz):
        out = np.zeros((nz + 1, ny + 1, nx + 1))  # nodes 1..n+1 per axis (the +1 row feeds symmetry / O)
        acc = np.zeros((nz + 1, ny + 1, nx + 1))
        for cz in ch[oz]:
            for cy in ch[oy]:
                for cx in ch[ox]:
                    # node index n in 1..N+1 -> cell index n + c in [0, N]; clip out-of-range cells
                    zi = np.arange(1, nz + 2) + cz
                    yi = np.arange(1, ny + 2) + cy
                    xi = np.arange(1, nx + 2) + cx
                    mz = (zi >= 0) & (zi <= nz)
                    my = (yi >= 0) & (yi <= ny)
                    mx = (xi >= 0) & (xi <= nx)
                    blk = D[np.clip(zi, 0, nz)][:, np.clip(yi, 0, ny)][:, :, np.clip(xi, 0, nx)]
                    acc += blk * (mz[:, None, None] & my[None, :, None] & mx[None, None, :])
        out[:] = acc * _kref(ox, oy, oz, ax, ay, az)
        return out

    for name, (dx, dy, dz) in zip(NAMES13, LOWER13):
        P = np.zeros(sh)
        P[1:, 1:, 1:] = cell_sum(dx, dy, dz)
        planes[name] = P
    O = np.zeros(sh)
    O[1:, 1:, 1:] = cell_sum(0, 0, 0)
    O[nz + 1, :, :] = 0.0
    O[:, ny + 1, :] = 0.0
    O[:, :, nx + 1] = 0.0
    planes["O"] = O
    return Stencil3(27, nx, ny, nz, planes)


def poisson7(n, ny=None, nz=None) -> Stencil3:
    ny = n if ny is None else ny
    nz = n if nz is None else nz
    return fv7(d3_constant(n, ny, nz))


# ----------------------------------------------------------------- fields
def rhs_const(nx, ny, nz, value=1.0) -> np.ndarray:
    """f = h^2 * value on the interior (h from nx), ring 0."""
    g = np.zeros((nz + 2, ny + 2, nx + 2))
    g[1:-1, 1:-1, 1:-1] = value * h_of(nx) ** 2
    return g


def random_interior(nx, ny, nz, seed=42, lo=-1.0, hi=1.0) -> np.ndarray:
    rng = np.random.Generator(np.random.PCG64(seed))
    g = np.zeros((nz + 2, ny + 2, nx + 2))
    g[1:-1, 1:-1, 1:-1] = rng.uniform(lo, hi, (nz, ny, nx))
    return g


WORKLOADS3 = {
    # name: (builder(n) -> Stencil3, relax mode, description) -- DESIGN.md §4
    "poisson7": (lambda n: poisson7(n), "point", "7-point Poisson, D = 1"),
    "aniso7": (lambda n: fv7(d3_constant(n, n, n), az=1e-3), "planes",
               "7-point, z-coupling 1e-3 (strong xy planes)"),
    "checkeraniso7": (lambda n: fv7(d3_checkerboard(n, n, n, max(1, (n + 1) // 8), 1e4), az=1e-3), "planes",
                      "7-point, 1e4 checkerboard of (n+1)/8-cell cubes, z-coupling 1e-3"),
    "checker27": (lambda n: q1_27(d3_checkerboard(n, n, n, max(1, (n + 1) // 8), 1e4)), "point",
                  "27-point Q1, 1e4 checkerboard of (n+1)/8-cell cubes"),
    "lognormal7": (lambda n: fv7(d3_lognormal(n, n, n)), "point", "7-point, lognormal D (parity)"),
}
