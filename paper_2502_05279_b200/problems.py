"""Seeded synthetic inputs for the BoxMG path (the problem of Eq. (1)).

This module is shared by the oracle tests, the GPU parity tests and bench.py.
It holds NO multigrid arithmetic: it only discretises the model problem
-div(D grad u) = f into the per-point stencil planes the C ABI takes
(``include/bmg.h``) and draws seeded fields.  Recipes (SURVEY.md
§8(c) c2 and §8(d)):

* vertex-centred unknowns on an nx*ny interior with a homogeneous Dirichlet
  ghost ring, h = 1/(n+1); D is cell-wise constant on the (nx+1)*(ny+1) cells,
  cell (a,b) spanning nodes [a,a+1]x[b,b+1];
* 5-point couplings are the arithmetic mean of the two cells sharing the dual
  edge: W(i,j) = -(D(i-1,j-1)+D(i-1,j))/2, S(i,j) = -(D(i-1,j-1)+D(i,j-1))/2,
  O = -(W(i,j)+W(i+1,j)+S(i,j)+S(i,j+1)) (before Dirichlet elimination);
  D == 1 gives O=4, W=S=-1;
* 9-point anisotropic: the Q1 bilinear-FE stencil of -(eps u_xx + u_yy);
* rhs = h^2 f; random fields use numpy PCG64 (seed 42 default,
  SPEC S:529).

Arrays are float64 numpy arrays of shape (ny+2, nx+2) (row-major, x fastest,
pitch nx+2) with the ghost ring included.  Plane entries are matrix entries
(SURVEY §8(b) sign convention): plane_d(i,j) = A[(i,j), (i,j)+off_d] with
off_W=(-1,0), off_S=(0,-1), off_SW=(-1,-1), off_NW=(-1,+1).  Couplings that
point into the ghost ring are left as generated; the solver drops them.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class Stencil:
    """Symmetric-half stencil planes of an nx*ny interior (ghost ring included)."""

    kind: int  # 5 -> planes O,W,S ; 9 -> planes O,W,S,SW,NW
    nx: int
    ny: int
    planes: dict  # name -> (ny+2, nx+2) float64

    def plane_list(self):
        names = ["O", "W", "S"] + (["SW", "NW"] if self.kind == 9 else [])
        return [self.planes[n] for n in names]


def h_of(n: int) -> float:
    """Mesh width on the unit square with n interior points."""
    return 1.0 / (n + 1)


# ----------------------------------------------------------------- D fields
def d_constant(nx: int, ny: int, value: float = 1.0) -> np.ndarray:
    """Cell field D of shape (ny+1, nx+1): D[b, a] is cell (a, b)."""
    return np.full((ny + 1, nx + 1), float(value))


def d_checkerboard(nx: int, ny: int, block: int, jump: float = 1e6, offset: int = 0) -> np.ndarray:
    """D = jump on cells with (floor((a+offset)/block) + floor((b+offset)/block)) odd, else 1.

    Config 2 uses block=128 on 1023^2 (8x8 coarse-aligned blocks), config 5
    block=512; ``offset`` shifts the pattern off the coarse grid.
    """
    a = np.arange(nx + 1) + offset
    b = np.arange(ny + 1) + offset
    odd = ((b[:, None] // block) + (a[None, :] // block)) % 2 == 1
    return np.where(odd, float(jump), 1.0)


def d_lognormal(nx: int, ny: int, sigma: float = 2.0, seed: int = 42) -> np.ndarray:
    """D = exp(sigma * N(0,1)) per cell, numpy PCG64."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return np.exp(sigma * rng.standard_normal((ny + 1, nx + 1)))


def d_node_jump(nx: int, ny: int, x_node: int, jump: float = 1e6) -> np.ndarray:
    """D = jump on cells a >= x_node (a vertical interface through node column x_node)."""
    a = np.arange(nx + 1)
    return np.where(a[None, :] >= x_node, float(jump), 1.0) * np.ones((ny + 1, 1))


# ------------------------------------------------------------- stencils
def stencil5_from_D(D: np.ndarray) -> Stencil:
    """5-point finite-volume stencil of -div(D grad u) (Eq. (1)).

    Couplings on the dual edges are the arithmetic mean of the two adjacent
    cells (reading c2).  Returns matrix-entry planes O, W, S on (ny+2, nx+2).
    """
    ny, nx = D.shape[0] - 1, D.shape[1] - 1
    W = np.zeros((ny + 2, nx + 2))
    S = np.zeros((ny + 2, nx + 2))
    # W(i,j), i in [1,nx+1], j in [1,ny]: cells (i-1, j-1) and (i-1, j)
    W[1:ny + 1, 1:nx + 2] = -0.5 * (D[0:ny, 0:nx + 1] + D[1:ny + 1, 0:nx + 1])
    # S(i,j), i in [1,nx], j in [1,ny+1]: cells (i-1, j-1) and (i, j-1)
    S[1:ny + 2, 1:nx + 1] = -0.5 * (D[0:ny + 1, 0:nx] + D[0:ny + 1, 1:nx + 1])
    O = np.zeros((ny + 2, nx + 2))
    O[1:ny + 1, 1:nx + 1] = -(W[1:ny + 1, 1:nx + 1] + W[1:ny + 1, 2:nx + 2]
                              + S[1:ny + 1, 1:nx + 1] + S[2:ny + 2, 1:nx + 1])
    return Stencil(5, nx, ny, {"O": O, "W": W, "S": S})


def stencil9_q1_aniso(nx: int, ny: int, eps: float = 1e-3) -> Stencil:
    """Q1 bilinear-FE stencil of -(eps u_xx + u_yy) (config 3, reading c2).

    O = 8(1+eps)/6, W = E = (2-4eps)/6, S = N = (2eps-4)/6, corners -(1+eps)/6.
    """
    shape = (ny + 2, nx + 2)
    O = np.zeros(shape)
    O[1:ny + 1, 1:nx + 1] = 8.0 * (1.0 + eps) / 6.0
    W = np.full(shape, (2.0 - 4.0 * eps) / 6.0)
    S = np.full(shape, (2.0 * eps - 4.0) / 6.0)
    C = np.full(shape, -(1.0 + eps) / 6.0)
    return Stencil(9, nx, ny, {"O": O, "W": W, "S": S, "SW": C.copy(), "NW": C.copy()})


def stencil9_random_spd(nx: int, ny: int, seed: int = 42) -> Stencil:
    """A random 9-point M-matrix-like stencil: negative couplings U(0.1,1),
    diagonal = sum |couplings| + U(0, 0.1) (strictly diagonally dominant, SPD)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    shape = (ny + 2, nx + 2)
    W = -rng.uniform(0.1, 1.0, shape)
    S = -rng.uniform(0.1, 1.0, shape)
    SW = -rng.uniform(0.1, 1.0, shape)
    NW = -rng.uniform(0.1, 1.0, shape)
    O = np.zeros(shape)
    tot = (-W[1:-1, 1:-1] - W[1:-1, 2:] - S[1:-1, 1:-1] - S[2:, 1:-1]
           - SW[1:-1, 1:-1] - SW[2:, 2:] - NW[1:-1, 1:-1] - NW[:-2, 2:])
    O[1:-1, 1:-1] = tot + rng.uniform(0.0, 0.1, (ny, nx))
    return Stencil(9, nx, ny, {"O": O, "W": W, "S": S, "SW": SW, "NW": NW})


# ------------------------------------------------------------- grid functions
def rhs_const(nx: int, ny: int, value: float = 1.0) -> np.ndarray:
    """rhs = h^2 * value on the interior (h from nx)."""
    h = h_of(max(nx, ny))
    f = np.zeros((ny + 2, nx + 2))
    f[1:ny + 1, 1:nx + 1] = h * h * value
    return f


def field_uniform(nx: int, ny: int, seed: int = 42, scale: float = 1.0) -> np.ndarray:
    """U(-1,1)*scale on the interior, 0 on the ghost ring (parity inputs, §8(d))."""
    rng = np.random.Generator(np.random.PCG64(seed))
    g = np.zeros((ny + 2, nx + 2))
    g[1:ny + 1, 1:nx + 1] = scale * rng.uniform(-1.0, 1.0, (ny, nx))
    return g


# ------------------------------------------------------------- named workloads
def workload(name: str, nx: int | None = None, ny: int | None = None) -> Stencil:
    """The BASELINE.json configs' operators by name."""
    if name == "poisson":
        return stencil5_from_D(d_constant(nx, ny))
    if name == "checker":  # config 2: 8x8 coarse-aligned blocks on 1023^2
        return stencil5_from_D(d_checkerboard(nx, ny, block=(nx + 1) // 8))
    if name == "checker_off3":
        return stencil5_from_D(d_checkerboard(nx, ny, block=(nx + 1) // 8, offset=3))
    if name == "checker512":  # config 5: fixed 512-cell blocks
        return stencil5_from_D(d_checkerboard(nx, ny, block=512))
    if name == "lognormal":
        return stencil5_from_D(d_lognormal(nx, ny))
    if name == "aniso":  # config 3
        return stencil9_q1_aniso(nx, ny, 1e-3)
    if name == "random9":
        return stencil9_random_spd(nx, ny)
    raise ValueError(f"unknown workload {name!r}")
