"""Seeded synthetic inputs shared by tests, bench.py and the oracle harness.

This module holds NONE of the method's arithmetic: it only produces the
problem data (h, f, boundary ring g, initial guess x0) that both the CUDA path
and the CPU oracle consume.  Recipes:

* ``P`` — the paper's workload: f = 1, x0 = 1, g = 0.
* ``M`` — manufactured: f = pi^2 sin(pi x) (1D) or 2 pi^2 sin(pi x) sin(pi y)
  (2D), x0 = 0, g = 0 (the north star's sin(pi x) check).
* ``R`` — parity stress: f, x0 ~ U[-1, 1) from splitmix64(seed + linear index),
  g ~ U[-1, 1) from the same stream offset by nx*ny.
* ``Q`` — exact polynomial solutions the 3/5-point stencils reproduce exactly:
  1D u = x^3 - x (f = -6x, g = 0); 2D u = x^2 + y^2 (f = -4, g = u on the
  ring, non-zero Dirichlet data).  x0 = 0.

General coefficients (``make_general``; f is then b, h unused):

* ``A`` — 2D anisotropic Poisson on the unit square with nx != ny: dx = 1/(nx+1), dy = 1/(ny+1),
  {a, c, e, f, d} = {-1/dx^2, -1/dx^2, -1/dy^2, -1/dy^2, 2/dx^2 + 2/dy^2},
  b = 1, x0 = 1, g = 0 (the paper's protocol on a rectangular grid).
* ``G`` — random diagonally dominant coefficients with mixed signs (2D: five constants; 1D: a_i,
  d_i, c_i per point), b, x0, g ~ U[-1, 1) (parity stress for every coefficient's position).
* ``V`` — 1D variable-coefficient diffusion -(k u')' = 1, k(x) = 1 + 0.5 sin(2 pi x + 0.1 p) for
  problem p: a_i = -k(x_i - h/2)/h^2, c_i = -k(x_i + h/2)/h^2, d_i = -(a_i + c_i); x0 = 1, g = 0.

Grid: h = 1/(nx+1); interior node i (0-based) sits at x = (i+1) h; in 2D the
same h is used along y (the ABI has one spacing, "if dx = dy").
Arrays are row-major with x fastest: f[j*nx + i].  The 2D ring layout is
[south(nx) | north(nx) | west(ny) | east(ny)]; 1D is [g_left, g_right].
"""
from __future__ import annotations

import numpy as np

SEED = 2006164650
_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix64(idx: np.ndarray) -> np.ndarray:
    """splitmix64 of a uint64 counter array (vectorised, wrapping arithmetic)."""
    with np.errstate(over="ignore"):
        z = idx.astype(np.uint64) + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def uniform_pm1(start: int, count: int) -> np.ndarray:
    """U[-1, 1) doubles from splitmix64(start + 0..count-1)."""
    idx = np.arange(count, dtype=np.uint64) + np.uint64(start)
    u = (splitmix64(idx) >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)
    return 2.0 * u - 1.0


def make_problem(protocol: str, dim: int, nx: int, ny: int | None = None, seed: int = SEED,
                 batch: int = 1):
    """Return dict(dim, nx, ny, h, f, bc, x0) as float64 numpy arrays.

    dim 1 with batch > 1: `batch` independent problems stacked row-major (ny = batch); P, M and Q
    give identical copies (the paper's "1024 copies"), R independent random data.
    """
    if dim == 1:
        if batch > 1:
            one = make_problem(protocol, 1, nx, seed=seed)
            if protocol == "R":
                n = nx * batch
                f = uniform_pm1(seed, n)
                x0 = uniform_pm1(seed + 7 * n + 13, n)
                bc = uniform_pm1(seed + n, 2 * batch)
            else:
                f, x0, bc = np.tile(one["f"], batch), np.tile(one["x0"], batch), np.tile(one["bc"], batch)
            return dict(dim=1, nx=nx, ny=batch, h=one["h"], f=f, bc=bc, x0=x0)
        ny = 1
    elif ny is None:
        ny = nx
    n = nx * ny
    h = 1.0 / (nx + 1)
    xs = (np.arange(nx, dtype=np.float64) + 1.0) * h
    ys = (np.arange(ny, dtype=np.float64) + 1.0) * h
    nbc = 2 if dim == 1 else 2 * nx + 2 * ny
    bc = np.zeros(nbc)
    if protocol == "P":
        f = np.ones(n)
        x0 = np.ones(n)
    elif protocol == "M":
        if dim == 1:
            f = np.pi ** 2 * np.sin(np.pi * xs)
        else:
            f = (2.0 * np.pi ** 2 * np.outer(np.sin(np.pi * ys), np.sin(np.pi * xs))).reshape(-1)
        x0 = np.zeros(n)
    elif protocol == "R":
        f = uniform_pm1(seed, n)
        x0 = uniform_pm1(seed + 7 * n + 13, n)
        bc = uniform_pm1(seed + n, nbc)
    elif protocol == "Q":
        if dim == 1:
            f = -6.0 * xs
        else:
            f = np.full(n, -4.0)
            xe = (np.arange(nx + 2, dtype=np.float64)) * h
            ye = (np.arange(ny + 2, dtype=np.float64)) * h
            south = xe[1:-1] ** 2 + ye[0] ** 2
            north = xe[1:-1] ** 2 + ye[-1] ** 2
            west = xe[0] ** 2 + ye[1:-1] ** 2
            east = xe[-1] ** 2 + ye[1:-1] ** 2
            bc = np.concatenate([south, north, west, east])
        x0 = np.zeros(n)
    else:
        raise ValueError(f"unknown protocol {protocol!r}")
    return dict(dim=dim, nx=nx, ny=ny, h=h, f=np.ascontiguousarray(f), bc=bc,
                x0=np.ascontiguousarray(x0))


def exact_solution_Q(dim: int, nx: int, ny: int | None = None) -> np.ndarray:
    """Nodal values of protocol Q's exact solution (interior, row-major)."""
    h = 1.0 / (nx + 1)
    xs = (np.arange(nx, dtype=np.float64) + 1.0) * h
    if dim == 1:
        return xs ** 3 - xs
    ny = nx if ny is None else ny
    ys = (np.arange(ny, dtype=np.float64) + 1.0) * h
    return (xs[None, :] ** 2 + ys[:, None] ** 2).reshape(-1)


def make_general(recipe: str, dim: int, nx: int, ny: int | None = None, seed: int = SEED,
                 batch: int = 1):
    """General-coefficient problem: dict(dim, nx, ny, h, f (= b), bc, x0, stencil).

    stencil: 2D {a, c, e, f, d} (west, east, south, north, centre; Eq. 10);
    1D the planes [a | d | c] of nx*batch values (Eq. 4; ny = batch)."""
    if dim == 1:
        ny = batch
    elif ny is None:
        ny = nx
    n = nx * ny
    nbc = 2 * ny if dim == 1 else 2 * nx + 2 * ny
    if recipe == "A":
        if dim != 2:
            raise ValueError("recipe A is 2D")
        dx, dy = 1.0 / (nx + 1), 1.0 / (ny + 1)
        st = np.array([-1 / dx ** 2, -1 / dx ** 2, -1 / dy ** 2, -1 / dy ** 2, 2 / dx ** 2 + 2 / dy ** 2])
        f, x0, bc = np.ones(n), np.ones(n), np.zeros(nbc)
    elif recipe == "G":
        u = (uniform_pm1(seed + 3 * n + 101, 3 * n + 8) + 1.0) / 2.0   # U[0, 1)
        if dim == 2:
            a, c, e, fn = -(0.2 + 0.8 * u[0]), -(0.2 + 0.8 * u[1]), 0.1 + 0.4 * u[2], -(0.2 + 0.8 * u[3])
            d = (abs(a) + abs(c) + abs(e) + abs(fn)) * (1.02 + 0.3 * u[4])
            st = np.array([a, c, e, fn, d])
        else:
            a = -(0.1 + 0.9 * u[:n])
            c = u[n:2 * n] - 0.3
            d = (np.abs(a) + np.abs(c)) * (1.02 + 0.5 * u[2 * n:3 * n])
            st = np.concatenate([a, d, c])
        f = uniform_pm1(seed, n)
        x0 = uniform_pm1(seed + 7 * n + 13, n)
        bc = uniform_pm1(seed + n, nbc)
    elif recipe == "V":
        if dim != 1:
            raise ValueError("recipe V is 1D")
        h = 1.0 / (nx + 1)
        xs = (np.arange(nx, dtype=np.float64) + 1.0) * h
        ph = 0.1 * np.arange(ny, dtype=np.float64)[:, None]
        kl = 1.0 + 0.5 * np.sin(2 * np.pi * (xs[None, :] - h / 2) + ph)
        kr = 1.0 + 0.5 * np.sin(2 * np.pi * (xs[None, :] + h / 2) + ph)
        a, c = (-kl / h ** 2).reshape(-1), (-kr / h ** 2).reshape(-1)
        st = np.concatenate([a, -(a + c), c])
        f, x0, bc = np.ones(n), np.ones(n), np.zeros(nbc)
    else:
        raise ValueError(f"unknown recipe {recipe!r}")
    return dict(dim=dim, nx=nx, ny=ny, h=1.0, f=np.ascontiguousarray(f), bc=bc,
                x0=np.ascontiguousarray(x0), stencil=np.ascontiguousarray(st, dtype=np.float64))
