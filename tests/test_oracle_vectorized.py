"""An independent, vectorised NumPy implementation of the hierarchical cycle (§3.3,
:380-387 §4.1: copy the augmented subdomain, k sub-iterations of the update with the halo frozen,
write the owned interior into the next array), written from the paper and tests/_brute.plan_1d's
block rule — no code shared with oracle/hjo.cpp — must reproduce the oracle's iterates BIT FOR BIT
on grids with many tiles and k > 1 (the regime no closed form pins), 1D and 2D, f64 and f32,
ragged tiles and overlap.  NumPy evaluates the same parenthesisation elementwise in IEEE round-
to-nearest, so any disagreement is a bug in one of the two."""
import numpy as np
import pytest

import oracle
from paper_2006_16465_b200.inputs import make_problem
from tests import _brute


def _ringed(p, dim, dt):
    nx, ny = p["nx"], p["ny"]
    if dim == 1:
        z = np.zeros(nx + 2, dtype=dt)
        z[1:-1] = p["x0"].astype(dt)
        z[0], z[-1] = dt(p["bc"][0]), dt(p["bc"][1])
        return z
    z = np.zeros((ny + 2, nx + 2), dtype=dt)
    z[1:-1, 1:-1] = p["x0"].reshape(ny, nx).astype(dt)
    bc = p["bc"].astype(dt)
    z[0, 1:-1], z[-1, 1:-1] = bc[:nx], bc[nx:2 * nx]
    z[1:-1, 0], z[1:-1, -1] = bc[2 * nx:2 * nx + ny], bc[2 * nx + ny:]
    return z


def cycle_np(z, rhs, dim, tx, ty, k, ox, oy, dt):
    """One hierarchical cycle; rhs = T(h^2 f) on the interior (ny x nx or nx)."""
    out = z.copy()
    quarter, half = dt(0.25), dt(0.5)
    if dim == 1:
        for lo, hi, a0, a1 in _brute.plan_1d(len(z) - 2, tx, ox):
            A = z[lo - 1:hi + 2].copy()
            r = rhs[lo - 1:hi]
            for _ in range(k):
                B = A.copy()
                B[1:-1] = half * ((A[:-2] + A[2:]) + r)
                A = B
            out[a0:a1 + 1] = A[a0 - lo + 1:a1 - lo + 2]
        return out
    nyi, nxi = z.shape[0] - 2, z.shape[1] - 2
    for ylo, yhi, b0, b1 in _brute.plan_1d(nyi, ty, oy):
        for xlo, xhi, a0, a1 in _brute.plan_1d(nxi, tx, ox):
            A = z[ylo - 1:yhi + 2, xlo - 1:xhi + 2].copy()
            r = rhs[ylo - 1:yhi, xlo - 1:xhi]
            for _ in range(k):
                B = A.copy()
                B[1:-1, 1:-1] = quarter * (((A[1:-1, :-2] + A[1:-1, 2:]) + (A[:-2, 1:-1] + A[2:, 1:-1])) + r)
                A = B
            out[b0:b1 + 1, a0:a1 + 1] = A[b0 - ylo + 1:b1 - ylo + 2, a0 - xlo + 1:a1 - xlo + 2]
    return out


CASES = [  # (dim, nx, ny, tile, k, overlap, dtype, proto, cycles)
    (2, 128, 96, (32, 32), 16, 0, "f64", "R", 3),
    (2, 100, 70, (32, 32), 7, 0, "f64", "P", 4),      # ragged tiles
    (2, 96, 80, (16, 8), 11, 0, "f32", "R", 3),
    (2, 90, 64, (32, 32), 9, (4, 6), "f64", "R", 2),  # overlapping blocks, shifted last block
    (2, 64, 64, (12, 10), 5, (2, 4), "f32", "Q", 3),
    (1, 1000, 1, (32, 1), 16, 0, "f64", "R", 5),
    (1, 777, 1, (64, 1), 9, 10, "f32", "R", 4),
]


@pytest.mark.parametrize("dim,nx,ny,tile,k,overlap,dtype,proto,cycles", CASES)
def test_oracle_equals_independent_vectorised_cycle(dim, nx, ny, tile, k, overlap, dtype, proto, cycles):
    p = make_problem(proto, dim, nx, ny)
    dt = np.float64 if dtype == "f64" else np.float32
    ox, oy = overlap if isinstance(overlap, tuple) else (overlap, overlap if dim == 2 else 0)
    h2 = p["h"] * p["h"]
    rhs = (h2 * p["f"]).astype(dt)                 # T(h^2 f): the double product, one rounding
    if dim == 2:
        rhs = rhs.reshape(ny, nx)
    z = _ringed(p, dim, dt)
    for _ in range(cycles):
        z = cycle_np(z, rhs, dim, tile[0], tile[1], k, ox, oy, dt)
    x_np = z[1:-1] if dim == 1 else z[1:-1, 1:-1]
    o = oracle.solve(dim, nx, ny if dim == 2 else 1, p["h"], p["f"], p["bc"], p["x0"], mode="hier",
                     tile=tile if dim == 2 else tile[0], k=k, overlap=(ox, oy) if dim == 2 else ox, dtype=dtype,
                     tol=0.0, max_cycles=cycles)
    assert np.array_equal(o["x"].reshape(x_np.shape), x_np.astype(np.float64))
