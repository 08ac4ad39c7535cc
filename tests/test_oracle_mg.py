"""Pins of the multigrid oracle (reading c24) — CPU only.

The V-cycle with the hierarchical smoother has no closed form, so the oracle is pinned against
what the mathematics fixes:
  * the transfer operators on polynomials: full weighting maps x^2 + y^2 + xy to itself plus the
    exact second-moment term, annihilates the discrete residual of a discrete-harmonic field, and
    (bi)linear interpolation reproduces bilinear functions exactly;
  * one oracle V-cycle equals a dense matrix-level V-cycle (tests/_brute.py: smoother maps from
    per-tile damped Jacobi matrices, R, P, K of every level) on tiny grids, for several tiles, k,
    nu1/nu2 and omega;
  * two-grid with an exact coarse solve equals x + P A_c^-1 R r (textbook formula);
  * the asymptotic V-cycle rate equals the spectral radius of the dense V-cycle matrix;
  * the direct solution is a fixed point; the converged iterate meets the residual error bound;
  * h-independent convergence (the multigrid property) and omega = 1 failing to smooth the
    checkerboard mode (why the reading damps).
"""
from __future__ import annotations

import numpy as np
import pytest

import oracle
from paper_2006_16465_b200.inputs import make_problem
from tests import _brute


def _ring_of(dim, nx, ny, bc):
    z = _brute.ringed_vector(dim, nx, ny, bc, np.zeros(nx * (ny if dim == 2 else 1)))
    return z


def test_restriction_of_quadratic_is_exact():
    # x = 0, ring 0 => s = a.  2D full weighting: FW(i^2) = i^2 + 1/2, FW(j^2) = j^2 + 1/2,
    # FW(ij) = ij (index units), so the coarse h2f = 4 FW(a) = 4 (a(2I, 2J) + 1).
    nx, ny = 9, 7
    i, j = np.meshgrid(np.arange(1, nx + 1), np.arange(1, ny + 1))
    a = (i * i + j * j + i * j).astype(np.float64)
    out = oracle.mg_transfer(2, "restrict", nx, ny, np.zeros(nx * ny), a).reshape(3, 4)
    I, J = np.meshgrid(np.arange(1, 5), np.arange(1, 4))
    want = 4.0 * ((2 * I) ** 2 + (2 * J) ** 2 + (2 * I) * (2 * J) + 1.0)
    assert np.array_equal(out, want)
    # 1D: s_L + 2 s_C + s_R of i^2 = 4 i^2 + 2 at i = 2I, per independent problem
    n, B = 11, 3
    a1 = np.tile(np.arange(1, n + 1, dtype=np.float64) ** 2, B) * np.repeat([1.0, 2.0, -1.0], n)
    out1 = oracle.mg_transfer(1, "restrict", n, B, np.zeros(n * B), a1).reshape(B, 5)
    I1 = np.arange(1, 6)
    for b, sc in enumerate([1.0, 2.0, -1.0]):
        assert np.array_equal(out1[b], sc * (4.0 * (2 * I1) ** 2 + 2.0))


def test_restriction_uses_the_residual_of_the_iterate():
    # x = i^2 - j^2 is discrete-harmonic (its 5-point Laplacian is 0), ring values included, so
    # with a = c (constant) the residual is s = c everywhere and the coarse h2f = 4 c; a sign or
    # neighbour error in the residual breaks this.
    nx, ny = 7, 9
    f = lambda i, j: float(i * i - j * j)
    x = np.array([[f(i, j) for i in range(1, nx + 1)] for j in range(1, ny + 1)])
    bc = np.concatenate([[f(i, 0) for i in range(1, nx + 1)], [f(i, ny + 1) for i in range(1, nx + 1)],
                         [f(0, j) for j in range(1, ny + 1)], [f(nx + 1, j) for j in range(1, ny + 1)]])
    out = oracle.mg_transfer(2, "restrict", nx, ny, x, np.full(nx * ny, 3.0), bc=bc)
    assert np.array_equal(out, np.full(3 * 4, 12.0))
    # without the ring data the boundary-adjacent residuals change (ring is read)
    out0 = oracle.mg_transfer(2, "restrict", nx, ny, x, np.full(nx * ny, 3.0), bc=None)
    assert not np.array_equal(out0, out)
    # 1D: x = i (linear, harmonic) with its ring values
    n = 9
    x1 = np.arange(1, n + 1, dtype=np.float64)
    o1 = oracle.mg_transfer(1, "restrict", n, 1, x1, np.full(n, -1.0), bc=np.array([0.0, n + 1.0]))
    assert np.array_equal(o1, np.full(4, -4.0))


def test_interpolation_reproduces_bilinear_functions():
    nx, ny = 9, 11
    nxc, nyc = 4, 5
    g = 0.75
    Ic, Jc = np.meshgrid(np.arange(1, nxc + 1), np.arange(1, nyc + 1))
    e = g * Ic * Jc                                  # zero on the coarse rings I = 0, J = 0
    x = np.linspace(-1, 1, nx * ny)
    out = oracle.mg_transfer(2, "correct", nx, ny, x, e).reshape(ny, nx) - x.reshape(ny, nx)
    i, j = np.meshgrid(np.arange(1, nx + 1), np.arange(1, ny + 1))
    want = g * (i / 2.0) * (j / 2.0)
    inner = (i <= nx - 2) & (j <= ny - 2)            # stencils that stay inside [0, n_c]
    assert np.allclose(out[inner], want[inner], rtol=0, atol=1e-15)
    # the last fine column/row lies between coarse point n_c and the zero ring
    assert np.allclose(out[1, nx - 1], 0.5 * g * nxc * 1.0, atol=1e-15)
    assert np.allclose(out[ny - 1, 1], 0.5 * g * 1.0 * nyc, atol=1e-15)
    # 1D: linear e = I reproduced, last point half of e(n_c)
    n = 9
    o1 = oracle.mg_transfer(1, "correct", n, 1, np.zeros(n), np.arange(1.0, 5.0))
    assert np.array_equal(o1[:-1], np.arange(1, n) / 2.0) and o1[-1] == 2.0


CASES_2D = [  # (nx, ny, tile, k, nu1, nu2, omega, coarse_cycles)
    (7, 7, (4, 4), 2, 1, 1, 0.8, 3),
    (15, 7, (8, 4), 3, 2, 1, 0.7, 2),
    (15, 15, (16, 16), 1, 1, 2, 0.8, 1),
    (15, 15, (5, 3), 4, 0, 1, 0.6, 2),
]


@pytest.mark.parametrize("nx,ny,tile,k,nu1,nu2,omega,cc", CASES_2D)
def test_vcycle_equals_dense_vcycle_2d(nx, ny, tile, k, nu1, nu2, omega, cc):
    p = make_problem("R", 2, nx, ny)
    V, L = _brute.vcycle_dense(2, nx, ny, tile, k, nu1, nu2, omega, cc)
    h2f = p["h"] ** 2 * p["f"]
    ring = _ring_of(2, nx, ny, p["bc"])
    x = p["x0"].copy()
    o = oracle.solve_mg(2, nx, ny, p["h"], p["f"], p["bc"], p["x0"], tile=tile, k=k, nu1=nu1, nu2=nu2,
                        omega=omega, coarse_cycles=cc, tol=0.0, max_cycles=2)
    assert o["levels"] == L
    for c in range(2):
        x = V(0, x, h2f, ring)
    assert np.allclose(o["x"].reshape(-1), x, rtol=0, atol=1e-12 * np.abs(x).max())


@pytest.mark.parametrize("n,tile,k,nu1,nu2,omega", [(15, 4, 2, 1, 1, 2 / 3), (31, 8, 3, 2, 0, 0.5)])
def test_vcycle_equals_dense_vcycle_1d(n, tile, k, nu1, nu2, omega):
    B = 3
    p = make_problem("R", 1, n, batch=B)
    V, L = _brute.vcycle_dense(1, n, 1, (tile, 1), k, nu1, nu2, omega, 2)
    o = oracle.solve_mg(1, n, B, p["h"], p["f"], p["bc"], p["x0"], tile=tile, k=k, nu1=nu1, nu2=nu2,
                        omega=omega, coarse_cycles=2, tol=0.0, max_cycles=1)
    assert o["levels"] == L
    for b in range(B):
        ring = np.zeros(n + 2)
        ring[0], ring[-1] = p["bc"][2 * b], p["bc"][2 * b + 1]
        x = V(0, p["x0"][b * n:(b + 1) * n].copy(), p["h"] ** 2 * p["f"][b * n:(b + 1) * n], ring)
        assert np.allclose(o["x"][b], x, rtol=0, atol=1e-12 * np.abs(x).max())


def test_two_grid_with_exact_coarse_solve_is_textbook_formula():
    # levels = 2 and many undamped coarse cycles on a single 3x3 tile: the coarse problem is
    # solved to machine precision, so one V-cycle is S2 (x1 + P A_c^-1 R r(x1)), x1 = S1 x0.
    nx = ny = 7
    p = make_problem("R", 2, nx, ny)
    h2f = p["h"] ** 2 * p["f"]
    ring = _ring_of(2, nx, ny, p["bc"])
    M, G = _brute.smoother_affine(2, nx, ny, 4, 4, 2, 0.8)
    K = _brute.stencil_ringed(2, nx, ny)
    R = _brute.full_weighting(2, nx, ny)
    P = _brute.linear_interpolation(2, nx, ny)
    Kc = _brute.stencil_ringed(2, 3, 3)
    Ac = Kc[:, [j * 5 + i for j in range(1, 4) for i in range(1, 4)]]   # interior columns
    z = lambda x: ring + _brute.ringed_vector(2, nx, ny, None, x)
    x1 = M @ z(p["x0"]) + G @ h2f
    e = np.linalg.solve(Ac, 4.0 * (R @ (h2f - K @ z(x1))))
    x2 = x1 + P @ e
    x3 = M @ z(x2) + G @ h2f
    o = oracle.solve_mg(2, nx, ny, p["h"], p["f"], p["bc"], p["x0"], tile=(4, 4), k=2, nu1=1, nu2=1,
                        omega=0.8, coarse_cycles=200, levels=2, tol=0.0, max_cycles=1)
    assert o["levels"] == 2
    assert np.allclose(o["x"].reshape(-1), x3, rtol=0, atol=1e-12 * np.abs(x3).max())


def test_asymptotic_rate_is_spectral_radius_of_vcycle():
    nx = ny = 15
    tile, k, nu1, nu2, om = (4, 4), 2, 1, 1, 0.8
    V, _ = _brute.vcycle_dense(2, nx, ny, tile, k, nu1, nu2, om, 2)
    n = nx * ny
    ring = np.zeros((nx + 2) * (ny + 2))
    Mv = np.column_stack([V(0, np.eye(n)[:, q], np.zeros(n), ring) for q in range(n)])
    rho = max(abs(np.linalg.eigvals(Mv)))
    assert 0.0 < rho < 0.3
    p = make_problem("R", 2, nx, ny)
    o = oracle.solve_mg(2, nx, ny, p["h"], np.zeros(n), None, p["x0"], tile=tile, k=k, nu1=nu1, nu2=nu2,
                        omega=om, coarse_cycles=2, tol=0.0, max_cycles=200)
    h = o["history"]
    rate = (h[200] / h[150]) ** (1 / 50)
    # the second eigenvalue is 0.194 (|l2/l1| = 0.964): after 150 cycles its share is < 0.5%
    assert abs(rate - rho) < 2e-3 * rho, (rate, rho)


@pytest.mark.parametrize("dim,n,ny", [(2, 31, 15), (1, 63, 2)])
def test_direct_solution_is_a_fixed_point(dim, n, ny):
    p = make_problem("R", dim, n, ny) if dim == 2 else make_problem("R", 1, n, batch=ny)
    xs = _brute.direct_solve(dim, n, ny if dim == 2 else 1, p["h"], p["f"], p["bc"]) if dim == 2 else \
        np.concatenate([_brute.direct_solve(1, n, 1, p["h"], p["f"][b * n:(b + 1) * n],
                                            p["bc"][2 * b:2 * b + 2]) for b in range(ny)])
    o = oracle.solve_mg(dim, n, ny, p["h"], p["f"], p["bc"], xs, tile=(8, 8) if dim == 2 else 8, k=3,
                        tol=0.0, max_cycles=1)
    assert np.max(np.abs(o["x"].reshape(-1) - xs)) <= 1e-12 * np.max(np.abs(xs))


def test_converged_error_within_residual_bound():
    n = 63
    p = make_problem("M", 2, n)
    o = oracle.solve_mg(2, n, n, p["h"], p["f"], p["bc"], p["x0"], tile=(32, 32), k=4, tol=1e-10,
                        max_cycles=50)
    assert o["converged"] and o["cycles"] <= 20
    xs = _brute.direct_solve(2, n, n, p["h"], p["f"], p["bc"])
    lam_min = 8 * np.sin(np.pi * p["h"] / 2) ** 2 / p["h"] ** 2
    err = np.linalg.norm(o["x"].reshape(-1) - xs)
    assert err <= o["history"][-1] / lam_min * (1 + 1e-6) + 1e-12


def test_h_independent_convergence_and_damping_needed():
    rates = []
    for n in (31, 63, 127, 255):
        p = make_problem("M", 2, n)
        o = oracle.solve_mg(2, n, n, p["h"], p["f"], p["bc"], p["x0"], tile=(32, 32), k=4, tol=0.0,
                            max_cycles=6)
        h = o["history"]
        rates.append((h[6] / h[1]) ** (1 / 5))
    assert max(rates) < 0.2, rates                      # textbook V(1,1): ~0.1-0.2 per cycle
    assert max(rates) / min(rates) < 1.6, rates          # grid-size independent
    # undamped smoothing leaves the checkerboard mode: the same V-cycle with omega = 1 on a
    # checkerboard initial error converges far slower (or not at all)
    n = 63
    i, j = np.meshgrid(np.arange(n), np.arange(n))
    x0 = ((-1.0) ** (i + j)).reshape(-1)
    r = {}
    for om in (0.8, 1.0):
        o = oracle.solve_mg(2, n, n, 1.0 / (n + 1), np.zeros(n * n), None, x0, tile=(64, 64), k=1,
                            omega=om, tol=0.0, max_cycles=5)
        r[om] = (o["history"][5] / o["history"][0]) ** (1 / 5)
    assert r[0.8] < 0.5 and r[1.0] > 0.95, r


def test_fp32_tracks_fp64_and_invalid_configs():
    n = 63
    p = make_problem("P", 2, n)
    kw = dict(tile=(32, 32), k=4, tol=1e-5, max_cycles=50)
    o64 = oracle.solve_mg(2, n, n, p["h"], p["f"], p["bc"], p["x0"], **kw)
    o32 = oracle.solve_mg(2, n, n, p["h"], p["f"], p["bc"], p["x0"], dtype="f32", **kw)
    assert o64["converged"] and o32["converged"] and abs(o64["cycles"] - o32["cycles"]) <= 1
    assert np.max(np.abs(o64["x"] - o32["x"])) < 1e-4 * np.max(np.abs(o64["x"]))
    with pytest.raises(ValueError):   # even grid: no coarse level
        oracle.solve_mg(2, 64, 64, 1 / 65, np.ones(64 * 64), tile=(32, 32))
    with pytest.raises(ValueError):
        oracle.solve_mg(2, 63, 63, 1 / 64, np.ones(63 * 63), omega=1.5)
    with pytest.raises(ValueError):
        oracle.solve_mg(2, 63, 63, 1 / 64, np.ones(63 * 63), nu1=0, nu2=0)
