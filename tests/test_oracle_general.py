"""Pins of the oracle's general-coefficient path (reading c23)
against things other than itself: a closed-form eigenmode decay (anisotropic grid, catches a
transposed x/y coefficient pair), direct solves of the matrices of Eq. 4 / Eq. 10 assembled here
(catches sign, position and rhs errors), the brute-force affine map of one hierarchical cycle with
exact quotients, the reduction to the paper's model problem, and the residual definition."""
import numpy as np
import pytest
import scipy.linalg as sla

import oracle
from paper_2006_16465_b200.inputs import make_general, make_problem
from tests import _brute


def _x(r):
    return np.asarray(r["x"], dtype=np.float64).reshape(-1)


@pytest.mark.parametrize("mode,tile,k", [("classic", (1, 1), 1), ("hier", (24, 40), 5)])
def test_anisotropic_mode_decay_closed_form(mode, tile, k):
    # PAPER.md:413-419 with dx != dy: the Jacobi iteration matrix of the 5-point operator has the
    # eigenvector sin(pi x) sin(pi y) with eigenvalue (cos(pi dx)/dx^2 + cos(pi dy)/dy^2) /
    # (1/dx^2 + 1/dy^2); one tile covering the grid = k plain sweeps.
    nx, ny = 24, 40
    p = make_general("A", 2, nx, ny)
    dx, dy = 1.0 / (nx + 1), 1.0 / (ny + 1)
    xs, ys = np.arange(1, nx + 1) * dx, np.arange(1, ny + 1) * dy
    x0 = np.outer(np.sin(np.pi * ys), np.sin(np.pi * xs)).reshape(-1)
    rho = (np.cos(np.pi * dx) / dx ** 2 + np.cos(np.pi * dy) / dy ** 2) / (1 / dx ** 2 + 1 / dy ** 2)
    rho_t = (np.cos(np.pi * dy) / dx ** 2 + np.cos(np.pi * dx) / dy ** 2) / (1 / dx ** 2 + 1 / dy ** 2)
    assert abs(rho - rho_t) > 1e-4       # the pin can see a transposition
    cyc = 5 if mode == "classic" else 1
    r = oracle.solve(2, nx, ny, 1.0, np.zeros(nx * ny), None, x0, mode=mode, tile=tile, k=k, tol=0.0,
                     max_cycles=cyc, stencil=p["stencil"])
    np.testing.assert_allclose(_x(r), rho ** 5 * x0, rtol=1e-12, atol=1e-15)


@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("ovl", [(0, 0), (2, 2), (4, 0)])
def test_general_2d_fixed_point_is_direct_solve(dtype, ovl):
    nx, ny = 20, 13
    p = make_general("G", 2, nx, ny)
    A = _brute.general_matrix(2, nx, ny, p["stencil"])
    xs = np.linalg.solve(A, _brute.general_rhs(2, nx, ny, p["stencil"], p["f"], p["bc"]))
    tol = 1e-12 if dtype == "f64" else 1e-5
    r = oracle.solve(2, nx, ny, 1.0, p["f"], p["bc"], p["x0"], mode="hier", tile=(8, 4), k=6,
                     overlap=ovl, tol=tol, dtype=dtype, stencil=p["stencil"], max_cycles=4000)
    assert r["converged"]
    np.testing.assert_allclose(_x(r), xs, atol=(1e-9 if dtype == "f64" else 2e-4) * np.abs(xs).max())


@pytest.mark.parametrize("recipe,batch", [("G", 3), ("V", 2)])
@pytest.mark.parametrize("mode", ["hier", "classic"])
def test_general_1d_fixed_point_is_banded_solve(recipe, batch, mode):
    nx = 37
    p = make_general(recipe, 1, nx, batch=batch)
    st = p["stencil"].reshape(3, batch, nx)
    r = oracle.solve(1, nx, batch, 1.0, p["f"], p["bc"], p["x0"], mode=mode, tile=(8, 1), k=4,
                     overlap=2, tol=1e-12, stencil=p["stencil"], max_cycles=20000)
    assert r["converged"]
    got = np.asarray(r["x"]).reshape(batch, nx)
    for b in range(batch):
        a, d, c = st[0, b], st[1, b], st[2, b]
        ab = np.zeros((3, nx))
        ab[0, 1:], ab[1], ab[2, :-1] = c[:-1], d, a[1:]
        rhs = p["f"].reshape(batch, nx)[b].copy()
        rhs[0] -= a[0] * p["bc"][2 * b]
        rhs[-1] -= c[-1] * p["bc"][2 * b + 1]
        xs = sla.solve_banded((1, 1), ab, rhs)
        np.testing.assert_allclose(got[b], xs, atol=1e-9 * np.abs(xs).max())


@pytest.mark.parametrize("dim,nx,ny,tile,ovl,k", [
    (2, 9, 7, (4, 3), (0, 0), 3), (2, 11, 8, (6, 4), (2, 2), 4), (2, 10, 9, (4, 4), (0, 2), 2),
    (1, 23, 1, (6, 1), (0, 0), 5), (1, 23, 1, (8, 1), (4, 0), 3)])
def test_general_cycle_is_brute_affine_map(dim, nx, ny, tile, ovl, k):
    p = make_general("G", dim, nx, ny if dim == 2 else None)
    M, g = _brute.cycle_affine_general(dim, nx, ny, p["stencil"], p["f"], tile[0], tile[1], k,
                                       ovl[0], ovl[1])
    z = _brute.ringed_vector(dim, nx, ny, p["bc"], p["x0"])
    want = M @ z + g
    r = oracle.solve(dim, nx, ny, 1.0, p["f"], p["bc"], p["x0"], mode="hier", tile=tile, k=k,
                     overlap=ovl, tol=0.0, max_cycles=1, stencil=p["stencil"])
    np.testing.assert_allclose(_x(r), want, rtol=0, atol=1e-13 * max(1.0, np.abs(want).max()))


def test_poisson_coefficients_reduce_to_the_model_problem():
    # {a, c, e, f, d} = {-1, -1, -1, -1, 4}/h^2 and b = f is the paper's 2D Poisson system
    # (PAPER.md:413-420): same iteration up to rounding, same residual history.
    n = 40
    pp = make_problem("R", 2, n)
    h = pp["h"]
    st = np.array([-1, -1, -1, -1, 4.0]) / h ** 2
    kw = dict(mode="hier", tile=(16, 8), k=5, overlap=(2, 0), tol=1e-8)
    r0 = oracle.solve(2, n, n, h, pp["f"], pp["bc"], pp["x0"], **kw)
    r1 = oracle.solve(2, n, n, h, pp["f"], pp["bc"], pp["x0"], stencil=st, **kw)
    assert r0["cycles"] == r1["cycles"]
    np.testing.assert_allclose(r1["history"], r0["history"], rtol=1e-9)
    np.testing.assert_allclose(_x(r1), _x(r0), atol=1e-12 * np.abs(_x(r0)).max())


@pytest.mark.parametrize("dim", [1, 2])
def test_general_residual_definition(dim):
    nx, ny = (30, 2) if dim == 1 else (17, 12)
    p = make_general("G", dim, nx, ny if dim == 2 else None, batch=ny if dim == 1 else 1)
    # the definition against the assembled matrix
    if dim == 2:
        A = _brute.general_matrix(2, nx, ny, p["stencil"])
        want = np.linalg.norm(_brute.general_rhs(2, nx, ny, p["stencil"], p["f"], p["bc"]) - A @ p["x0"])
    else:
        st = p["stencil"].reshape(3, ny, nx)
        parts = []
        for b in range(ny):
            sb = np.concatenate([st[0, b], st[1, b], st[2, b]])
            A = _brute.general_matrix(1, nx, 1, sb)
            rb = _brute.general_rhs(1, nx, 1, sb, p["f"].reshape(ny, nx)[b], p["bc"][2 * b:2 * b + 2])
            parts.append((rb - A @ p["x0"].reshape(ny, nx)[b]) / st[1, b])
        want = np.linalg.norm(np.concatenate(parts))
    got = oracle.residual_general(dim, nx, ny, p["f"], p["bc"], p["x0"], p["stencil"])
    assert got == pytest.approx(want, rel=1e-12)
    # the solver's history uses the same norm (reading c23)
    r = oracle.solve(dim, nx, ny, 1.0, p["f"], p["bc"], p["x0"], mode="hier", tile=(8, 4), k=3,
                     tol=0.0, max_cycles=3, stencil=p["stencil"])
    assert r["history"][0] == pytest.approx(want, rel=1e-12)
    assert r["history"][3] == pytest.approx(
        oracle.residual_general(dim, nx, ny, p["f"], p["bc"], _x(r), p["stencil"]), rel=1e-10)


def test_general_validation():
    p = make_general("G", 2, 8, 8)
    bad = p["stencil"].copy()
    bad[4] = 0.0
    with pytest.raises(ValueError):
        oracle.solve(2, 8, 8, 1.0, p["f"], None, None, tile=(4, 4), k=2, stencil=bad)
    bad[4] = np.nan
    with pytest.raises(ValueError):
        oracle.solve(2, 8, 8, 1.0, p["f"], None, None, tile=(4, 4), k=2, stencil=bad)
    q = make_general("G", 1, 10, batch=2)
    bad = q["stencil"].copy()
    bad[20 + 3] = 0.0   # a d_i
    with pytest.raises(ValueError):
        oracle.solve(1, 10, 2, 1.0, q["f"], None, None, tile=(4, 1), k=2, stencil=bad)
