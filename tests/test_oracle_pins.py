"""Pins for the CPU oracle.  CPU only.

Each test checks the oracle against something other than itself: a closed
form, a value the paper prints (tests/golden/paper_values.json), a library
direct solve (scipy), a brute-force dense construction (tests/_brute.py), a
structural invariant, or cycle counts from an independent implementation
(tests/golden/cross_impl_counts.json).
"""
import json
import math
import os

import numpy as np
import pytest

import oracle
from paper_2006_16465_b200.inputs import make_problem, exact_solution_Q
from tests import _brute

GOLD = os.path.join(os.path.dirname(__file__), "golden")
PAPER = json.load(open(os.path.join(GOLD, "paper_values.json")))
COUNTS = json.load(open(os.path.join(GOLD, "cross_impl_counts.json")))


def run(p, **kw):
    return oracle.solve(p["dim"], p["nx"], p["ny"], p["h"], p["f"], p["bc"], p["x0"], **kw)


# ---------------------------------------------------------------- P10 ---------
def test_resource_figures_match_paper():
    """Shared-memory formula and block counts printed in the paper (P10)."""
    assert oracle.resource_figures(1, 1024, 1, 32)[2] == PAPER["smem_bytes_1d_tpb32_f64"]["value"]
    assert oracle.resource_figures(2, 1024, 1024, 32, 32)[2] == PAPER["smem_bytes_2d_32x32_f64"]["value"]
    assert oracle.resource_figures(1, 12, 1, 4)[0] == PAPER["blocks_1d_n12_tpb4"]["value"]
    assert oracle.resource_figures(2, 12, 12, 4, 4)[0] == PAPER["blocks_2d_12x12_4x4"]["value"]
    # "doubling either dimension of the subdomain would cause us to exceed" 48 kB
    lim = PAPER["smem_limit_2d_double_either_dim"]["value"]
    assert oracle.resource_figures(2, 1024, 1024, 64, 32)[2] > lim
    assert oracle.resource_figures(2, 1024, 1024, 32, 64)[2] > lim
    # one thread per DOF: N=1024, tpb=32 -> 32 blocks, 1024 threads (Eqs. 8-9 at o=0)
    assert oracle.resource_figures(1, 1024, 1, 32)[:2] == (32, 1024)
    # 4-byte figure for floats
    assert oracle.resource_figures(1, 1024, 1, 32, bytes_per_value=4)[2] == 400


# ------------------------------------------------ elemental update examples --
def test_single_sweep_from_zero_is_h2f_over_diag():
    """x_i = (b_i dx^2 + x_{i-1} + x_{i+1})/2; /4 in 2D."""
    for dim, n in ((1, 7), (2, 5)):
        p = make_problem("P", dim, n)
        p["x0"] = np.zeros_like(p["x0"])
        r = run(p, mode="classic", tol=0.0, max_cycles=1)
        expect = p["h"] ** 2 / (2.0 if dim == 1 else 4.0)
        x = r["x"].reshape(-1)
        # interior-of-interior points see zero neighbours after one sweep from zero
        assert np.all(x == expect)
    # 1D n=1: the direct solution is dx^2/2 and is a fixed point
    p = make_problem("P", 1, 1)
    r = run(p, mode="classic", tol=0.0, max_cycles=3)
    assert r["x"][0] == 0.25 / 2


# ---------------------------------------------------------------- P1 / P2 -----
@pytest.mark.parametrize("dim,nx,ny,tile", [(1, 37, 1, (8, 1)), (1, 64, 1, (16, 1)),
                                            (2, 19, 13, (4, 5)), (2, 16, 16, (8, 8)),
                                            (2, 33, 40, (32, 32))])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_k1_equals_classic_bitwise(dim, nx, ny, tile, dtype):
    """k = 1 'is exactly equivalent to performing Jacobi iteration'."""
    p = make_problem("R", dim, nx, ny)
    a = run(p, mode="hier", tile=tile, k=1, tol=0.0, max_cycles=60, dtype=dtype)
    b = run(p, mode="classic", tol=0.0, max_cycles=60, dtype=dtype)
    assert np.array_equal(a["x"], b["x"])
    assert np.array_equal(a["history"], b["history"])


@pytest.mark.parametrize("dim,n,k,c", [(1, 40, 5, 7), (2, 12, 3, 9), (2, 9, 4, 4)])
def test_single_tile_equals_classic_times_k(dim, n, k, c):
    """One tile covering the grid: its halo is the true ring, so a cycle is k exact sweeps (P2)."""
    p = make_problem("R", dim, n)
    a = run(p, mode="hier", tile=(n, n), k=k, tol=0.0, max_cycles=c)
    b = run(p, mode="classic", tol=0.0, max_cycles=c * k)
    assert np.array_equal(a["x"], b["x"])


# ---------------------------------------------------------------- P3 / P4 -----
def closed_form_sweeps(n, tol):
    """n* = ceil(ln tol / ln cos(pi h)), ln cos(pi h) = log1p(-2 sin^2(pi h/2))."""
    h = 1.0 / (n + 1)
    return math.ceil(math.log(tol) / math.log1p(-2.0 * math.sin(math.pi * h / 2) ** 2))


@pytest.mark.parametrize("dim,n,tol", [(1, 256, 1e-8), (1, 63, 1e-6), (2, 32, 1e-6)])
def test_manufactured_classic_decays_by_cos_pi_h(dim, n, tol):
    """sin is an eigenvector of the Jacobi matrix: r_{n+1} = cos(pi h) r_n every sweep (P3)."""
    p = make_problem("M", dim, n)
    r = run(p, mode="classic", tol=tol, max_cycles=10**6)
    rho = math.cos(math.pi / (n + 1))
    hist = r["history"]
    ratios = hist[1:] / hist[:-1]
    assert np.allclose(ratios[:2000], rho, rtol=1e-9, atol=0)
    assert r["converged"] and r["cycles"] == closed_form_sweeps(n, tol)


def test_manufactured_single_tile_cycles():
    """One tile of k sweeps on the sin mode: cycles = ceil(n*/k) (P4; SURVEY N=64,k=4 -> 3942)."""
    n, k, tol = 64, 4, 1e-8
    p = make_problem("M", 1, n)
    r = run(p, mode="hier", tile=n, k=k, tol=tol, max_cycles=10**6)
    assert r["cycles"] == math.ceil(closed_form_sweeps(n, tol) / k) == 3942


# ---------------------------------------------------------------- P5 / P6 -----
@pytest.mark.parametrize("dim,n", [(1, 64), (2, 24)])
def test_discrete_sine_solution_and_h2_error(dim, n):
    """u_h = s sin(pi x)[sin(pi y)], s = (pi h/2)^2 / sin^2(pi h/2) (P5 i); error vs u is O(h^2)."""
    p = make_problem("M", dim, n)
    r = run(p, mode="hier", tile=(8, 8), k=6, tol=1e-11, max_cycles=10**6)
    h = p["h"]
    s = (math.pi * h / 2) ** 2 / math.sin(math.pi * h / 2) ** 2
    xs = np.arange(1, n + 1) * h
    u = np.sin(np.pi * xs) if dim == 1 else np.outer(np.sin(np.pi * xs), np.sin(np.pi * xs))
    uh = s * u
    lam_min = (4 if dim == 1 else 8) * math.sin(math.pi * h / 2) ** 2 / h ** 2
    bound = r["history"][-1] / lam_min + 1e-13
    assert np.linalg.norm((r["x"] - uh).reshape(-1)) <= bound
    # the discretisation error max|u_h - u| = (s - 1) max|u|, s - 1 ~ pi^2 h^2 / 12
    err = np.abs(r["x"] - u).max()
    assert abs(err - (s - 1) * np.abs(u).max()) <= bound + 1e-12
    assert abs((s - 1) / (math.pi ** 2 * h ** 2 / 12) - 1) < 1e-2


def test_sine_error_is_second_order():
    """Halving h quarters max|x - sin(pi x)| (north star's O(h^2) check)."""
    errs = []
    for n in (15, 31, 63):
        p = make_problem("M", 1, n)
        r = run(p, mode="hier", tile=8, k=8, tol=1e-12, max_cycles=10**6)
        errs.append(np.abs(r["x"] - np.sin(np.pi * np.arange(1, n + 1) / (n + 1))).max())
    assert 3.9 < errs[0] / errs[1] < 4.1 and 3.9 < errs[1] / errs[2] < 4.1


@pytest.mark.parametrize("dim,n", [(1, 50), (2, 20)])
def test_polynomial_exact_solution(dim, n):
    """3/5-point stencils are exact for cubics/quadratics (P5 ii), incl. non-zero Dirichlet ring."""
    p = make_problem("Q", dim, n)
    r = run(p, mode="hier", tile=(8, 8), k=4, tol=1e-12, max_cycles=10**6)
    u = exact_solution_Q(dim, n)
    h = p["h"]
    lam_min = (4 if dim == 1 else 8) * math.sin(math.pi * h / 2) ** 2 / h ** 2
    assert np.linalg.norm(r["x"].reshape(-1) - u) <= r["history"][-1] / lam_min + 1e-12


@pytest.mark.parametrize("dim,n,ny,tile,k", [(1, 45, 1, (8, 1), 7), (2, 17, 11, (4, 4), 5)])
def test_error_bounded_by_residual(dim, n, ny, tile, k):
    """||x_c - x*|| <= ||r_c|| / lambda_min with x* from a sparse direct solve (P6, P7)."""
    p = make_problem("R", dim, n, ny)
    xs = _brute.direct_solve(dim, n, ny, p["h"], p["f"], p["bc"])
    h = p["h"]
    if dim == 1:
        lam_min = 4 * math.sin(math.pi * h / 2) ** 2 / h ** 2
    else:
        lam_min = (4 * math.sin(math.pi / (2 * (n + 1))) ** 2 + 4 * math.sin(math.pi / (2 * (ny + 1))) ** 2) / h ** 2
    for c in (1, 10, 100, 1000):
        r = run(p, mode="hier", tile=tile, k=k, tol=0.0, max_cycles=c)
        err = np.linalg.norm(r["x"].reshape(-1) - xs)
        assert err <= r["history"][-1] / lam_min * (1 + 1e-9) + 1e-12


@pytest.mark.parametrize("dim,n,ny,tile,k", [(1, 30, 1, (7, 1), 3), (2, 14, 10, (4, 3), 4),
                                             (2, 32, 32, (32, 32), 16)])
def test_direct_solution_is_a_fixed_point(dim, n, ny, tile, k):
    """x* (scipy) is a fixed point of one hierarchical cycle and of a classic sweep (P7)."""
    p = make_problem("R", dim, n, ny)
    xs = _brute.direct_solve(dim, n, ny, p["h"], p["f"], p["bc"])
    p["x0"] = xs
    for mode in ("hier", "classic"):
        r = run(p, mode=mode, tile=tile, k=k, tol=0.0, max_cycles=1)
        assert np.abs(r["x"].reshape(-1) - xs).max() <= 1e-13 * max(1.0, np.abs(xs).max())


# ---------------------------------------------------------------- P8 ----------
@pytest.mark.parametrize("dim,nx,ny,tile,k", [(1, 29, 1, (8, 1), 3), (1, 16, 1, (4, 1), 6),
                                              (2, 9, 7, (4, 3), 2), (2, 12, 12, (4, 4), 5)])
def test_cycle_equals_dense_affine_map(dim, nx, ny, tile, k):
    """One oracle cycle == M z + g from per-tile Jacobi matrices (P8, brute force)."""
    p = make_problem("R", dim, nx, ny)
    M, g, _, _ = _brute.cycle_affine(dim, nx, ny, p["h"], p["f"], tile[0], tile[1], k)
    z = _brute.ringed_vector(dim, nx, ny, p["bc"], p["x0"])
    r = run(p, mode="hier", tile=tile, k=k, tol=0.0, max_cycles=1)
    ref = M @ z + g
    assert np.allclose(r["x"].reshape(-1), ref, rtol=0, atol=1e-13 * max(1, np.abs(ref).max()))


@pytest.mark.parametrize("dim,nx,ny,tile,k", [(1, 24, 1, (6, 1), 3), (2, 8, 8, (4, 4), 2)])
def test_asymptotic_rate_is_spectral_radius_of_cycle(dim, nx, ny, tile, k):
    """rho(M) < 1 and the observed residual ratio tends to rho(M) (P8)."""
    p = make_problem("R", dim, nx, ny)
    p["f"] = np.zeros_like(p["f"])     # homogeneous problem: x* = 0, no rounding floor
    p["bc"] = np.zeros_like(p["bc"])
    M, _, interior, idx = _brute.cycle_affine(dim, nx, ny, p["h"], p["f"], tile[0], tile[1], k)
    cols = [idx(i, j) for (i, j) in interior]
    rho = max(abs(np.linalg.eigvals(M[:, cols])))
    assert rho < 1
    r = run(p, mode="hier", tile=tile, k=k, tol=0.0, max_cycles=400)
    hist = r["history"]
    assert abs(hist[-1] / hist[-2] - rho) < 1e-6


# ---------------------------------------------------------------- P9 ----------
def test_classic_power_iteration_gives_cos_pi_h():
    """Power iteration with the oracle's sweep (f = 0, g = 0): rho(D^-1(A-D)) = cos(pi h) (P9)."""
    n = 16
    p = make_problem("R", 1, n)
    p["f"] = np.zeros(n)
    p["bc"] = np.zeros(2)
    r = run(p, mode="classic", tol=0.0, max_cycles=3000)
    hist = r["history"]
    assert abs(hist[-1] / hist[-2] - math.cos(math.pi / 17)) < 1e-9
    assert abs(hist[-1] / hist[-2] - 0.98297) < 1e-3   # SPEC.md:127 example


# ---------------------------------------------------------------- P11 ---------
def test_halo_freeze_locality_and_order_independence():
    """Perturbing a DOF outside tile t's halo leaves t's output bit-identical; tile order is irrelevant (P11)."""
    nx, ny, tx, ty, k = 40, 24, 8, 8, 5
    p = make_problem("R", 2, nx, ny)
    base = run(p, mode="hier", tile=(tx, ty), k=k, tol=0.0, max_cycles=1)["x"]
    rev = run(p, mode="hier", tile=(tx, ty), k=k, tol=0.0, max_cycles=1, tile_order=1)["x"]
    assert np.array_equal(base, rev)
    rng = np.random.default_rng(5)
    # tile (a, b) = (2, 1): interior x in [16, 24), y in [8, 16) (0-based interior indices)
    a, b = 2, 1
    x0, x1, y0, y1 = a * tx, (a + 1) * tx, b * ty, (b + 1) * ty
    for _ in range(30):
        i, j = int(rng.integers(nx)), int(rng.integers(ny))
        in_tile = x0 <= i < x1 and y0 <= j < y1
        in_edge_halo = ((x0 <= i < x1) and (j == y0 - 1 or j == y1)) or ((y0 <= j < y1) and (i == x0 - 1 or i == x1))
        q = dict(p)
        q["x0"] = p["x0"].copy()
        q["x0"][j * nx + i] += 0.5
        out = run(q, mode="hier", tile=(tx, ty), k=k, tol=0.0, max_cycles=1)["x"]
        same = np.array_equal(out[y0:y1, x0:x1], base[y0:y1, x0:x1])
        if in_tile or in_edge_halo:
            assert not same
        else:
            assert same


# ---------------------------------------------------------------- P13 ---------
@pytest.mark.parametrize("case", [c for c in COUNTS["cases"]], ids=lambda c: f"{c['dim']}d-n{c['n']}-k{c['k']}-{c['protocol']}-{c['tol']}")
def test_cross_implementation_counts(case):
    """Cycle counts agree exactly with an independent implementation."""
    if case.get("slow") and os.environ.get("HJ_SLOW") != "1":
        pytest.skip("slow oracle run; set HJ_SLOW=1")
    p = make_problem(case["protocol"], case["dim"], case["n"])
    r = run(p, mode="hier", tile=(case["tile"], case["tile"]), k=case["k"], tol=case["tol"],
            max_cycles=10**7, history=False)
    assert r["cycles"] == case["hier"]
    if case["classic"] is not None and case["k"] != 1:
        c = run(p, mode="classic", tol=case["tol"], max_cycles=10**7, history=False)
        assert c["cycles"] == case["classic"]


@pytest.mark.slow
def test_paper_time_ratio_matches_count_ratio():
    """The paper's 1D and 2D classic runs move the same 2^20 DOFs on one bandwidth-bound GPU, so
    t_1D / t_2D must equal the sweep-count ratio (P12, to 0.1%)."""
    c1 = run(make_problem("P", 1, 1024), mode="classic", tol=1e-4, max_cycles=10**7, history=False)["cycles"]
    c2 = run(make_problem("P", 2, 1024), mode="classic", tol=1e-4, max_cycles=10**7, history=False)["cycles"]
    t1 = min(PAPER["classic_ms_1d_tpb"]["value"][1:])
    t2 = PAPER["classic_ms_2d_best"]["value"]
    assert abs((c1 / c2) / (t1 / t2) - 1) < 1e-3


# ------------------------------------------------------- trends / fp32 --------
def test_cycles_non_increasing_in_k():
    """SPEC.md:290 / Fig. 5 restated as cycle counts: more sub-iterations never need more cycles."""
    p = make_problem("P", 1, 256)
    counts = [run(p, mode="hier", tile=32, k=k, tol=1e-4, max_cycles=10**6, history=False)["cycles"]
              for k in (4, 8, 16, 32, 64, 128)]
    assert all(a >= b for a, b in zip(counts, counts[1:]))


def test_fp32_tracks_fp64():
    """fp32 iterates (reading c16) stay within fp32 rounding of the fp64 iterates over a few cycles."""
    p = make_problem("R", 2, 40, 40)
    a = run(p, mode="hier", tile=(8, 8), k=8, tol=0.0, max_cycles=5, dtype="f64")
    b = run(p, mode="hier", tile=(8, 8), k=8, tol=0.0, max_cycles=5, dtype="f32")
    assert np.allclose(a["x"], b["x"], rtol=0, atol=1e-5 * np.abs(a["x"]).max())
    assert not np.array_equal(a["x"], b["x"])


def test_driver_edge_cases():
    """c = 0 when x0 is exact; max_cycles = 0; NOT_CONVERGED status; resume with ref_residual."""
    p = make_problem("P", 1, 20)
    xs = _brute.direct_solve(1, 20, 1, p["h"], p["f"], p["bc"])
    q = dict(p)
    q["x0"] = np.zeros(20)
    r = run(q, mode="hier", tile=4, k=2, tol=1e-3, max_cycles=0)
    assert r["cycles"] == 0 and not r["converged"] and r["status"] == 1
    r = run(p, mode="hier", tile=4, k=2, tol=1e-30, max_cycles=5)
    assert r["cycles"] == 5 and r["status"] == 1 and len(r["history"]) == 6
    # resume: 40 cycles, then 40 more with ref_residual = r_0, equals 80 straight
    full = run(p, mode="hier", tile=4, k=2, tol=1e-6, max_cycles=10**6)
    half = run(p, mode="hier", tile=4, k=2, tol=0.0, max_cycles=40)
    q = dict(p)
    q["x0"] = half["x"]
    rest = run(q, mode="hier", tile=4, k=2, tol=1e-6, max_cycles=10**6, ref_residual=half["history"][0])
    assert rest["cycles"] + 40 == full["cycles"]
    assert np.array_equal(rest["x"], full["x"])
    # exact x0: relative test with ref_residual satisfied at c = 0
    q["x0"] = xs
    r = run(q, mode="hier", tile=4, k=2, tol=1e-6, max_cycles=10, ref_residual=1.0)
    assert r["cycles"] == 0 and r["converged"]


# ---------------------------------------------------------- batched 1D (NEXT #2) --
def test_batched_1d_rows_are_independent_problems():
    """ny independent 1D problems: every row equals the single-problem oracle run on
    that row's data; identical copies converge in the single problem's cycle count."""
    B, n = 5, 45
    p = make_problem("R", 1, n, batch=B)
    r = oracle.solve(1, n, B, p["h"], p["f"], p["bc"], p["x0"], mode="hier", tile=8, k=5, tol=0.0, max_cycles=7)
    for b in range(B):
        one = oracle.solve(1, n, 1, p["h"], p["f"][b * n:(b + 1) * n], p["bc"][2 * b:2 * b + 2],
                           p["x0"][b * n:(b + 1) * n], mode="hier", tile=8, k=5, tol=0.0, max_cycles=7)
        assert np.array_equal(r["x"][b], one["x"])
    q = make_problem("P", 1, 1024, batch=4)
    single = make_problem("P", 1, 1024)
    for mode, k in (("hier", 16), ("classic", 1)):
        a = oracle.solve(1, 1024, 4, q["h"], q["f"], q["bc"], q["x0"], mode=mode, tile=32, k=k, tol=1e-4,
                         max_cycles=10**6, history=False)
        s = oracle.solve(1, 1024, 1, single["h"], single["f"], single["bc"], single["x0"], mode=mode, tile=32,
                         k=k, tol=1e-4, max_cycles=10**6, history=False)
        assert a["cycles"] == s["cycles"]
    assert oracle.resource_figures(1, 1024, 1024, 32)[0] == 1024 * 32   # PAPER.md:215 block count


@pytest.mark.parametrize("dim,nx,ny,tile,k", [(2, 48, 40, (16, 16), 3), (1, 200, 1, (32, 1), 5)])
def test_fp32_residual_is_that_of_the_rounded_system(dim, nx, ny, tile, k):
    """Reading c16 pinned: the fp32 history[c] is ||b32 - A x_c||_2 where x_c is
    the fp32 iterate, A the textbook Poisson matrix (assembled here with scipy, h^2-scaled) and b32 the
    right-hand side the fp32 iteration solves — float(h^2 f) and the ring float(g) — evaluated as a
    sparse matrix-vector product and an exactly rounded sum (math.fsum), to 1e-12.  The true-rhs reading
    (||f - A x_c|| with h^2 f and g in double) differs by far more than that, so the pin tells them apart."""
    p = make_problem("R", dim, nx, ny)
    h = p["h"]
    A = _brute.poisson_matrix(dim, nx, ny)

    def rhs(f, bc):
        r = f.copy()
        if dim == 1:
            r[0] += bc[0]
            r[-1] += bc[1]
        else:
            r = r.reshape(ny, nx)
            r[0, :] += bc[:nx]
            r[-1, :] += bc[nx:2 * nx]
            r[:, 0] += bc[2 * nx:2 * nx + ny]
            r[:, -1] += bc[2 * nx + ny:]
            r = r.reshape(-1)
        return r

    r32 = lambda a: np.asarray(a, dtype=np.float64).astype(np.float32).astype(np.float64)
    b32 = rhs(r32((h * h) * p["f"]), r32(p["bc"]))        # the system the fp32 iteration solves
    b64 = rhs((h * h) * p["f"], p["bc"])                  # the true system
    norm = lambda v: math.sqrt(math.fsum((v * v).tolist())) / (h * h)
    for c in (0, 1, 2, 5):
        r = run(p, mode="hier", dtype="f32", tile=tile, k=k, tol=0.0, max_cycles=c)
        x = r["x"].reshape(-1)
        assert np.array_equal(x, r32(x))                  # the iterate is an fp32 vector
        want = norm(b32 - A @ x)
        assert abs(r["history"][c] - want) <= 1e-12 * want, (c, r["history"][c], want)
        other = norm(b64 - A @ x)
        assert abs(other - want) > 10e-12 * want           # the pin discriminates the two readings (> 10x its bar)
