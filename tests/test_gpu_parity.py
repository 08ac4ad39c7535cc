"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle on the same seeded inputs.

Bar: iterates bitwise equal to the oracle after a fixed number of cycles (f64 and
f32 — both sides evaluate the same canonical expression); residual history within 1e-12
relative (different summation order); cycle counts to tolerance exactly equal.
"""
import os

import numpy as np
import pytest

import oracle
from paper_2006_16465_b200 import hj
from paper_2006_16465_b200.inputs import make_problem
from tests import _exact

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

pytestmark = pytest.mark.gpu


def both(p, *, cycles, **prm):
    o = oracle.solve(p["dim"], p["nx"], p["ny"], p["h"], p["f"], p["bc"], p["x0"], tol=0.0,
                     max_cycles=cycles, **{k: v for k, v in prm.items() if k != "kernel"})
    g = hj.jacobi_solve(p["dim"], p["nx"], p["ny"], p["h"], p["f"], p["bc"], p["x0"], tol=0.0,
                        max_cycles=cycles, **prm)
    return o, g


def assert_parity(o, g, hist_rtol=1e-12):
    assert g["cycles"] == o["cycles"]
    assert g["x"].shape == o["x"].shape
    bad = np.argwhere(g["x"] != o["x"])
    assert bad.size == 0, f"{len(bad)} mismatching cells, first {bad[:5].tolist()}"
    np.testing.assert_allclose(g["history"], o["history"], rtol=hist_rtol, atol=0)


CASES_2D = [
    # (nx, ny, tile, k, kernel)  — several tiles, ragged tails, both kernel families
    (64, 64, (32, 32), 16, "auto"),
    (100, 70, (32, 32), 5, "auto"),      # ragged in x and y
    (33, 40, (32, 32), 3, "auto"),
    (33, 40, (32, 32), 3, "smem"),
    (12, 12, (4, 4), 4, "auto"),          # the paper's 12x12 / 4x4 example
    (19, 13, (4, 5), 7, "auto"),
    (130, 96, (32, 16), 16, "auto"),
    (96, 64, (16, 8), 2, "smem"),
]


@pytest.mark.parametrize("proto", ["R", "P", "Q"])
@pytest.mark.parametrize("nx,ny,tile,k,kernel", CASES_2D)
@pytest.mark.parametrize("cycles", [1, 2, 3, 17])
def test_hier2d_bitwise(nx, ny, tile, k, kernel, cycles, proto):
    p = make_problem(proto, 2, nx, ny)
    o, g = both(p, cycles=cycles, mode="hier", tile=tile, k=k, kernel=kernel)
    assert_parity(o, g)


@pytest.mark.parametrize("dtype", ["f32"])
@pytest.mark.parametrize("nx,ny,tile,k,kernel", [(100, 70, (32, 32), 5, "auto"), (64, 64, (32, 32), 16, "auto"),
                                                 (33, 40, (32, 32), 3, "smem"), (19, 13, (4, 5), 7, "auto")])
def test_hier2d_f32_bitwise(nx, ny, tile, k, kernel, dtype):
    p = make_problem("R", 2, nx, ny)
    o, g = both(p, cycles=5, mode="hier", tile=tile, k=k, kernel=kernel, dtype=dtype)
    assert_parity(o, g)


@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("nx,ny", [(300, 37), (256, 16), (513, 33), (1, 1), (7, 3)])
def test_classic2d_bitwise(nx, ny, dtype):
    p = make_problem("R", 2, nx, ny)
    o, g = both(p, cycles=9, mode="classic", dtype=dtype)
    assert_parity(o, g)


CASES_1D = [
    (256, 32, 16, "auto"),      # config 1 shape (8 tiles of 32)
    (16384 + 37, 1024, 4, "auto"),
    (5000, 128, 7, "auto"),
    (1000, 96, 5, "auto"),      # not a power-of-two multiple of 32 -> shared-memory kernel
    (1000, 64, 3, "smem"),
    (12, 4, 2, "auto"),         # the paper's 12-point / 4-point example
]


@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("n,tile,k,kernel", CASES_1D)
@pytest.mark.parametrize("cycles", [1, 4, 17])
def test_hier1d_bitwise(n, tile, k, kernel, cycles, dtype):
    p = make_problem("R", 1, n)
    o, g = both(p, cycles=cycles, mode="hier", tile=tile, k=k, kernel=kernel, dtype=dtype)
    assert_parity(o, g)


@pytest.mark.parametrize("n", [1, 5, 2048, 5000, 2**16 + 3])
def test_classic1d_bitwise(n):
    p = make_problem("R", 1, n)
    o, g = both(p, cycles=6, mode="classic")
    assert_parity(o, g)


def test_k1_equals_classic_on_gpu():
    """PAPER.md:177 on the device: hierarchical k=1 iterates == classic iterates, bitwise."""
    p = make_problem("R", 2, 100, 70)
    a = hj.jacobi_solve(2, 100, 70, p["h"], p["f"], p["bc"], p["x0"], mode="hier", tile=(32, 32), k=1,
                        tol=0.0, max_cycles=11)
    b = hj.jacobi_solve(2, 100, 70, p["h"], p["f"], p["bc"], p["x0"], mode="classic", tol=0.0, max_cycles=11)
    assert np.array_equal(a["x"], b["x"])


# ------------------------------------------------------------ cycle counts ---------
@pytest.mark.parametrize("dim,n,tile,k,proto,tol,mode", [
    (1, 256, 32, 16, "M", 1e-8, "hier"), (1, 256, 32, 16, "P", 1e-8, "hier"),
    (1, 256, 32, 1, "M", 1e-8, "classic"), (1, 256, 32, 1, "P", 1e-8, "classic"),
    (2, 128, 32, 16, "P", 1e-6, "hier"), (2, 128, 32, 1, "P", 1e-6, "classic"),
    (2, 64, 16, 5, "R", 1e-7, "hier"), (1, 1000, 96, 9, "R", 1e-6, "hier"),
])
def test_cycle_counts_match_oracle(dim, n, tile, k, proto, tol, mode):
    """Cycle counts to tolerance are exactly the oracle's (config 1 = BASELINE configs[0])."""
    p = make_problem(proto, dim, n)
    tl = (tile, tile) if dim == 2 else tile
    o = oracle.solve(dim, p["nx"], p["ny"], p["h"], p["f"], p["bc"], p["x0"], mode=mode, tile=tl, k=k,
                     tol=tol, max_cycles=10**7)
    g = hj.jacobi_solve(dim, p["nx"], p["ny"], p["h"], p["f"], p["bc"], p["x0"], mode=mode, tile=tl,
                        k=k if mode == "hier" else 1, tol=tol, max_cycles=10**7 if dim == 1 else 10**6)
    assert o["converged"] and g["converged"]
    assert g["cycles"] == o["cycles"]
    assert np.array_equal(g["x"], o["x"])
    np.testing.assert_allclose(g["history"], o["history"], rtol=1e-12, atol=0)


def test_config3_count_1024sq():
    """Config 3 (2D 1024^2, 32x32, k=16, paper protocol, 1e-4): 20,153 cycles — the count of
    the independent implementation (tests/golden/cross_impl_counts.json), which the oracle
    reproduces (tests/test_oracle_pins.py, HJ_SLOW)."""
    p = make_problem("P", 2, 1024)
    g = hj.jacobi_solve(2, 1024, 1024, p["h"], p["f"], p["bc"], p["x0"], mode="hier", tile=(32, 32), k=16,
                        tol=1e-4, max_cycles=100000)
    assert g["converged"] and g["cycles"] == 20153


# ------------------------------------------------------------ driver semantics -----
def test_driver_edge_cases_match_oracle():
    p = make_problem("P", 2, 40, 40)
    kw = dict(mode="hier", tile=(32, 32), k=4)
    for extra in [dict(tol=1e-3, max_cycles=0), dict(tol=1e-30, max_cycles=5),
                  dict(tol=1e-3, tol_mode="abs", max_cycles=10**5),
                  dict(tol=1e-6, max_cycles=10**5, ref_residual=123.0)]:
        o = oracle.solve(2, 40, 40, p["h"], p["f"], p["bc"], p["x0"], **kw, **extra)
        g = hj.jacobi_solve(2, 40, 40, p["h"], p["f"], p["bc"], p["x0"], **kw, **extra)
        assert (g["cycles"], g["converged"], g["status"]) == (o["cycles"], o["converged"], o["status"])
        assert np.array_equal(g["x"], o["x"])


def test_exact_initial_guess_converges_at_zero_cycles():
    p = make_problem("P", 1, 64)
    p["f"] = np.zeros(64)
    p["x0"] = np.zeros(64)
    g = hj.jacobi_solve(1, 64, 1, p["h"], p["f"], p["bc"], p["x0"], mode="hier", tile=32, k=4, tol=1e-6)
    assert g["cycles"] == 0 and g["converged"]


def test_numeric_error_detected():
    p = make_problem("R", 2, 64, 64)
    p["f"][100] = np.inf
    g = hj.jacobi_solve(2, 64, 64, p["h"], p["f"], p["bc"], p["x0"], mode="hier", tile=(32, 32), k=4,
                        tol=1e-6, max_cycles=50)
    assert g["status"] == hj.HJ_ERR_NUMERIC


def test_determinism_repeated_runs():
    p = make_problem("R", 2, 200, 150)
    runs = [hj.jacobi_solve(2, 200, 150, p["h"], p["f"], p["bc"], p["x0"], mode="hier", tile=(32, 32), k=9,
                            tol=0.0, max_cycles=20) for _ in range(3)]
    for r in runs[1:]:
        assert np.array_equal(r["x"], runs[0]["x"])
        assert np.array_equal(r["history"], runs[0]["history"])


def test_device_api_and_plan_resume():
    """jacobi_solve_device (torch device buffers) and hj_plan_* reproduce the host API."""
    import torch
    p = make_problem("R", 2, 96, 64)
    ref = hj.jacobi_solve(2, 96, 64, p["h"], p["f"], p["bc"], p["x0"], mode="hier", tile=(32, 32), k=6,
                          tol=1e-6, max_cycles=10**5)
    dev = torch.device("cuda:0")
    t = {k: torch.from_numpy(p[k]).to(dev) for k in ("f", "bc", "x0")}
    d = hj.jacobi_solve_device(2, 96, 64, p["h"], t["f"], t["bc"], t["x0"], mode="hier", tile=(32, 32), k=6,
                               tol=1e-6, max_cycles=10**5)
    assert d["cycles"] == ref["cycles"]
    assert np.array_equal(d["x"].cpu().numpy(), ref["x"])
    plan = hj.Plan(2, 96, 64, p["h"], t["f"], t["bc"], t["x0"], mode="hier", tile=(32, 32), k=6,
                   tol=1e-6, max_cycles=10**5)
    plan.run(10)                     # 10 cycles, then solve continues from x_10
    r = plan.solve()
    assert r["cycles"] == ref["cycles"]
    assert np.array_equal(r["x"].cpu().numpy(), ref["x"])
    plan.reset()
    assert plan.solve()["cycles"] == ref["cycles"]
    plan.close()


# ------------------------------------------------------------ full size ------------
def _window_oracle(p, tx0, ty0, ntile, cycles, dtype="f64", T=32):
    """Oracle on a tile-aligned window of (2*cycles-1) tiles around tile (tx0, ty0): the window
    ring holds x0 (or the true Dirichlet ring); after `cycles` cycles the centre tile is exact."""
    nx, ny = p["nx"], p["ny"]
    r = cycles - 1
    a0, a1 = max(tx0 - r, 0), min(tx0 + r, ntile - 1)
    b0, b1 = max(ty0 - r, 0), min(ty0 + r, ntile - 1)
    i0, i1 = a0 * T, min((a1 + 1) * T, nx)
    j0, j1 = b0 * T, min((b1 + 1) * T, ny)
    x0 = p["x0"].reshape(ny, nx)
    f = p["f"].reshape(ny, nx)
    bc = p["bc"]
    sub = np.zeros((j1 - j0 + 2, i1 - i0 + 2))
    sub[1:-1, 1:-1] = x0[j0:j1, i0:i1]

    def ringval(jj, ii):  # padded global coordinates
        if jj == 0:
            return bc[ii - 1] if 1 <= ii <= nx else 0.0
        if jj == ny + 1:
            return bc[nx + ii - 1] if 1 <= ii <= nx else 0.0
        if ii == 0:
            return bc[2 * nx + jj - 1]
        if ii == nx + 1:
            return bc[2 * nx + ny + jj - 1]
        return x0[jj - 1, ii - 1]

    w, hgt = i1 - i0, j1 - j0
    south = np.array([ringval(j0, i0 + 1 + q) for q in range(w)])
    north = np.array([ringval(j1 + 1, i0 + 1 + q) for q in range(w)])
    west = np.array([ringval(j0 + 1 + q, i0) for q in range(hgt)])
    east = np.array([ringval(j0 + 1 + q, i1 + 1) for q in range(hgt)])
    o = oracle.solve(2, w, hgt, p["h"], f[j0:j1, i0:i1], np.concatenate([south, north, west, east]),
                     x0[j0:j1, i0:i1], mode="hier", tile=(T, T), k=16, tol=0.0, max_cycles=cycles,
                     dtype=dtype)
    cx, cy = (tx0 - a0) * T, (ty0 - b0) * T
    return o["x"][cy:cy + T, cx:cx + T]


@pytest.mark.parametrize("n,proto,dtype", [(16384, "R", "f64"), (16384, "P", "f64"), (16384, "R", "f32"),
                                           (32768, "P", "f64")])
def test_full_size_sampled_tiles(n, proto, dtype):
    """BASELINE config 4 (16384^2, the bench's launch configuration: 32x32 register kernel, k=16) and
    config 5's 32768^2: sampled tiles after 1 and 2 cycles equal the oracle's (computed on tile
    windows), and the initial residual equals the oracle's full-grid residual."""
    import torch
    p = make_problem(proto, 2, n)
    dev = torch.device("cuda:0")
    t = {k: torch.from_numpy(p[k]).to(dev) for k in ("f", "bc", "x0")}
    rng = np.random.default_rng(11)
    nt = n // 32
    samples = [(0, 0), (nt - 1, nt - 1), (0, nt - 1), (nt - 1, 0)] + \
              [tuple(int(v) for v in rng.integers(0, nt, 2)) for _ in range(4)]
    for cycles in (1, 2):
        d = hj.jacobi_solve_device(2, n, n, p["h"], t["f"], t["bc"], t["x0"], mode="hier", tile=(32, 32),
                                   k=16, tol=0.0, max_cycles=cycles, dtype=dtype)
        xg = d["x"].cpu().numpy()
        for (a, b) in samples:
            ref = _window_oracle(p, a, b, nt, cycles, dtype)
            got = xg[b * 32:(b + 1) * 32, a * 32:(a + 1) * 32]
            assert np.array_equal(got, ref), (cycles, a, b)
        if cycles == 1 and dtype == "f64":
            r0 = oracle.residual(2, n, n, p["h"], p["f"], p["bc"], p["x0"])
            np.testing.assert_allclose(d["history"][0].item(), r0, rtol=1e-12)
        del d, xg


def test_full_size_full_grid_one_cycle_bench_config():
    """The bench's exact launch configuration (16384^2, protocol P, 32x32 register kernel, k = 16):
    after one cycle EVERY cell equals the oracle's full-grid cycle (the oracle needs ~10 GB of host
    memory and ~15 s), and after two cycles too."""
    n = 16384
    p = make_problem("P", 2, n)
    xs = [p["x0"]]
    for cycles in (1, 2):
        o, g = both(p, cycles=cycles, mode="hier", tile=(32, 32), k=16)
        assert g["cycles"] == o["cycles"] == cycles
        assert np.array_equal(g["x"], o["x"])
        xs.append(g["x"])
        # residual history: the GPU's tile tree to 1e-12 of the exactly summed definition evaluated
        # on the (bit-identical) iterates x_0 .. x_c (tests/_exact.py) ...
        for c in range(cycles + 1):
            want = _exact.residual_2d(n, n, p["h"], p["f"], p["bc"], xs[c])
            assert abs(g["history"][c] - want) <= 1e-12 * want, (c, g["history"][c], want)
        # ... and the oracle's naive sequential sum within its recursive-summation bound (reading c15)
        np.testing.assert_allclose(g["history"], o["history"], rtol=n * n * np.finfo(np.float64).eps / 2, atol=0)
        del o, g
    # the classic comparison sweep at the same size
    o, g = both(p, cycles=2, mode="classic")
    assert np.array_equal(g["x"], o["x"])


def test_dist_path_single_rank_matches_single_gpu():
    """jacobi_solve_dist with one rank (1-rank NCCL communicator, rowpart_local + allreduce path,
    NCCL inside the graph-captured cycle) reproduces the single-GPU solve bit for bit."""
    p = make_problem("R", 2, 96, 64)
    ref = hj.jacobi_solve(2, 96, 64, p["h"], p["f"], p["bc"], p["x0"], mode="hier", tile=(32, 32), k=6,
                          tol=1e-7, max_cycles=10**5)
    nid = hj.hj_nccl_unique_id()
    d = hj.jacobi_solve_dist(96, 64, p["h"], p["f"], p["bc"], p["x0"], rank=0, nranks=1, nccl_id=nid,
                             row_begin=0, row_end=64, mode="hier", tile=(32, 32), k=6, tol=1e-7,
                             max_cycles=10**5)
    assert d["cycles"] == ref["cycles"]
    assert np.array_equal(d["x"], ref["x"])
    np.testing.assert_allclose(d["history"], ref["history"], rtol=1e-14, atol=0)
    # classic through the same path
    ref = hj.jacobi_solve(2, 96, 64, p["h"], p["f"], p["bc"], p["x0"], mode="classic", tol=0.0, max_cycles=9)
    d = hj.jacobi_solve_dist(96, 64, p["h"], p["f"], p["bc"], p["x0"], rank=0, nranks=1,
                             nccl_id=hj.hj_nccl_unique_id(), row_begin=0, row_end=64, mode="classic",
                             tol=0.0, max_cycles=9)
    assert np.array_equal(d["x"], ref["x"])


def test_dist_plan_single_rank_bench_path():
    """hj_plan_create_dist (the bench's N>1 entry point) with one rank."""
    import torch
    n = 128
    p = make_problem("P", 2, n)
    dev = torch.device("cuda:0")
    t = {k: torch.from_numpy(p[k]).to(dev) for k in ("f", "bc", "x0")}
    s = torch.cuda.Stream(dev)
    plan = hj.DistPlan(n, n, p["h"], t["f"], t["bc"], t["x0"], rank=0, nranks=1,
                       nccl_id=hj.hj_nccl_unique_id(), row_begin=0, row_end=n, stream=s.cuda_stream,
                       mode="hier", tile=(32, 32), k=16, tol=1e-6, max_cycles=10**5)
    ms = plan.run(6, timed=True)
    assert ms > 0
    plan.reset()
    r = plan.solve()
    assert r["converged"] and r["cycles"] == 2515     # cross_impl_counts.json (2D 128^2, 1e-6)
    plan.close()


# --------------------------------------------------- batched 1D (NEXT #2) ----------
@pytest.mark.parametrize("n,B,tile,k,ov,mode,kernel", [
    (1024, 7, 32, 16, 0, "hier", "auto"),      # register kernel, C = 1
    (5000, 3, 1024, 5, 0, "hier", "auto"),     # register kernel, ragged last tile
    (1000, 4, 96, 5, 0, "hier", "auto"),       # shared-memory kernel
    (1024, 5, 32, 16, 4, "hier", "auto"),      # overlapping subdomains
    (3000, 6, 1, 1, 0, "classic", "auto"),
])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_batched_1d_bitwise(n, B, tile, k, ov, mode, kernel, dtype):
    p = make_problem("R", 1, n, batch=B)
    kw = dict(mode=mode, tol=0.0, max_cycles=9, dtype=dtype)
    if mode == "hier":
        kw.update(tile=tile, k=k, overlap=ov)
    o = oracle.solve(1, n, B, p["h"], p["f"], p["bc"], p["x0"], **kw)
    g = hj.jacobi_solve(1, n, B, p["h"], p["f"], p["bc"], p["x0"], kernel=kernel, **kw)
    assert_parity(o, g)


@pytest.mark.parametrize("k,o,cycles", [(1, 0, 128760), (8, 0, 25481), (16, 0, 19555), (16, 4, 8093)])
def test_paper_1d_workload_counts(k, o, cycles):
    """The paper's 1D workload: 1024 copies of N = 1024, tpb 32, 1e-4: the counts of
    the independent implementation (tests/golden/cross_impl_counts*.json)."""
    p = make_problem("P", 1, 1024, batch=1024)
    kw = dict(mode="hier", tile=32, k=k, overlap=o) if k > 1 else dict(mode="classic")
    g = hj.jacobi_solve(1, 1024, 1024, p["h"], p["f"], p["bc"], p["x0"], tol=1e-4, max_cycles=10**6,
                        history=False, **kw)
    assert g["converged"] and g["cycles"] == cycles


def test_split_cycle_launch_order_bitwise():
    """The overlapped NCCL transport's launch order — the slab's boundary tile rows first, then the
    interior tile rows — forced on one GPU with HJ_SPLIT_CYCLE=1 (NCCL cannot run
    several ranks on one device): iterates bitwise and history 1e-12 against the oracle, the
    per-cycle path (HJ_RESIDENT=0) through plan graphs, several cycles."""
    import subprocess
    import sys
    import textwrap
    code = textwrap.dedent("""
        import numpy as np, oracle
        from paper_2006_16465_b200 import hj
        from paper_2006_16465_b200.inputs import make_problem
        for (nx, ny, k, c) in ((96, 96, 5, 7), (128, 160, 16, 4)):
            p = make_problem("R", 2, nx, ny)
            kw = dict(mode="hier", tile=(32, 32), k=k, tol=0.0, max_cycles=c)
            o = oracle.solve(2, nx, ny, p["h"], p["f"], p["bc"], p["x0"], **kw)
            g = hj.jacobi_solve(2, nx, ny, p["h"], p["f"], p["bc"], p["x0"], **kw)
            assert np.array_equal(g["x"], o["x"]), (nx, ny)
            np.testing.assert_allclose(g["history"], o["history"], rtol=1e-12, atol=0)
        p = make_problem("P", 2, 96, 96)
        kw = dict(mode="hier", tile=(32, 32), k=8, tol=1e-6, max_cycles=10**6, history=False)
        o = oracle.solve(2, 96, 96, p["h"], p["f"], p["bc"], p["x0"], **kw)
        g = hj.jacobi_solve(2, 96, 96, p["h"], p["f"], p["bc"], p["x0"], **kw)
        assert g["cycles"] == o["cycles"]
        print("ok")
    """)
    env = dict(os.environ, HJ_SPLIT_CYCLE="1", HJ_RESIDENT="0")
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout + r.stderr


REGT_CASES = [  # (nx, ny, tile): BASELINE config 5's tile sweep shapes on small grids (several tiles each way)
    (96, 64, (16, 16)), (64, 96, (32, 16)), (96, 64, (16, 32)), (192, 96, (64, 32)), (96, 192, (32, 64)),
    (128, 192, (64, 64)), (256, 96, (128, 32)),
]


@pytest.mark.parametrize("nx,ny,tile", REGT_CASES, ids=[f"{t[0]}x{t[1]}" for _, _, t in REGT_CASES])
@pytest.mark.parametrize("k", [1, 4, 7])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_regt_tile_shapes_bitwise(nx, ny, tile, k, dtype):
    """The register kernel for other tile shapes (kernels_2dt.cu; several tiles per warp, or a warp
    group per tile with a per-sub-iteration block-edge exchange) equals the oracle bit for bit, history
    1e-12, and the plan really runs it (hj_plan_kernel_kind)."""
    import torch
    p = make_problem("R", 2, nx, ny)
    kw = dict(mode="hier", tile=tile, k=k, dtype=dtype, tol=0.0, max_cycles=3)
    o = oracle.solve(2, nx, ny, p["h"], p["f"], p["bc"], p["x0"], **kw)
    dev = torch.device("cuda", 0)
    t = lambda a: torch.as_tensor(a, device=dev)
    plan = hj.Plan(2, nx, ny, p["h"], t(p["f"]), t(p["bc"]), t(p["x0"]), **kw)
    assert plan.kernel_kind() == "regt"
    r = plan.solve()
    plan.close()
    assert np.array_equal(r["x"].cpu().numpy(), o["x"])
    np.testing.assert_allclose(r["history"].cpu().numpy(), o["history"], rtol=1e-12, atol=0)


@pytest.mark.parametrize("tile", [(16, 16), (64, 64), (128, 32)])
def test_regt_counts_to_tolerance(tile):
    """Cycle counts to 1e-6 (paper protocol) with the REGT tile shapes equal the oracle's exactly."""
    n = 128 if tile[0] <= 64 else 256
    p = make_problem("P", 2, n, 128)
    kw = dict(mode="hier", tile=tile, k=16, tol=1e-6, max_cycles=10**6, history=False)
    o = oracle.solve(2, n, 128, p["h"], p["f"], p["bc"], p["x0"], **kw)
    g = hj.jacobi_solve(2, n, 128, p["h"], p["f"], p["bc"], p["x0"], **kw)
    assert o["converged"] and g["cycles"] == o["cycles"]
