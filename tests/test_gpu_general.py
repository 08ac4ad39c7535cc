"""GPU parity of the general-coefficient path (reading c23):
Eq. 10's constant pentadiagonal stencil (2D) and Eq. 4's per-point tridiagonal stencil (1D)
through the C-ABI against the oracle (tests/test_oracle_general.py pins the oracle).

Bar: iterates bitwise equal after a fixed number of cycles (both sides evaluate the
same FMA chain on the same T-rounded weights and q = T(b/d)); history within 1e-12 relative;
cycle counts to tolerance exactly equal.
"""
import numpy as np
import pytest

import oracle
from paper_2006_16465_b200 import hj
from paper_2006_16465_b200.inputs import make_general

pytestmark = pytest.mark.gpu


def both(p, *, cycles, tol=0.0, **prm):
    o = oracle.solve(p["dim"], p["nx"], p["ny"], 1.0, p["f"], p["bc"], p["x0"], tol=tol,
                     max_cycles=cycles, stencil=p["stencil"],
                     **{k: v for k, v in prm.items() if k != "kernel"})
    g = hj.jacobi_solve(p["dim"], p["nx"], p["ny"], 1.0, p["f"], p["bc"], p["x0"], tol=tol,
                        max_cycles=cycles, stencil=p["stencil"], **prm)
    return o, g


def assert_parity(o, g, hist_rtol=1e-12):
    assert g["cycles"] == o["cycles"]
    bad = np.argwhere(np.asarray(g["x"]) != np.asarray(o["x"]))
    assert bad.size == 0, f"{len(bad)} mismatching cells, first {bad[:5].tolist()}"
    np.testing.assert_allclose(g["history"], o["history"], rtol=hist_rtol, atol=0)


CASES_2D = [
    # (nx, ny, tile, k, overlap, kernel): register kernel (32x32, aligned overlap), ragged edge
    # tiles (smem edge mode), the paper's smem kernel, misaligned overlap
    (64, 64, (32, 32), 16, 0, "auto"),
    (100, 70, (32, 32), 5, 0, "auto"),
    (130, 96, (32, 16), 6, 0, "auto"),
    (33, 40, (32, 32), 3, 0, "smem"),
    (96, 96, (32, 32), 8, 8, "auto"),
    (90, 70, (32, 32), 4, (6, 2), "auto"),
    (19, 13, (4, 5), 7, 2, "auto"),
]


@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("recipe", ["G", "A"])
@pytest.mark.parametrize("nx,ny,tile,k,ovl,kernel", CASES_2D)
def test_general2d_bitwise(nx, ny, tile, k, ovl, kernel, recipe, dtype):
    p = make_general(recipe, 2, nx, ny)
    o, g = both(p, cycles=3, mode="hier", tile=tile, k=k, overlap=ovl, kernel=kernel, dtype=dtype)
    assert_parity(o, g)


@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("nx,ny", [(300, 37), (7, 3), (513, 33)])
def test_general2d_classic_bitwise(nx, ny, dtype):
    p = make_general("G", 2, nx, ny)
    o, g = both(p, cycles=9, mode="classic", dtype=dtype)
    assert_parity(o, g)


CASES_1D = [
    # (nx, batch, tile, k, overlap, kernel)
    (256, 1, 32, 16, 0, "auto"),       # register kernel
    (1000, 3, 64, 5, 0, "auto"),       # ragged last tile
    (5000, 2, 256, 7, 0, "auto"),      # the largest register tile with coefficients
    (5000, 2, 512, 7, 0, "auto"),      # -> shared-memory kernel (x, q, wL, wR exceed registers)
    (1000, 4, 96, 5, 4, "auto"),       # overlap
    (1000, 2, 64, 3, 0, "smem"),
]


@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("recipe", ["G", "V"])
@pytest.mark.parametrize("nx,batch,tile,k,ovl,kernel", CASES_1D)
def test_general1d_bitwise(nx, batch, tile, k, ovl, kernel, recipe, dtype):
    p = make_general(recipe, 1, nx, batch=batch)
    o, g = both(p, cycles=4, mode="hier", tile=(tile, 1), k=k, overlap=ovl, kernel=kernel, dtype=dtype)
    assert_parity(o, g)


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_general1d_classic_bitwise(dtype):
    p = make_general("G", 1, 5000, batch=3)
    o, g = both(p, cycles=7, mode="classic", dtype=dtype)
    assert_parity(o, g)


@pytest.mark.parametrize("case", ["2d_aniso", "2d_random_ovl", "1d_var"])
def test_general_counts_to_tolerance(case):
    if case == "2d_aniso":       # the paper's protocol on a 128 x 96 anisotropic grid
        p, prm = make_general("A", 2, 128, 96), dict(tile=(32, 32), k=16)
    elif case == "2d_random_ovl":
        p, prm = make_general("G", 2, 96, 64), dict(tile=(32, 32), k=8, overlap=4)
    else:
        p, prm = make_general("V", 1, 256, batch=4), dict(tile=(32, 1), k=16)
    o, g = both(p, cycles=10**6, tol=1e-6, mode="hier", **prm)
    assert o["converged"] and g["converged"]
    assert_parity(o, g)


def test_general_device_api_and_plan():
    import torch
    p = make_general("G", 2, 100, 70)
    dev = torch.device("cuda:0")
    t = {k: torch.as_tensor(p[k], device=dev) for k in ("f", "bc", "x0", "stencil")}
    o = oracle.solve(2, 100, 70, 1.0, p["f"], p["bc"], p["x0"], tile=(32, 32), k=5, tol=0.0,
                     max_cycles=4, stencil=p["stencil"])
    g = hj.jacobi_solve_device(2, 100, 70, 1.0, t["f"], t["bc"], t["x0"], tile=(32, 32), k=5, tol=0.0,
                               max_cycles=4, stencil=t["stencil"])
    assert np.array_equal(g["x"].cpu().numpy(), o["x"])
    pl = hj.Plan(2, 100, 70, 1.0, t["f"], t["bc"], t["x0"], tile=(32, 32), k=5, tol=0.0, max_cycles=4,
                 stencil=p["stencil"])   # host stencil through the plan API
    r = pl.solve()
    pl.close()
    assert np.array_equal(r["x"].cpu().numpy(), o["x"])


def test_general_invalid_stencil():
    p = make_general("G", 2, 64, 64)
    bad = p["stencil"].copy()
    bad[4] = 0.0
    with pytest.raises(hj.HJError, match="INVALID_ARG"):
        hj.jacobi_solve(2, 64, 64, 1.0, p["f"], None, None, tile=(32, 32), k=4, stencil=bad)
    q = make_general("G", 1, 300, batch=2)
    bad = q["stencil"].copy()
    bad[0] = np.inf
    with pytest.raises(hj.HJError, match="INVALID_ARG"):
        hj.jacobi_solve(1, 300, 2, 1.0, q["f"], None, None, tile=(32, 1), k=4, stencil=bad)


def test_general_full_size_sampled_tiles():
    """Bench-size launch (16384^2, 32x32, k=16, anisotropic coefficients, f64): after one cycle,
    sampled tiles equal the oracle on a 3x3-tile window (its ring holds x0: exact for the centre
    tile after one cycle), and the initial residual equals the oracle's full-grid definition."""
    import torch
    n = 16384
    dx = 1.0 / (n + 1)
    st = np.array([-1 / dx ** 2, -1 / dx ** 2, -0.5 / dx ** 2, -0.5 / dx ** 2, 3 / dx ** 2])  # anisotropic
    rng = np.random.default_rng(7)
    dev = torch.device("cuda:0")
    f = torch.rand(n * n, dtype=torch.float64, device=dev) * 2 - 1
    x0 = torch.rand(n * n, dtype=torch.float64, device=dev) * 2 - 1
    pl = hj.Plan(2, n, n, 1.0, f, None, x0, tile=(32, 32), k=16, tol=0.0, max_cycles=1, stencil=st)
    r = pl.solve()
    pl.close()
    x1 = r["x"]
    fh, xh = f.view(n, n), x0.view(n, n)
    for _ in range(3):
        ty, tx = rng.integers(1, n // 32 - 1, size=2)
        ys, xs = slice(32 * (ty - 1), 32 * (ty + 2)), slice(32 * (tx - 1), 32 * (tx + 2))
        wf, wx = fh[ys, xs].cpu().numpy().copy(), xh[ys, xs].cpu().numpy().copy()
        ring = np.concatenate([xh[32 * (ty - 1) - 1, xs].cpu().numpy(), xh[32 * (ty + 2), xs].cpu().numpy(),
                               xh[ys, 32 * (tx - 1) - 1].cpu().numpy(), xh[ys, 32 * (tx + 2)].cpu().numpy()])
        o = oracle.solve(2, 96, 96, 1.0, wf.reshape(-1), ring, wx.reshape(-1), tile=(32, 32), k=16,
                         tol=0.0, max_cycles=1, stencil=st)
        got = x1[32 * ty:32 * ty + 32, 32 * tx:32 * tx + 32].cpu().numpy()
        assert np.array_equal(got, o["x"][32:64, 32:64])
    want0 = oracle.residual_general(2, n, n, f.cpu().numpy(), None, x0.cpu().numpy(), st)
    assert r["history"][0].item() == pytest.approx(want0, rel=1e-10)
