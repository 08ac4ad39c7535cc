"""Seeded random configurations, GPU (through the C-ABI) vs the oracle, bitwise iterates after a few
cycles: grid sizes (ragged and multiples of 32, so both the per-cycle and the resident paths run),
tile shapes, k, overlap, dtype, protocols, 1D batches, general coefficients and multigrid.  A
net for interactions the structured parity suites do not enumerate."""
import numpy as np
import pytest

import oracle
from paper_2006_16465_b200 import hj
from paper_2006_16465_b200.inputs import make_general, make_problem

pytestmark = pytest.mark.gpu

rng = np.random.default_rng(2006_16465)


def _cases():
    out = []
    for i in range(60):  # 2D hierarchical / classic
        nx = int(rng.choice([32, 64, 96, 128, int(rng.integers(20, 150))]))
        ny = int(rng.choice([32, 64, 96, int(rng.integers(20, 150))]))
        if rng.random() < 0.6:
            tx = ty = 32
        else:
            tx, ty = int(rng.integers(2, min(nx, 32) + 1)), int(rng.integers(2, min(ny, 32) + 1))
        tx, ty = min(tx, nx), min(ty, ny)
        k = int(rng.integers(1, 20))
        o = 0
        if rng.random() < 0.3 and min(tx, ty) > 4:
            o = int(2 * rng.integers(1, min(tx, ty) // 2))
            o = o if o < min(tx, ty) else 0
        mode = "classic" if rng.random() < 0.15 else "hier"
        out.append(dict(kind="2d", nx=nx, ny=ny, tile=(tx, ty), k=k if mode == "hier" else 1, overlap=o,
                        mode=mode, dtype=str(rng.choice(["f64", "f32"])), proto=str(rng.choice(["R", "P", "Q"])),
                        cycles=int(rng.integers(1, 6))))
    for i in range(25):  # 1D (batched)
        n = int(rng.choice([256, 512, 1024, int(rng.integers(40, 3000))]))
        b = int(rng.choice([1, 3, 17, 64]))
        t = int(rng.choice([32, 64, 128, 256, int(rng.integers(8, min(n, 200) + 1))]))
        t = min(t, n)
        out.append(dict(kind="1d", nx=n, ny=b, tile=t, k=int(rng.integers(1, 20)), overlap=0, mode="hier",
                        dtype=str(rng.choice(["f64", "f32"])), proto="R", cycles=int(rng.integers(1, 5))))
    for i in range(14):  # multigrid
        nx = int(rng.choice([31, 63, 127, 255, 95, 191]))
        ny = int(rng.choice([31, 63, 127, 95]))
        out.append(dict(kind="mg", nx=nx, ny=ny, tile=(32, 32) if rng.random() < 0.7 else (8, 16),
                        k=int(rng.integers(1, 6)), nu1=int(rng.integers(0, 3)), nu2=int(rng.integers(1, 3)),
                        omega=float(rng.choice([0.6, 0.7, 0.8])), dtype=str(rng.choice(["f64", "f32"])),
                        proto=str(rng.choice(["R", "P"])), cycles=int(rng.integers(1, 4))))
    for i in range(8):  # general coefficients
        nx, ny = int(rng.choice([64, 96, 70])), int(rng.choice([64, 33, 50]))
        out.append(dict(kind="gen", nx=nx, ny=ny, tile=(32, 32) if nx >= 32 and ny >= 32 else (16, 16),
                        k=int(rng.integers(1, 12)), dtype=str(rng.choice(["f64", "f32"])),
                        cycles=int(rng.integers(1, 5))))
    return out


CASES = _cases()


@pytest.mark.parametrize("c", CASES, ids=[f"{c['kind']}-{i}" for i, c in enumerate(CASES)])
def test_fuzz_bitwise(c):
    if c["kind"] == "mg":
        p = make_problem(c["proto"], 2, c["nx"], c["ny"])
        kw = dict(tile=c["tile"], k=c["k"], nu1=c["nu1"], nu2=c["nu2"], omega=c["omega"], dtype=c["dtype"],
                  tol=0.0, max_cycles=c["cycles"])
        o = oracle.solve_mg(2, c["nx"], c["ny"], p["h"], p["f"], p["bc"], p["x0"], **kw)
        g = hj.jacobi_solve(2, c["nx"], c["ny"], p["h"], p["f"], p["bc"], p["x0"], mode="mg", **kw)
    elif c["kind"] == "gen":
        p = make_general("G", 2, c["nx"], c["ny"])
        kw = dict(mode="hier", tile=c["tile"], k=c["k"], dtype=c["dtype"], tol=0.0, max_cycles=c["cycles"])
        o = oracle.solve(2, c["nx"], c["ny"], p["h"], p["f"], p["bc"], p["x0"], stencil=p["stencil"], **kw)
        g = hj.jacobi_solve(2, c["nx"], c["ny"], p["h"], p["f"], p["bc"], p["x0"], stencil=p["stencil"], **kw)
    else:
        dim = 2 if c["kind"] == "2d" else 1
        p = make_problem(c["proto"], 2, c["nx"], c["ny"]) if dim == 2 else make_problem("R", 1, c["nx"], batch=c["ny"])
        kw = dict(mode=c["mode"], dtype=c["dtype"], tol=0.0, max_cycles=c["cycles"])
        if c["mode"] == "hier":
            kw.update(tile=c["tile"], k=c["k"], overlap=c["overlap"])
        o = oracle.solve(dim, p["nx"], p["ny"], p["h"], p["f"], p["bc"], p["x0"], **kw)
        g = hj.jacobi_solve(dim, p["nx"], p["ny"], p["h"], p["f"], p["bc"], p["x0"], **kw)
    assert g["cycles"] == o["cycles"]
    bad = np.argwhere(g["x"] != o["x"])
    assert bad.size == 0, f"{len(bad)} mismatching cells, first {bad[:5].tolist()} ({c})"
    np.testing.assert_allclose(g["history"], o["history"], rtol=1e-12, atol=0)
