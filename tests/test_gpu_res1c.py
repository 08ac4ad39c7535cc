"""res1c_kernel (one small 1D problem in one CTA: C points per lane, ghost depth D, one __syncthreads
per cycle; kernels_1d.cu) against the oracle for every compiled layout: bitwise iterates, exact cycle
counts, histories within the 1e-12 bar (its residual sum is a warp tree + the warps in order).
PAPER.md:380-387 (§4.1) for the cycle; BASELINE config 1 (1D N = 256, 8 tiles of 32, k = 16, 1e-8)."""
import os

import numpy as np
import pytest

import oracle
from paper_2006_16465_b200 import hj
from paper_2006_16465_b200.inputs import make_problem

pytestmark = pytest.mark.gpu

LAYOUTS = [(1, 1), (1, 2), (1, 4), (2, 1), (2, 2), (2, 4), (4, 1), (4, 2), (4, 4), (8, 1), (8, 2), (8, 4)]
CASES = [
    ("M", 256, dict(tile=32, k=16, tol=1e-8, max_cycles=10**6)),                 # config 1, protocol M
    ("P", 256, dict(tile=32, k=16, tol=1e-8, max_cycles=10**6)),                 # config 1, protocol P
    ("R", 256, dict(tile=64, k=9, tol=0.0, max_cycles=7)),                       # odd k: singles, then groups
    ("R", 128, dict(tile=32, k=5, tol=0.0, max_cycles=6, dtype="f32")),          # f32: separate residual pass
    ("R", 512, dict(tile=128, k=6, tol=0.0, max_cycles=5)),
    ("R", 64, dict(tile=4, k=7, tol=0.0, max_cycles=6)),                         # tiles narrower than D ghosts
    ("R", 256, dict(tile=256, k=1, tol=0.0, max_cycles=4)),                      # k < D, one tile
    ("R", 256, dict(tile=32, k=4, tol=0.0, max_cycles=0)),                       # residual-only cycle
    ("R", 2048, dict(tile=256, k=6, tol=0.0, max_cycles=4)),                     # eight warps of C = 8
    ("P", 1024, dict(tile=32, k=16, tol=1e-6, max_cycles=10**6)),                # the paper's single N = 1024
]


def _applies(C, D, nx, tile):
    """engine.cu res1c_ok for a single 1D Poisson problem."""
    if nx % (32 * C) or nx // (32 * C) > 8 or tile % C or nx % tile:
        return False
    tpl = tile // C
    return tpl <= 32 and tpl & (tpl - 1) == 0


@pytest.mark.parametrize("C,D", LAYOUTS)
@pytest.mark.parametrize("proto,nx,kw", CASES)
def test_res1c_vs_oracle(C, D, proto, nx, kw):
    if not _applies(C, D, nx, kw["tile"]):
        pytest.skip("layout does not apply")
    p = make_problem(proto, 1, nx)
    old = os.environ.get("HJ_RES1C")
    os.environ["HJ_RES1C"] = f"{C},{D}"
    try:
        a = hj.jacobi_solve(1, nx, 1, p["h"], p["f"], p["bc"], p["x0"], mode="hier", **kw)
    finally:
        if old is None:
            os.environ.pop("HJ_RES1C", None)
        else:
            os.environ["HJ_RES1C"] = old
    o = oracle.solve(1, nx, 1, p["h"], p["f"], p["bc"], p["x0"], mode="hier", **kw)
    assert a["cycles"] == o["cycles"] and a["status"] == o["status"]
    assert np.array_equal(a["x"], o["x"])
    np.testing.assert_allclose(a["history"], o["history"], rtol=1e-12, atol=0)
