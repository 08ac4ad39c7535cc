"""GPU parity with overlapping subdomains (§3.5 / §4.3): iterates bitwise equal to the
oracle, cycle counts exactly equal (including the independent Table-3/Table-4 counts)."""
import json
import os

import numpy as np
import pytest

import oracle
from paper_2006_16465_b200 import hj
from paper_2006_16465_b200.inputs import make_problem

pytestmark = pytest.mark.gpu
COUNTS = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "cross_impl_counts_overlap.json")))


@pytest.mark.parametrize("dim,nx,ny,tile,k,ov,kernel", [
    (2, 100, 70, (32, 32), 5, 4, "auto"),       # register kernel, shifted last blocks
    (2, 96, 64, (32, 32), 16, 2, "auto"),
    (2, 64, 64, (32, 32), 3, (6, 2), "auto"),
    (2, 99, 70, (32, 32), 4, 4, "auto"),       # odd nx: misaligned last block -> smem kernel
    (2, 128, 64, (32, 32), 6, 8, "auto"),      # fp32-aligned overlap -> register kernel
    # overlap on ONE axis: a ragged axis without overlap must not run as full tiles
    (2, 100, 70, (32, 32), 5, (0, 4), "auto"),  # ragged x, o_x = 0 -> smem kernel
    (2, 100, 70, (32, 32), 5, (4, 0), "auto"),  # ragged y, o_y = 0 -> smem kernel
    (2, 128, 70, (32, 32), 5, (0, 4), "auto"),  # x multiple of 32 -> register kernel
    (2, 100, 64, (32, 32), 5, (4, 0), "auto"),  # y multiple of 32 -> register kernel
    (2, 100, 70, (32, 32), 5, 4, "smem"),
    (2, 40, 30, (8, 8), 4, 2, "auto"),
    (2, 37, 29, (10, 6), 3, (4, 2), "auto"),
    (1, 1024, 1, 32, 16, 4, "auto"),
    (1, 1000, 1, 64, 7, 10, "auto"),
    (1, 37, 1, 8, 3, 2, "auto"),
])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_overlap_bitwise(dim, nx, ny, tile, k, ov, kernel, dtype):
    p = make_problem("R", dim, nx, ny)
    kw = dict(mode="hier", tile=tile, k=k, overlap=ov, tol=0.0, max_cycles=7, dtype=dtype)
    o = oracle.solve(dim, nx, ny, p["h"], p["f"], p["bc"], p["x0"], **kw)
    g = hj.jacobi_solve(dim, nx, ny, p["h"], p["f"], p["bc"], p["x0"], kernel=kernel, **kw)
    assert np.array_equal(g["x"], o["x"])
    np.testing.assert_allclose(g["history"], o["history"], rtol=1e-12, atol=0)


@pytest.mark.parametrize("case", COUNTS["cases"], ids=lambda c: f"{c['dim']}d-k{c['k']}-o{c['o']}")
def test_overlap_counts_on_gpu(case):
    """Cycle counts with overlap = the independent implementation's."""
    p = make_problem(case["protocol"], case["dim"], case["n"])
    tl = (case["tile"], case["tile"]) if case["dim"] == 2 else case["tile"]
    g = hj.jacobi_solve(case["dim"], p["nx"], p["ny"], p["h"], p["f"], p["bc"], p["x0"], mode="hier", tile=tl,
                        k=case["k"], overlap=case["o"], tol=case["tol"], max_cycles=10**6, history=False)
    assert g["converged"] and g["cycles"] == case["cycles"]


def test_overlap_rejected_with_row_slabs_and_bad_values():
    p = make_problem("P", 2, 64)
    for ov in (3, -2, 32):
        with pytest.raises(hj.HJError) as ei:
            hj.jacobi_solve(2, 64, 64, p["h"], p["f"], p["bc"], p["x0"], tile=(32, 32), k=4, overlap=ov, max_cycles=2)
        assert ei.value.status == hj.HJ_ERR_INVALID_CONFIG
