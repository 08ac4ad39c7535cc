"""CPU pins of the test-side full-size residual reference (tests/_exact.py): it must equal the
residual's definition as a sparse matrix-vector product with an exactly rounded sum (math.fsum), on
small grids, f64 and f32 (reading c16), several chunk sizes (so the chunk seams are exercised), and
the oracle's full-grid history on a fixed number of cycles."""
import math

import numpy as np
import pytest

import oracle
from paper_2006_16465_b200.inputs import make_problem
from tests import _brute, _exact


def _matrix_norm(nx, ny, h, f, bc, x, dtype):
    r32 = (lambda a: np.asarray(a, dtype=np.float64).astype(np.float32).astype(np.float64)) if dtype == "f32" \
        else (lambda a: np.asarray(a, dtype=np.float64))
    A = _brute.poisson_matrix(2, nx, ny)
    b = r32((h * h) * f).reshape(ny, nx).copy()
    g = r32(bc)
    b[0, :] += g[:nx]
    b[-1, :] += g[nx:2 * nx]
    b[:, 0] += g[2 * nx:2 * nx + ny]
    b[:, -1] += g[2 * nx + ny:]
    r = b.reshape(-1) - A @ np.asarray(x, dtype=np.float64).reshape(-1)
    return math.sqrt(math.fsum((r * r).tolist())) / (h * h)


@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("chunk", [1, 7, 1024])
def test_exact_residual_equals_matrix_definition(dtype, chunk):
    nx, ny = 45, 37
    p = make_problem("R", 2, nx, ny)
    for c in (0, 1, 3):
        o = oracle.solve(2, nx, ny, p["h"], p["f"], p["bc"], p["x0"], tile=(16, 16), k=4, tol=0.0, max_cycles=c,
                         dtype=dtype)
        got = _exact.residual_2d(nx, ny, p["h"], p["f"], p["bc"], o["x"], dtype=dtype, chunk=chunk)
        want = _matrix_norm(nx, ny, p["h"], p["f"], p["bc"], o["x"], dtype)
        assert abs(got - want) <= 1e-13 * want
        np.testing.assert_allclose(o["history"][c], want, rtol=1e-12)


def test_exact_residual_protocol_p():
    n = 200
    p = make_problem("P", 2, n)
    o = oracle.solve(2, n, n, p["h"], p["f"], p["bc"], p["x0"], tile=(32, 32), k=16, tol=0.0, max_cycles=2)
    got = _exact.residual_2d(n, n, p["h"], p["f"], p["bc"], o["x"], chunk=33)
    want = _matrix_norm(n, n, p["h"], p["f"], p["bc"], o["x"], "f64")
    assert abs(got - want) <= 1e-13 * want
