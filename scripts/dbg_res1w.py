import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2006_16465_b200 import hj
from paper_2006_16465_b200.inputs import make_problem
import oracle
for (n, t, k, cyc, dt) in [(256, 32, 16, 3, "f64"), (512, 64, 7, 4, "f64"), (1024, 32, 5, 3, "f64"), (512, 128, 3, 3, "f32")]:
    p = make_problem("R", 1, n)
    kw = dict(mode="hier", tile=t, k=k, tol=0.0, max_cycles=cyc, dtype=dt)
    print("case", n, t, k, cyc, dt, flush=True)
    g = hj.jacobi_solve(1, n, 1, p["h"], p["f"], p["bc"], p["x0"], **kw)
    o = oracle.solve(1, n, 1, p["h"], p["f"], p["bc"], p["x0"], **kw)
    print("  cycles", g["cycles"], o["cycles"], "bitwise", np.array_equal(g["x"], o["x"]), flush=True)
