"""Config 1 through the one-warp resident solver once (for ncu): 1D N = 256, 8 tiles of 32, k = 16, 1e-8."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_16465_b200 import hj
from paper_2006_16465_b200.inputs import make_problem
p = make_problem("P", 1, 256)
for _ in range(2):
    r = hj.jacobi_solve(1, 256, 1, p["h"], p["f"], p["bc"], p["x0"], mode="hier", tile=32, k=16, tol=1e-8,
                        max_cycles=10**6, history=False)
    print(r["cycles"], r["seconds_solve"])
