"""One config-1 solve (1D N = 256, 8 tiles of 32, k = 16, protocol P, 1e-8) through jacobi_solve_device —
the resident one-warp kernel (res1w), for an ncu capture."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2006_16465_b200 import hj
from paper_2006_16465_b200.inputs import make_problem
dev = torch.device("cuda:0")
p = make_problem("P", 1, 256)
t = {k: torch.from_numpy(p[k]).to(dev) for k in ("f", "bc", "x0")}
r = hj.jacobi_solve_device(1, 256, 1, p["h"], t["f"], t["bc"], t["x0"], mode="hier", tile=32, k=16, tol=1e-8,
                           max_cycles=int(os.environ.get("CFG1_MAX", 10**8)), history=False)
print("cycles", r["cycles"], "ms", r["seconds_solve"] * 1e3)
