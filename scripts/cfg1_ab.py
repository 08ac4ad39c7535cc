"""Config 1 (1D N = 256, k = 16, 1e-8, protocols P and M) and the paper's single N = 1024 to 1e-6: device
loop time of the resident solve, best of 5 after a warm-up; one line per workload.  Run once per
setting of HJ_RES1W_UNROLL / HJ_RES1C (the library reads HJ_RES1W_UNROLL once per process)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2006_16465_b200 import hj
from paper_2006_16465_b200.inputs import make_problem
dev = torch.device("cuda:0")
out = {}
for name, proto, n, tol in (("config1 P", "P", 256, 1e-8), ("config1 M", "M", 256, 1e-8), ("1D N=1024 P", "P", 1024, 1e-6)):
    p = make_problem(proto, 1, n)
    t = {k: torch.from_numpy(p[k]).to(dev) for k in ("f", "bc", "x0")}
    ts = []
    for rep in range(6):
        r = hj.jacobi_solve_device(1, n, 1, p["h"], t["f"], t["bc"], t["x0"], mode="hier", tile=32, k=16, tol=tol,
                                   max_cycles=10**8, history=False)
        if rep:
            ts.append(r["seconds_solve"])
    out[name] = {"cycles": r["cycles"], "ms": round(min(ts) * 1e3, 3), "us_per_cycle": round(min(ts) * 1e6 / r["cycles"], 4)}
print(json.dumps({"HJ_RES1W_UNROLL": os.environ.get("HJ_RES1W_UNROLL", "2"), "HJ_RES1C": os.environ.get("HJ_RES1C", "default"), **out}))
