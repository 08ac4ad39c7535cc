"""Measured cycles and time to 1e-6 at 8192^2 (paper protocol P, fp64) for the hierarchical solver —
the fourth point of the cycles-vs-size fit behind bench.py's labelled 16384^2 projection."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2006_16465_b200 import hj
from paper_2006_16465_b200.inputs import make_problem

dev = torch.device("cuda:0")
n = 8192
p = make_problem("P", 2, n)
t = {k: torch.from_numpy(p[k]).to(dev) for k in ("f", "bc", "x0")}
out = {"n": n, "tol": 1e-6, "protocol": "P", "runs": {}}
for name, kw in (("hier_k64_o10", dict(mode="hier", tile=(32, 32), k=64, overlap=10)),
                 ("hier_k16_o0", dict(mode="hier", tile=(32, 32), k=16))):
    t0 = time.time()
    r = hj.jacobi_solve_device(2, n, n, p["h"], t["f"], t["bc"], t["x0"], tol=1e-6, max_cycles=10**8,
                               history=False, **kw)
    out["runs"][name] = {"cycles": r["cycles"], "seconds_solve": r["seconds_solve"], "converged": r["converged"],
                         "wall": time.time() - t0}
    print(name, json.dumps(out["runs"][name]), flush=True)
    os.makedirs("gpurun_out", exist_ok=True)
    json.dump(out, open("gpurun_out/convergence_8192.json", "w"), indent=1)
