"""Small single 1D problems (BASELINE config 1 and the paper's single N = 1024): time to tolerance of the
resident one-warp kernel (res1w, HJ_RES1C=0) against the one-CTA kernel (res1c) for every layout (C, D),
device loop time (CUDA events inside hj_plan_solve), best of 3 after one warm-up solve.
    python scripts/res1c_sweep.py   -> gpurun_out/res1c_sweep.json"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2006_16465_b200 import hj
from paper_2006_16465_b200.inputs import make_problem

dev = torch.device("cuda:0")
WL = [("config1 M", "M", 256, 32, 16, 1e-8), ("config1 P", "P", 256, 32, 16, 1e-8),
      ("1D N=1024 P", "P", 1024, 32, 16, 1e-6)]
LAY = ["0", "1,1", "1,2", "1,4", "2,1", "2,2", "2,4", "4,1", "4,2", "4,4", "8,1", "8,2", "8,4"]
out = {}
for name, proto, n, tile, k, tol in WL:
    p = make_problem(proto, 1, n)
    t = {kk: torch.from_numpy(p[kk]).to(dev) for kk in ("f", "bc", "x0")}
    for lay in LAY:
        os.environ["HJ_RES1C"] = lay
        best, cyc = None, None
        for rep in range(4):
            r = hj.jacobi_solve_device(1, n, 1, p["h"], t["f"], t["bc"], t["x0"], mode="hier", tile=tile, k=k,
                                       tol=tol, max_cycles=10**8, history=False)
            if rep:
                best = r["seconds_solve"] if best is None else min(best, r["seconds_solve"])
            cyc = r["cycles"]
        out[f"{name} {'res1w' if lay == '0' else 'res1c ' + lay}"] = {"cycles": cyc, "ms": round(best * 1e3, 3),
                                                                      "us_per_cycle": round(best * 1e6 / cyc, 4)}
        print(name, lay, out[f"{name} {'res1w' if lay == '0' else 'res1c ' + lay}"], flush=True)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/res1c_sweep.json", "w"), indent=1)
