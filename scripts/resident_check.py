"""Resident solver vs per-cycle path: time to tolerance on 2D 1024^2 (config 3) and cycle counts.

    python scripts/resident_check.py
"""
import os
import subprocess
import sys

code = r'''
import os, sys, json
sys.path.insert(0, os.getcwd())
import torch
from paper_2006_16465_b200 import hj
from paper_2006_16465_b200.inputs import make_problem
dev = torch.device("cuda:0")
out = {}
for dim, n, mode, k, tol, proto in ((2, 1024, "hier", 16, 1e-4, "P"), (2, 1024, "hier", 16, 1e-6, "P"),
                                    (2, 512, "hier", 8, 1e-6, "P"), (1, 256, "hier", 16, 1e-8, "M"),
                                    (1, 256, "hier", 16, 1e-8, "P"), (1, 1024, "hier", 16, 1e-6, "P"),
                                    (1, 1 << 20, "hier", 64, 1e-4, "P"), (1, 1024, "hier", 16, 1e-4, "B")):
    p = make_problem("P", 1, n, batch=1024) if proto == "B" else make_problem(proto, dim, n)
    t = {kk: torch.from_numpy(p[kk]).to(dev) for kk in ("f", "bc", "x0")}
    args = (p["dim"], p["nx"], p["ny"], p["h"], t["f"], t["bc"], t["x0"])
    kw = dict(mode=mode, tile=(32, 32) if dim == 2 else (1024 if n >= 1 << 20 else 32), k=k, tol=tol,
              max_cycles=10**8, history=False)
    hj.jacobi_solve_device(*args, **kw)
    r = hj.jacobi_solve_device(*args, **kw)
    out[f"{dim}D {n} {proto} {mode} k={k} tol={tol}"] = (r["cycles"], round(r["seconds_solve"] * 1e3, 2))
print(json.dumps(out))
'''
for env in ("1", "0"):
    e = dict(os.environ, HJ_RESIDENT=env)
    r = subprocess.run([sys.executable, "-c", code], env=e, capture_output=True, text=True)
    print("resident" if env == "1" else "per-cycle", r.stdout.strip(), r.stderr[-500:])
