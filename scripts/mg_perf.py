"""Multigrid (NEXT #4) measurements on one B200: V-cycles and time to tolerance, per-V-cycle time.

    python scripts/mg_perf.py [--out profiles/r01_mg_perf.json]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2006_16465_b200 import hj
from paper_2006_16465_b200.inputs import make_problem


def run(n, proto, tol, k, nu1, nu2, dtype="f64", tile=(32, 32)):
    p = make_problem(proto, 2, n)
    dev = torch.device("cuda", 0)
    t = lambda a: torch.as_tensor(a, device=dev)
    prm = dict(mode="mg", tile=tile, k=k, nu1=nu1, nu2=nu2, tol=tol, max_cycles=500, dtype=dtype)
    tplan = hj.Plan(2, n, n, p["h"], t(p["f"]), t(p["bc"]), t(p["x0"]), **dict(prm, tol=0.0))
    tplan.run(2)
    torch.cuda.synchronize()
    ms = tplan.run(8, timed=True) / 8   # steady V-cycle time (tol 0: no early exit)
    tplan.close()
    plan = hj.Plan(2, n, n, p["h"], t(p["f"]), t(p["bc"]), t(p["x0"]), **prm)
    torch.cuda.synchronize()
    r = plan.solve(history=True)
    hist = r["history"].cpu().numpy()
    plan.reset()
    plan.solve(history=False)          # second solve: graphs already instantiated
    plan.reset()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r2 = plan.solve(history=False)
    wall = time.perf_counter() - t0
    out = dict(n=n, proto=proto, tol=tol, k=k, nu1=nu1, nu2=nu2, dtype=dtype, vcycles=r["cycles"],
               converged=r["converged"], seconds=r2["seconds_solve"], wall=wall, ms_per_vcycle=ms,
               launches_per_vcycle=plan.launches_per_cycle(),
               rate=float((hist[-1] / hist[0]) ** (1.0 / max(1, r["cycles"]))),
               cell_updates_per_s_fine=n * n * k * (nu1 + nu2) / (ms * 1e-3))
    plan.close()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--quick", action="store_true")
    a = ap.parse_args()
    rows = []
    sizes = [1023, 4095, 16383] if not a.quick else [1023]
    for n in sizes:
        for proto in ("P", "M"):
            for k, nu1, nu2 in ((4, 1, 1), (2, 1, 1), (8, 1, 1), (4, 2, 2), (4, 2, 1), (4, 1, 2),
                                (2, 2, 2), (4, 3, 3), (1, 1, 1)):
                if n == 1023 and (nu1, nu2) != (1, 1):
                    continue
                r = run(n, proto, 1e-6, k, nu1, nu2)
                rows.append(r)
                print(json.dumps(r), flush=True)
    for dtype in ("f32",):
        r = run(sizes[-1], "P", 1e-5, 4, 1, 1, dtype=dtype)
        rows.append(r)
        print(json.dumps(r), flush=True)
    if a.out:
        json.dump(rows, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
