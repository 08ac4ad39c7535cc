"""Measured cycles-to-1e-6 vs grid size (paper protocol, fp64) and a power-law projection to
16384^2 — the basis of bench.py's labelled time-to-1e-6 projection."""
import json, math, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2006_16465_b200 import hj
from paper_2006_16465_b200.inputs import make_problem

dev = torch.device("cuda:0")
TOL = 1e-6


def cycles(n, **kw):
    p = make_problem("P", 2, n)
    t = {k: torch.from_numpy(p[k]).to(dev) for k in ("f", "bc", "x0")}
    torch.cuda.synchronize()
    r = hj.jacobi_solve_device(2, n, n, p["h"], t["f"], t["bc"], t["x0"], tol=TOL, max_cycles=10**8,
                               history=False, **kw)
    return r["cycles"], r["seconds_solve"]


configs = {"hier_k16_o0": dict(mode="hier", tile=(32, 32), k=16),
           "hier_k64_o10": dict(mode="hier", tile=(32, 32), k=64, overlap=10),
           "classic": dict(mode="classic")}
sizes = {"hier_k16_o0": (256, 512, 1024, 2048, 4096), "hier_k64_o10": (256, 512, 1024, 2048, 4096),
         "classic": (256, 512, 1024, 2048)}
out = {"tol": TOL, "protocol": "P", "data": {}, "fit": {}}
for name, kw in configs.items():
    pts = []
    for n in sizes[name]:
        t0 = time.time()
        c, s = cycles(n, **kw)
        pts.append((n, c, s))
        print(name, n, c, f"{s:.2f}s", flush=True)
    out["data"][name] = pts
    # power law through the last three sizes
    xs = [math.log(n) for n, _, _ in pts[-3:]]
    ys = [math.log(c) for _, c, _ in pts[-3:]]
    mx, my = sum(xs) / 3, sum(ys) / 3
    b = sum((x - mx) * (y - my) for x, y in zip(xs, ys)) / sum((x - mx) ** 2 for x in xs)
    a = my - b * mx
    out["fit"][name] = {"exponent": b, "cycles_16384": math.exp(a + b * math.log(16384))}
    print(name, "fit exponent", b, "projected cycles at 16384^2:", out["fit"][name]["cycles_16384"], flush=True)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/convergence_scaling.json", "w"), indent=1)
