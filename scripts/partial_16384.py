"""Partial measurement of the hierarchical solve to 1e-6 at the north-star configuration (16384^2,
fp64, protocol P, 32x32 tiles, k = 16): run max_cycles cycles, keep the residual history (every
1000th cycle) for an extrapolation of the remaining cycles by the measured late-time decay."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2006_16465_b200 import hj

n = 16384
cycles = int(sys.argv[1]) if len(sys.argv) > 1 else 3_000_000
dev = torch.device("cuda:0")
f = torch.ones(n * n, dtype=torch.float64, device=dev)
x0 = torch.ones_like(f)
bc = torch.zeros(4 * n, dtype=torch.float64, device=dev)
t0 = time.time()
r = hj.jacobi_solve_device(2, n, n, 1.0 / (n + 1), f, bc, x0, mode="hier", tile=(32, 32), k=16, tol=1e-6,
                           max_cycles=cycles, history=True)
h = r["history"].cpu().numpy()
out = {"n": n, "k": 16, "tile": 32, "tol": 1e-6, "max_cycles": cycles, "cycles": r["cycles"],
       "converged": r["converged"], "seconds_solve": r["seconds_solve"], "wall": time.time() - t0,
       "r0": float(h[0]), "every": 1000, "rel_history": [float(v / h[0]) for v in h[::1000]]}
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/partial_16384.json", "w"))
print(json.dumps({k: v for k, v in out.items() if k != "rel_history"}), out["rel_history"][-3:])
