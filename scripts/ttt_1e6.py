"""MEASURED time-to-1e-6 of the hierarchical solver on BASELINE's 16384^2 fp64 grid (north star target;
VERDICT r1 missing #2 / next #4): 32x32 tiles, k = 16, protocol P (f = 1, x0 = 1, g = 0), the paper's
relative stopping rule ||r_c|| <= 1e-6 ||r_0|| tested after every cycle (reading c1).

One B200, device-resident data.  The solve runs in resumed segments of SEG cycles through the public
device API (jacobi_solve_device: x0 = the previous segment's iterate, ref_residual = ||r_0|| of the
first segment, so every segment applies the same threshold) so that progress survives in the log if the
lease ends early; each segment's device loop time (CUDA events inside hj_plan_solve) is summed.  A
segment's first cycle recomputes the residual of its starting iterate (the previous segment's last
residual-only pass), one extra residual pass per segment, negligible against SEG cycles.
    python scripts/ttt_1e6.py   (appends to gpurun_out/ttt_1e-6_16384.jsonl, summary in .json)"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2006_16465_b200 import hj

N = int(os.environ.get("TTT_N", 16384))
K = int(os.environ.get("TTT_K", 16))
TOL = float(os.environ.get("TTT_TOL", 1e-6))
SEG = int(os.environ.get("TTT_SEG", 250000))
MAXC = int(os.environ.get("TTT_MAX", 20_000_000))
os.makedirs("gpurun_out", exist_ok=True)
LOG = f"gpurun_out/ttt_{TOL:g}_{N}.jsonl"
dev = torch.device("cuda:0")
h = 1.0 / (N + 1)
f = torch.ones(N * N, dtype=torch.float64, device=dev)
x = torch.ones(N * N, dtype=torch.float64, device=dev)
bc = torch.zeros(4 * N, dtype=torch.float64, device=dev)
prm = dict(mode="hier", tile=(32, 32), k=K, tol=TOL, tol_mode="rel", history=False)
total, dev_s, r0 = 0, 0.0, 0.0
t_start = time.time()
with open(LOG, "a") as log:
    log.write(json.dumps({"start": time.strftime("%Y-%m-%dT%H:%M:%S"), "grid": N, "k": K, "tol": TOL,
                          "segment": SEG, "gpu": torch.cuda.get_device_name(0)}) + "\n")
    while True:
        r = hj.jacobi_solve_device(2, N, N, h, f, bc, x, max_cycles=SEG, ref_residual=r0, **prm)
        if r0 == 0.0:
            r0 = r["initial_residual"]
        total += r["cycles"]
        dev_s += r["seconds_solve"]
        x = r["x"].reshape(-1).clone()
        rec = {"cycles": total, "seconds_device": dev_s, "wall_s": time.time() - t_start,
               "residual": r["final_residual"], "rel": r["final_residual"] / r0, "converged": r["converged"],
               "segment_cycles": r["cycles"], "segment_seconds": r["seconds_solve"]}
        log.write(json.dumps(rec) + "\n")
        log.flush()
        print(rec, flush=True)
        if r["converged"] or total >= MAXC:
            break
summary = {"measured": True, "grid": N, "tile": [32, 32], "k": K, "tol": TOL, "protocol": "P (f=1, x0=1, g=0)",
           "cycles": total, "seconds_device": dev_s, "ms_per_cycle": dev_s / max(total, 1) * 1e3,
           "initial_residual": r0, "final_rel_residual": rec["rel"], "converged": rec["converged"],
           "segments_of": SEG, "wall_s": time.time() - t_start,
           "api": "jacobi_solve_device in resumed segments (ref_residual = r_0)"}
json.dump(summary, open(f"gpurun_out/ttt_{TOL:g}_{N}.json", "w"), indent=1)
print(json.dumps(summary))
