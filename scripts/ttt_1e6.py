"""MEASURED time-to-1e-6 of the hierarchical solver on BASELINE's 16384^2 fp64 grid (north star target;
VERDICT r1 missing #2 / next #4): 32x32 tiles, k = 16, protocol P (f = 1, x0 = 1, g = 0), the paper's
relative stopping rule ||r_c|| <= 1e-6 ||r_0|| tested after every cycle (reading c1).

One B200, device-resident data.  The solve runs in resumed segments of SEG cycles through the public
device API (jacobi_solve_device: x0 = the previous segment's iterate, ref_residual = ||r_0|| of the
first segment, so every segment applies the same threshold); each segment's device loop time (CUDA
events inside hj_plan_solve) is summed.  A segment's first cycle recomputes the residual of its starting
iterate (the previous segment's last residual-only pass): one extra residual pass per segment.

The solve needs hours and a lease is at most one hour, so after every segment the iterate and the
running totals are checkpointed on the box (CKPT, default /root/.cache/hj_ttt: it survives into the
next call when that call lands on the same box within minutes); a call resumes from a checkpoint of the
same configuration and stops starting segments after WALL seconds.  The iteration is deterministic
(bitwise the same iterate for any segmentation: a segment only changes where the loop pauses), so the
resumed count equals an uninterrupted solve's — checked at 256^2 (8,802 cycles segmented and not).
    TTT_WALL=2900 python scripts/ttt_1e6.py   (gpurun_out/ttt_1e-06_16384_<time>.jsonl per call, summary .json when done)"""
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
WALL = float(os.environ.get("TTT_WALL", 1e9))
CKPT = os.environ.get("TTT_CKPT", "/root/.cache/hj_ttt")
os.makedirs("gpurun_out", exist_ok=True)
LOG = f"gpurun_out/ttt_{TOL:g}_{N}_{time.strftime('%H%M%S')}.jsonl"  # one file per call (merged back)
tag = {"grid": N, "k": K, "tol": TOL, "segment": SEG}
dev = torch.device("cuda:0")
h = 1.0 / (N + 1)
f = torch.ones(N * N, dtype=torch.float64, device=dev)
bc = torch.zeros(4 * N, dtype=torch.float64, device=dev)
prm = dict(mode="hier", tile=(32, 32), k=K, tol=TOL, tol_mode="rel", history=False)
state = {"cycles": 0, "seconds_device": 0.0, "r0": 0.0, "segments": 0, "calls": 0}
x = None
st_path, x_path = os.path.join(CKPT, "state.json"), os.path.join(CKPT, "x.pt")
if os.path.exists(st_path) and os.path.exists(x_path):
    s = json.load(open(st_path))
    if s.get("tag") == tag:
        state = s["state"]
        x = torch.load(x_path, map_location=dev)
        print("resumed from checkpoint:", state, flush=True)
if x is None:
    x = torch.ones(N * N, dtype=torch.float64, device=dev)
state["calls"] += 1
t_start = time.time()
rec = None
with open(LOG, "a") as log:
    log.write(json.dumps({"start": time.strftime("%Y-%m-%dT%H:%M:%S"), **tag, "gpu": torch.cuda.get_device_name(0),
                          "resumed_at": state["cycles"], "call": state["calls"]}) + "\n")
    while True:
        if time.time() - t_start > WALL:
            print("wall budget of this call reached; resume in the next call", flush=True)
            break
        r = hj.jacobi_solve_device(2, N, N, h, f, bc, x, max_cycles=SEG, ref_residual=state["r0"], **prm)
        if state["r0"] == 0.0:
            state["r0"] = r["initial_residual"]
        state["cycles"] += r["cycles"]
        state["seconds_device"] += r["seconds_solve"]
        state["segments"] += 1
        x = r["x"].reshape(-1).clone()
        rec = {"cycles": state["cycles"], "seconds_device": state["seconds_device"], "wall_s": time.time() - t_start,
               "residual": r["final_residual"], "rel": r["final_residual"] / state["r0"],
               "converged": r["converged"], "segment_cycles": r["cycles"], "segment_seconds": r["seconds_solve"]}
        log.write(json.dumps(rec) + "\n")
        log.flush()
        print(rec, flush=True)
        done = r["converged"] or state["cycles"] >= MAXC
        if not done:
            os.makedirs(CKPT, exist_ok=True)
            torch.save(x, x_path + ".tmp")
            os.replace(x_path + ".tmp", x_path)
            json.dump({"tag": tag, "state": state}, open(st_path + ".tmp", "w"))
            os.replace(st_path + ".tmp", st_path)
        else:
            summary = {"measured": True, "grid": N, "tile": [32, 32], "k": K, "tol": TOL,
                       "protocol": "P (f=1, x0=1, g=0)", "cycles": state["cycles"],
                       "seconds_device": state["seconds_device"],
                       "ms_per_cycle": state["seconds_device"] / max(state["cycles"], 1) * 1e3,
                       "initial_residual": state["r0"], "final_rel_residual": rec["rel"],
                       "converged": rec["converged"], "segments_of": SEG, "segments": state["segments"],
                       "calls": state["calls"], "api": "jacobi_solve_device in resumed segments (ref_residual = r_0)"}
            json.dump(summary, open(f"gpurun_out/ttt_{TOL:g}_{N}.json", "w"), indent=1)
            print(json.dumps(summary), flush=True)
            for p in (x_path, st_path):
                if os.path.exists(p):
                    os.remove(p)
            break
