"""BASELINE config 5 on one B200: 32768^2, fp32 vs fp64, tile-size and k sweep — per-cycle time,
HBM roofline fraction (24 B/cell f64, 12 B/cell f32 vs MEASURED_PEAKS hbm_gbs) and measured
cycles/time to 1e-4 (paper protocol) for the main configurations."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2006_16465_b200 import hj

N = int(os.environ.get("C5_N", 32768))
dev = torch.device("cuda:0")
peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6650.0
h = 1.0 / (N + 1)
f = torch.ones(N * N, dtype=torch.float64, device=dev)
x0 = torch.ones(N * N, dtype=torch.float64, device=dev)
s = torch.cuda.Stream(dev)
rows = []
print(f"| dtype | tile | k | ms/cycle | cell-updates/s | HBM GB/s | frac of {peak:.0f} |")
print("|---|---|---|---|---|---|---|")
for dtype in ("f64", "f32"):
    for tile in ((32, 32), (16, 16), (32, 16), (16, 32)):
        for k in (1, 4, 8, 16, 32, 64):
            if tile != (32, 32) and k not in (4, 16):
                continue
            p = hj.Plan(2, N, N, h, f, None, x0, stream=s.cuda_stream, mode="hier", tile=tile, k=k, tol=0.0,
                        max_cycles=1 << 62, dtype=dtype)
            p.run(2, timed=True)
            ms = p.run(6, timed=True) / 6
            p.close()
            bpc = 24 if dtype == "f64" else 12
            gbs = bpc * N * N / ms / 1e6
            rows.append(dict(dtype=dtype, tile=tile, k=k, ms=ms, gbs=gbs))
            print(f"| {dtype} | {tile[0]}x{tile[1]} | {k} | {ms:.2f} | {N*N*k/ms*1e3:.3e} | {gbs:.0f} | {gbs/peak:.2f} |", flush=True)
print()
print("| dtype | tile | k | cycles to 1e-4 | seconds (device loop) |\n|---|---|---|---|---|")
for dtype, k in (("f64", 16), ("f32", 16), ("f32", 4)):
    p = hj.Plan(2, N, N, h, f, None, x0, stream=s.cuda_stream, mode="hier", tile=(32, 32), k=k, tol=1e-4,
                max_cycles=10**7, dtype=dtype)
    r = p.solve(history=False)
    p.close()
    rows.append(dict(dtype=dtype, tile=(32, 32), k=k, ttt_cycles=r["cycles"], ttt_s=r["seconds_solve"],
                     converged=r["converged"]))
    print(f"| {dtype} | 32x32 | {k} | {r['cycles']} | {r['seconds_solve']:.1f} |", flush=True)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(rows, open("gpurun_out/config5.json", "w"), indent=1)
