"""BASELINE config 5 on one B200 (round 2): 32768^2, fp32 vs fp64, the tile-size x k sweep with the
register kernels (32x32: REG2D; 16x16, 32x16, 16x32, 64x32, 32x64, 64x64, 128x32: REGT) — per-cycle
time (CUDA events around each cycle kernel), HBM roofline fraction (24 B/cell f64, 12 B/cell f32 vs
MEASURED_PEAKS hbm_gbs), the kernel family that ran, and MEASURED cycles / device time to 1e-4
(paper protocol f = 1, x0 = 1, g = 0).
    C5_N=32768 C5_TTT=1 python scripts/config5_r02.py"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2006_16465_b200 import hj

N = int(os.environ.get("C5_N", 32768))
TTT = os.environ.get("C5_TTT", "1") == "1"
dev = torch.device("cuda:0")
peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6650.0
h = 1.0 / (N + 1)
f = torch.ones(N * N, dtype=torch.float64, device=dev)
x0 = torch.ones(N * N, dtype=torch.float64, device=dev)
s = torch.cuda.Stream(dev)
TILES = [(32, 32), (16, 16), (32, 16), (16, 32), (64, 32), (32, 64), (64, 64), (128, 32)]
rows = []
print(f"grid {N}^2, peak {peak:.0f} GB/s (measured)")
print(f"| dtype | tile | kernel | k | ms/cycle | cell-updates/s | HBM GB/s | frac |")
print("|---|---|---|---|---|---|---|---|")
for dtype in ("f64", "f32"):
    for tile in TILES:
        for k in (1, 4, 16, 64):
            p = hj.Plan(2, N, N, h, f, None, x0, stream=s.cuda_stream, mode="hier", tile=tile, k=k, tol=0.0,
                        max_cycles=1 << 62, dtype=dtype)
            kind = p.kernel_kind()
            p.run(2, timed=True)
            ms = p.run(6, timed=True) / 6
            p.close()
            bpc = 24 if dtype == "f64" else 12
            gbs = bpc * N * N / ms / 1e6
            rows.append(dict(dtype=dtype, tile=tile, k=k, kernel=kind, ms=ms, gbs=gbs, frac=gbs / peak))
            print(f"| {dtype} | {tile[0]}x{tile[1]} | {kind} | {k} | {ms:.2f} | {N*N*k/ms*1e3:.3e} | {gbs:.0f} | "
                  f"{gbs/peak:.2f} |", flush=True)
if TTT:
    print()
    print("| dtype | tile | k | cycles to 1e-4 | seconds (device loop) | cell-updates/s |\n|---|---|---|---|---|---|")
    for dtype, tile in [("f64", t) for t in TILES] + [("f32", t) for t in ((32, 32), (16, 16), (64, 64))]:
        k = 16
        p = hj.Plan(2, N, N, h, f, None, x0, stream=s.cuda_stream, mode="hier", tile=tile, k=k, tol=1e-4,
                    max_cycles=10**7, dtype=dtype)
        r = p.solve(history=False)
        p.close()
        rows.append(dict(dtype=dtype, tile=tile, k=k, ttt_cycles=r["cycles"], ttt_s=r["seconds_solve"],
                         converged=r["converged"]))
        print(f"| {dtype} | {tile[0]}x{tile[1]} | {k} | {r['cycles']} | {r['seconds_solve']:.1f} | "
              f"{N*N*k*r['cycles']/r['seconds_solve']:.3e} |", flush=True)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(rows, open(f"gpurun_out/config5_r02_{N}.json", "w"), indent=1)
