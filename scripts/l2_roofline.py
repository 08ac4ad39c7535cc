"""BASELINE configs 2 and 3 (L2-resident working sets) against the MEASURED L2 bandwidth (VERDICT r1
missing #5).

* L2 peak: a device-to-device copy (torch copy_, the same measurement MEASURED_PEAKS.json uses for HBM)
  of a buffer whose read + write footprint fits the 126 MB L2 (2 x 24 MB), repeated back to back,
  best of 20 — bytes read + written / time.
* Config 2 (1D Poisson N = 2^20, subdomains of 1024, k in {1, 4, 16, 64}, fp64): the per-cycle path
  (HJ_RESIDENT=0: every cycle streams x_c, q and x_{c+1} — 24 B per point, 25 MB per cycle, L2-resident)
  timed with CUDA events around each cycle kernel -> GB/s and the fraction of the L2 peak; the FP64
  fraction (2k + 3 ops per point; 64 FP64 ops/clk/SM at the clock seen); and the resident solver's
  time to 1e-4 (paper protocol) beside the per-cycle path's.
* Config 3 (2D 1024^2, 32x32 tiles, k = 16, fp64): the same for the 2D cycle (24 B per cell, 4k + 3
  FP64 ops per cell).
    python scripts/l2_roofline.py   (writes gpurun_out/l2_roofline.json)"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2006_16465_b200 import hj

dev = torch.device("cuda:0")
st = torch.cuda.Stream(dev)


def l2_copy_gbs(mb=24):
    n = mb * (1 << 20) // 8
    a = torch.rand(n, dtype=torch.float64, device=dev)
    b = torch.empty_like(a)
    for _ in range(5):
        b.copy_(a)
    best = 0.0
    for _ in range(20):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(50):
            b.copy_(a)
        e1.record()
        e1.synchronize()
        best = max(best, 2 * 8 * n * 50 / (e0.elapsed_time(e1) * 1e-3) / 1e9)
    return best


def sm_clock_mhz():
    try:
        import subprocess
        out = subprocess.run(["nvidia-smi", "-i", "0", "--query-gpu=clocks.max.sm", "--format=csv,noheader,nounits"],
                             capture_output=True, text=True).stdout.strip()
        return float(out)
    except Exception:  # noqa: BLE001
        return 1965.0


def per_cycle(dim, nx, ny, tile, k, cycles=200):
    h = 1.0 / (nx + 1)
    f = torch.ones(nx * ny, dtype=torch.float64, device=dev)
    x0 = torch.ones(nx * ny, dtype=torch.float64, device=dev)
    p = hj.Plan(dim, nx, ny, h, f, None, x0, stream=st.cuda_stream, mode="hier", tile=tile, k=k, tol=0.0,
                max_cycles=1 << 62)
    p.run(20, timed=True)
    ms = p.run(cycles, timed=True) / cycles
    p.close()
    return ms


def to_tol(dim, nx, ny, tile, k, resident):
    os.environ["HJ_RESIDENT"] = "1" if resident else "0"
    h = 1.0 / (nx + 1)
    f = torch.ones(nx * ny, dtype=torch.float64, device=dev)
    x0 = torch.ones(nx * ny, dtype=torch.float64, device=dev)
    p = hj.Plan(dim, nx, ny, h, f, None, x0, stream=st.cuda_stream, mode="hier", tile=tile, k=k, tol=1e-4,
                max_cycles=10**7)
    p.solve(history=False)          # warm (graphs, first launch)
    p.reset()
    r = p.solve(history=False)
    p.close()
    os.environ.pop("HJ_RESIDENT", None)
    return r["cycles"], r["seconds_solve"]


def main():
    l2 = l2_copy_gbs()
    mhz = sm_clock_mhz()
    fp64_peak = 148 * 64 * mhz * 1e6
    out = {"l2_copy_gbs": l2, "l2_basis": "torch copy_ of 24 MB (48 MB read+write footprint), best of 20 x 50",
           "fp64_peak_ops": fp64_peak, "fp64_basis": f"148 SMs x 64 FP64 ops/clk x {mhz:.0f} MHz (measured "
                                                     f"achievable: scripts/fp64peak.cu)", "rows": []}
    print(f"L2 copy bandwidth (measured): {l2:.0f} GB/s; FP64 peak {fp64_peak:.3e} ops/s")
    print("| config | k | ms/cycle (per-cycle path) | GB/s (24 B/cell) | frac of L2 | FP64 frac | cycles to 1e-4 | "
          "per-cycle s | resident s |")
    print("|---|---|---|---|---|---|---|---|---|")
    cases = [("cfg2 1D 2^20, T=1024", 1, 1 << 20, 1, 1024, k) for k in (1, 4, 16, 64)] + \
            [("cfg3 2D 1024^2, 32x32", 2, 1024, 1024, (32, 32), 16)]
    for name, dim, nx, ny, tile, k in cases:
        os.environ["HJ_RESIDENT"] = "0"
        ms = per_cycle(dim, nx, ny, tile, k)
        os.environ.pop("HJ_RESIDENT", None)
        cells = nx * ny
        gbs = 24 * cells / (ms * 1e-3) / 1e9
        ops = (2 * k + 3 if dim == 1 else 4 * k + 3) * cells
        fpf = ops / (ms * 1e-3) / fp64_peak
        c1, s1 = to_tol(dim, nx, ny, tile, k, False)
        c2, s2 = to_tol(dim, nx, ny, tile, k, True)
        assert c1 == c2, (c1, c2)
        row = dict(config=name, k=k, ms_per_cycle=ms, gbs=gbs, frac_l2=gbs / l2, fp64_frac=fpf, cycles_1e4=c1,
                   per_cycle_s=s1, resident_s=s2)
        out["rows"].append(row)
        print(f"| {name} | {k} | {ms:.4f} | {gbs:.0f} | {gbs / l2:.2f} | {fpf:.2f} | {c1} | {s1:.3f} | {s2:.3f} |",
              flush=True)
    os.makedirs("gpurun_out", exist_ok=True)
    json.dump(out, open("gpurun_out/l2_roofline.json", "w"), indent=1)


if __name__ == "__main__":
    main()
