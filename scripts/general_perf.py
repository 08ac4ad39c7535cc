"""Cycle-kernel time of the general-coefficient stencils (Eq. 10 / Eq. 4) vs the Poisson stencil on
one B200 — same tiles, same k — plus time-to-1e-4 on an anisotropic grid.  Markdown to stdout."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2006_16465_b200 import hj
from paper_2006_16465_b200.inputs import make_general

dev = torch.device("cuda:0")
s = torch.cuda.Stream(dev)


def kernel_ms(dim, nx, ny, h, f, x0, stencil, **prm):
    p = hj.Plan(dim, nx, ny, h, f, None, x0, stream=s.cuda_stream, tol=0.0, max_cycles=1 << 62,
                stencil=stencil, **prm)
    p.run(3, timed=True)
    ms = p.run(10, timed=True) / 10
    p.close()
    return ms


n = 16384
f = torch.ones(n * n, dtype=torch.float64, device=dev)
x0 = torch.ones(n * n, dtype=torch.float64, device=dev)
dx = 1.0 / (n + 1)
aniso = np.array([-1 / dx ** 2, -1 / dx ** 2, -4 / dx ** 2, -4 / dx ** 2, 10 / dx ** 2])
print(f"### 2D {n}^2, 32x32 tiles: cycle-kernel ms (CUDA events), Poisson vs general (Eq. 10)\n")
print("| dtype | k | Poisson ms | general ms | general / Poisson | general HBM GB/s |")
print("|---|---|---|---|---|---|")
for dtype in ("f64", "f32"):
    for k in (4, 16, 64):
        a = kernel_ms(2, n, n, 1.0 / (n + 1), f, x0, None, mode="hier", tile=(32, 32), k=k, dtype=dtype)
        b = kernel_ms(2, n, n, 1.0, f, x0, aniso, mode="hier", tile=(32, 32), k=k, dtype=dtype)
        bpc = 24 if dtype == "f64" else 12
        print(f"| {dtype} | {k} | {a:.3f} | {b:.3f} | {b / a:.3f} | {bpc * n * n / b / 1e6:.0f} |", flush=True)
for dtype in ("f64",):
    a = kernel_ms(2, n, n, 1.0 / (n + 1), f, x0, None, mode="classic", dtype=dtype)
    b = kernel_ms(2, n, n, 1.0, f, x0, aniso, mode="classic", dtype=dtype)
    print(f"| {dtype} classic | 1 | {a:.3f} | {b:.3f} | {b / a:.3f} | {24 * n * n / b / 1e6:.0f} |")
del f, x0
torch.cuda.empty_cache()

print("\n### 1D: 1024 problems x 2^14 points (recipe V, per-point coefficients, 40 B/point/cycle f64)\n")
print("| tile | k | Poisson ms | general ms | general / Poisson | general HBM GB/s |")
print("|---|---|---|---|---|---|")
nx, B = 1 << 14, 1024
pv = make_general("V", 1, nx, batch=B)
f1 = torch.ones(nx * B, dtype=torch.float64, device=dev)
x1 = torch.ones(nx * B, dtype=torch.float64, device=dev)
for tile, k in ((256, 16), (256, 64), (1024, 64)):
    a = kernel_ms(1, nx, B, 1.0 / (nx + 1), f1, x1, None, mode="hier", tile=(tile, 1), k=k)
    b = kernel_ms(1, nx, B, 1.0, f1, x1, pv["stencil"], mode="hier", tile=(tile, 1), k=k)
    print(f"| {tile} | {k} | {a:.3f} | {b:.3f} | {b / a:.3f} | {40 * nx * B / b / 1e6:.0f} |", flush=True)

print("\n### Time to 1e-4 (relative), anisotropic Poisson, protocol P (b = 1, x0 = 1)\n")
print("| grid | k | cycles | seconds | classic sweeps | classic seconds | speedup |")
print("|---|---|---|---|---|---|---|")
for nx_, ny_ in ((512, 384),):
    p = make_general("A", 2, nx_, ny_)
    t = {k_: torch.as_tensor(p[k_], device=dev) for k_ in ("f", "x0")}
    pl = hj.Plan(2, nx_, ny_, 1.0, t["f"], None, t["x0"], stream=s.cuda_stream, tile=(32, 32), k=16,
                 tol=1e-4, max_cycles=10**7, stencil=p["stencil"])
    r = pl.solve(history=False); pl.close()
    pc = hj.Plan(2, nx_, ny_, 1.0, t["f"], None, t["x0"], stream=s.cuda_stream, mode="classic",
                 tol=1e-4, max_cycles=10**8, stencil=p["stencil"])
    rc = pc.solve(history=False); pc.close()
    print(f"| {nx_}x{ny_} | 16 | {r['cycles']} | {r['seconds_solve']:.3f} | {rc['cycles']} | "
          f"{rc['seconds_solve']:.3f} | {rc['seconds_solve'] / r['seconds_solve']:.2f} |", flush=True)
