"""Small solves over every kernel family, for compute-sanitizer runs (no oracle; just exercise)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_16465_b200 import hj
from paper_2006_16465_b200.inputs import make_problem

cases = [
    (2, 100, 70, dict(mode="hier", tile=(32, 32), k=5)),           # reg2d + ragged edge tiles
    (2, 96, 64, dict(mode="hier", tile=(32, 32), k=4, dtype="f32")),
    (2, 33, 40, dict(mode="hier", tile=(32, 32), k=3, kernel="smem")),
    (2, 19, 13, dict(mode="hier", tile=(4, 5), k=7)),
    (2, 300, 37, dict(mode="classic")),
    (1, 5000, 1, dict(mode="hier", tile=128, k=7)),
    (1, 1000, 1, dict(mode="hier", tile=96, k=5)),
    (1, 5000, 1, dict(mode="classic")),
    (2, 100, 70, dict(mode="hier", tile=(32, 32), k=5, overlap=4)),   # overlapping blocks, reg2d
    (2, 40, 30, dict(mode="hier", tile=(8, 8), k=4, overlap=2)),      # overlapping blocks, smem2d
    (2, 128, 64, dict(mode="hier", tile=(32, 32), k=4, overlap=8, dtype="f32")),
    (2, 96, 64, dict(mode="hier", tile=(32, 32), k=4, overlap=2, dtype="f32")),
    (1, 1000, 1, dict(mode="hier", tile=64, k=7, overlap=10)),         # overlapping blocks, smem1d
    (1, 1024, 9, dict(mode="hier", tile=32, k=16)),                     # batched 1D, reg1d
    (1, 1000, 5, dict(mode="hier", tile=96, k=3)),                      # batched 1D, smem1d
    (1, 3000, 4, dict(mode="classic")),                                 # batched 1D, classic
    (2, 127, 95, dict(mode="mg", tile=(32, 32), k=3, nu1=1, nu2=1)),    # multigrid, fused correction
    (2, 127, 95, dict(mode="mg", tile=(32, 32), k=3, nu1=2, nu2=1, dtype="f32")),  # unfused correction
    (2, 63, 63, dict(mode="mg", tile=(8, 8), k=2, nu1=0, nu2=2)),        # smem levels, residual-only pass
    (1, 1023, 3, dict(mode="mg", tile=64, k=3)),                         # 1D multigrid
    (2, 256, 128, dict(mode="hier", tile=(32, 32), k=6)),                # resident 2D (multi-CTA barrier)
    (1, 256, 1, dict(mode="hier", tile=32, k=16)),                      # resident 1D, one CTA
    (1, 4096, 2, dict(mode="hier", tile=128, k=5)),                     # resident 1D, multi-CTA
    # round 2
    (1, 1024, 1, dict(mode="hier", tile=32, k=5)),                      # resident 1D, one warp (res1w, C = 32)
    (1, 256, 1, dict(mode="hier", tile=64, k=4, dtype="f32")),          # res1w, C = 8
    (2, 96, 64, dict(mode="hier", tile=(16, 16), k=5)),                 # REGT: several tiles per warp
    (2, 64, 96, dict(mode="hier", tile=(32, 16), k=4, dtype="f32")),
    (2, 192, 96, dict(mode="hier", tile=(64, 32), k=5)),                # REGT: warp group per tile
    (2, 128, 192, dict(mode="hier", tile=(64, 64), k=6)),
    (2, 256, 96, dict(mode="hier", tile=(128, 32), k=3, dtype="f32")),
    (2, 100, 70, dict(mode="hier", tile=(32, 32), k=5, overlap=(0, 4))),  # one-axis overlap
]
for dim, nx, ny, kw in cases:
    p = make_problem("R", dim, nx, ny) if (dim == 2 or ny == 1) else make_problem("R", 1, nx, batch=ny)
    r = hj.jacobi_solve(dim, nx, ny, p["h"], p["f"], p["bc"], p["x0"], tol=1e-9, max_cycles=6, **kw)
    print(dim, nx, ny, kw, "cycles", r["cycles"], "status", r["status"])
for lay in ("1,4", "4,2", "8,1", "2,1", "0"):  # res1c layouts (C, D); "0" = res1w
    os.environ["HJ_RES1C"] = lay
    for dim, nx, ny, kw in [(1, 256, 1, dict(mode="hier", tile=32, k=7)),
                            (1, 256, 1, dict(mode="hier", tile=64, k=4, dtype="f32"))]:
        p = make_problem("R", dim, nx, ny)
        r = hj.jacobi_solve(dim, nx, ny, p["h"], p["f"], p["bc"], p["x0"], tol=1e-9, max_cycles=6, **kw)
        print(dim, nx, ny, kw, "HJ_RES1C", lay, "cycles", r["cycles"], "status", r["status"])
os.environ.pop("HJ_RES1C")
os.environ["HJ_RESIDENT"] = "0"   # the per-cycle path of a resident-eligible grid (run with HJ_SPLIT_CYCLE=1 too)
for dim, nx, ny, kw in [(2, 128, 128, dict(mode="hier", tile=(32, 32), k=4))]:
    p = make_problem("R", dim, nx, ny)
    r = hj.jacobi_solve(dim, nx, ny, p["h"], p["f"], p["bc"], p["x0"], tol=1e-9, max_cycles=6, **kw)
    print(dim, nx, ny, kw, "per-cycle", "cycles", r["cycles"], "status", r["status"])
print("sanitize cases done")
