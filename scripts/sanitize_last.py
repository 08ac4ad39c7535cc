"""compute-sanitizer cases for the kernels changed in the last session of round 2 (the rest of the
kernels: scripts/sanitize_cases.py): res1w with the software-pipelined exchange (C = 8, 4, 16, 32; odd
and even k; f32), res1c layouts, and the REGT large tiles' named-barrier exchange (mode 2, the default)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_16465_b200 import hj
from paper_2006_16465_b200.inputs import make_problem

cases = [
    (1, 256, 1, dict(mode="hier", tile=32, k=16)),                      # res1w C = 8, config 1 layout
    (1, 256, 1, dict(mode="hier", tile=64, k=7)),                       # odd k
    (1, 128, 1, dict(mode="hier", tile=32, k=6, dtype="f32")),          # C = 4, f32
    (1, 1024, 1, dict(mode="hier", tile=32, k=5)) ,                     # res1c (8, 4) default for nx >= 512
    (1, 512, 1, dict(mode="hier", tile=128, k=4, dtype="f32")),
    (2, 192, 96, dict(mode="hier", tile=(64, 32), k=5)),                # REGT large, named barrier
    (2, 96, 192, dict(mode="hier", tile=(32, 64), k=4)),
    (2, 128, 192, dict(mode="hier", tile=(64, 64), k=6)),
    (2, 256, 96, dict(mode="hier", tile=(128, 32), k=3, dtype="f32")),
]
for dim, nx, ny, kw in cases:
    p = make_problem("R", dim, nx, ny)
    r = hj.jacobi_solve(dim, nx, ny, p["h"], p["f"], p["bc"], p["x0"], tol=1e-9, max_cycles=6, **kw)
    print(dim, nx, ny, kw, "cycles", r["cycles"], "status", r["status"])
for lay in ("2,4", "4,2", "1,1"):
    os.environ["HJ_RES1C"] = lay
    p = make_problem("R", 1, 256, 1)
    r = hj.jacobi_solve(1, 256, 1, p["h"], p["f"], p["bc"], p["x0"], mode="hier", tile=32, k=9, tol=1e-9, max_cycles=5)
    print("HJ_RES1C", lay, "cycles", r["cycles"], "status", r["status"])
print("sanitize (last session) cases done")
