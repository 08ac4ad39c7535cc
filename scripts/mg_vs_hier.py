"""Time to tolerance on one B200: classic Jacobi vs the paper's hierarchical cycle vs multigrid with
the hierarchical smoother (NEXT #4), on the paper-style workloads at odd sizes (multigrid needs odd
n).  Device-resident inputs, jacobi_solve_device (graph loop, residual tested every cycle on the
device).  Protocol P (f = 1, x0 = 1, g = 0), relative tolerance, fp64.  Prints markdown.

    python scripts/mg_vs_hier.py > profiles/r01_mg_vs_hier.md
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2006_16465_b200 import hj
from paper_2006_16465_b200.inputs import make_problem

dev = torch.device("cuda:0")


def solve(dim, n, tol, batch=1, **kw):
    p = make_problem("P", dim, n, batch=batch)
    t = {k: torch.from_numpy(p[k]).to(dev) for k in ("f", "bc", "x0")}
    torch.cuda.synchronize()
    args = (dim, p["nx"], p["ny"], p["h"], t["f"], t["bc"], t["x0"])
    hj.jacobi_solve_device(*args, tol=tol, max_cycles=10**8, history=False, **kw)  # warm (graphs, caches)
    return hj.jacobi_solve_device(*args, tol=tol, max_cycles=10**8, history=False, **kw)


def row(name, r):
    return f"| {name} | {r['cycles']} | {r['seconds_solve'] * 1e3:.2f} | {'yes' if r['converged'] else 'no'} |"


def main():
    out = ["# Time to tolerance: classic vs hierarchical vs multigrid (one B200, fp64, protocol P)\n",
           "Device solve loop only (`seconds_solve`), second of two identical solves.  Multigrid: V(1,1),",
           "32x32 (2D) / 256 (1D) smoother tiles, k = 4, omega 4/5 (2D) / 2/3 (1D), coarsening to one point.\n"]
    for n, tol in ((1023, 1e-4), (1023, 1e-6), (4095, 1e-6)):
        out.append(f"\n## 2D {n}x{n}, relative tolerance {tol}\n")
        out.append("| solver | cycles | ms | converged |\n|---|---|---|---|")
        if n <= 1023:
            out.append(row("classic (global-memory Jacobi)", solve(2, n, tol, mode="classic")))
        out.append(row("hierarchical 32x32, k=16, o=0", solve(2, n, tol, mode="hier", tile=(32, 32), k=16)))
        if n <= 1023:
            out.append(row("hierarchical 32x32, k=64, o=10", solve(2, n, tol, mode="hier", tile=(32, 32), k=64,
                                                                 overlap=10)))
        out.append(row("multigrid V(1,1), hierarchical smoother k=4", solve(2, n, tol, mode="mg", tile=(32, 32), k=4)))
    for n, batch, tol in ((1023, 1024, 1e-6), ((1 << 20) - 1, 1, 1e-6)):
        out.append(f"\n## 1D {batch} problem(s) of N={n}, relative tolerance {tol}\n")
        out.append("| solver | cycles | ms | converged |\n|---|---|---|---|")
        t = 32 if n < 2048 else 1024
        out.append(row(f"hierarchical tile {t}, k=16", solve(1, n, tol, batch=batch, mode="hier", tile=t, k=16)))
        out.append(row("multigrid V(1,1), hierarchical smoother tile 256, k=4",
                       solve(1, n, tol, batch=batch, mode="mg", tile=256, k=4)))
    print("\n".join(out))


if __name__ == "__main__":
    main()
