"""B200 analogues of the paper's experiments (Tables 1-4, configs 1-3 of BASELINE.json).

Times are the device solve loop (CUDA graphs, residual checked every cycle on the device) via
jacobi_solve_device; 'total' adds allocation/initialisation.  Paper protocol P (f=1, x0=1,
g=0), relative residual reduction, fp64.  Prints markdown.
"""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2006_16465_b200 import hj
from paper_2006_16465_b200.inputs import make_problem

dev = torch.device("cuda:0")


def solve(dim, n, tol, **kw):
    p = make_problem(kw.pop("protocol", "P"), dim, n, batch=kw.pop("batch", 1))
    t = {k: torch.from_numpy(p[k]).to(dev) for k in ("f", "bc", "x0")}
    torch.cuda.synchronize()
    r = hj.jacobi_solve_device(dim, p["nx"], p["ny"], p["h"], t["f"], t["bc"], t["x0"], tol=tol,
                               max_cycles=10**8, history=False, **kw)
    return r


def table_2d(n=1024, tol=1e-4, ks=(4, 8, 16, 32, 64, 128), overlaps=(0, 2, 4, 6, 8, 10, 12)):
    out = []
    c = solve(2, n, tol, mode="classic")
    out.append(f"### 2D {n}x{n}, tol {tol} (paper Tables 2 and 4 analogue)\n")
    out.append(f"classic (global-memory Jacobi, classic2d_kernel): {c['cycles']} sweeps, "
               f"{c['seconds_solve']*1e3:.1f} ms ({c['seconds_solve']/c['cycles']*1e6:.2f} us/sweep)\n")
    out.append("| k | o | cycles | ms | us/cycle | speedup vs classic |\n|---|---|---|---|---|---|")
    best = {}
    for k in ks:
        for o in overlaps:
            if o >= 32:
                continue
            r = solve(2, n, tol, mode="hier", tile=(32, 32), k=k, overlap=o)
            sp = c["seconds_solve"] / r["seconds_solve"]
            out.append(f"| {k} | {o} | {r['cycles']} | {r['seconds_solve']*1e3:.1f} | "
                       f"{r['seconds_solve']/r['cycles']*1e6:.2f} | {sp:.2f} |")
            if o == 0:
                best.setdefault(k, {})["o0"] = sp
            if sp > best.setdefault(k, {}).get("best", (0, 0))[0]:
                best[k]["best"] = (sp, o)
    out.append("\n| k | speedup o=0 (paper Table 2) | best o | best speedup (paper Table 4) |\n|---|---|---|---|")
    paper2 = dict(zip((4, 8, 16, 32, 64, 128), (2.17, 3.67, 3.98, 2.96, 1.86, 1.09)))
    paper4 = dict(zip((4, 8, 16, 32, 64, 128), ((0, 2.18), (2, 4.22), (2, 5.58), (4, 5.84), (6, 4.88), (8, 3.50))))
    for k in ks:
        b = best[k]
        out.append(f"| {k} | {b['o0']:.2f} (paper {paper2[k]}) | {b['best'][1]} (paper {paper4[k][0]}) | "
                   f"{b['best'][0]:.2f} (paper {paper4[k][1]}) |")
    return "\n".join(out)


def table_1d(n=1024, tol=1e-4, ks=(4, 8, 16, 32, 64, 128), overlaps=(0, 2, 4, 8, 10, 12), batch=1024):
    out = []
    c = solve(1, n, tol, mode="classic", batch=batch)
    out.append(f"### 1D {batch} copies of N={n}, tol {tol} (paper Tables 1 and 3 analogue, PAPER.md:213)\n")
    out.append(f"classic: {c['cycles']} sweeps, {c['seconds_solve']*1e3:.1f} ms\n")
    out.append("| k | o | cycles | ms | speedup vs classic |\n|---|---|---|---|---|")
    for k in ks:
        for o in overlaps:
            r = solve(1, n, tol, mode="hier", tile=32, k=k, overlap=o, batch=batch)
            out.append(f"| {k} | {o} | {r['cycles']} | {r['seconds_solve']*1e3:.1f} | "
                       f"{c['seconds_solve']/r['seconds_solve']:.2f} |")
    return "\n".join(out)


def configs():
    out = ["### BASELINE configs 1-2 (1D)\n"]
    for proto in ("M", "P"):
        for mode in ("hier", "classic"):
            kw = dict(mode=mode, tile=32, k=16) if mode == "hier" else dict(mode="classic")
            r = solve(1, 256, 1e-8, protocol=proto, **kw)
            out.append(f"- cfg1 N=256 protocol {proto} {mode}: {r['cycles']} cycles, "
                       f"{r['seconds_solve']*1e3:.1f} ms solve, {r['seconds_total']*1e3:.1f} ms total")
    out.append("\n| cfg2 N=2^20, T=1024 | k | cycles to 1e-4 | ms | us/cycle | cell-updates/s |\n|---|---|---|---|---|---|")
    n = 1 << 20
    for k in (1, 4, 16, 64):
        r = solve(1, n, 1e-4, mode="hier", tile=1024, k=k)
        out.append(f"| hier | {k} | {r['cycles']} | {r['seconds_solve']*1e3:.1f} | "
                   f"{r['seconds_solve']/r['cycles']*1e6:.2f} | {n*k*r['cycles']/r['seconds_solve']:.3e} |")
    r = solve(1, n, 1e-4, mode="classic")
    out.append(f"| classic | 1 | {r['cycles']} | {r['seconds_solve']*1e3:.1f} | "
               f"{r['seconds_solve']/r['cycles']*1e6:.2f} | {n*r['cycles']/r['seconds_solve']:.3e} |")
    return "\n".join(out)


if __name__ == "__main__":
    parts = ["# Paper experiments on one B200 (fp64, protocol P)\n"]
    fns = [configs, table_2d, table_1d]
    if len(sys.argv) > 1:
        fns = [f for f in fns if f.__name__ in sys.argv[1:]]
    for fn in fns:
        t0 = time.time()
        parts.append(fn())
        parts.append(f"\n_({fn.__name__}: {time.time()-t0:.0f} s)_\n")
        print(parts[-2], flush=True)
    os.makedirs("gpurun_out", exist_ok=True)
    tag = "_".join(sys.argv[1:]) or "all"
    open(f"gpurun_out/paper_tables_{tag}.md", "w").write("\n".join(parts) + "\n")
