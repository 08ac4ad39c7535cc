"""The CPU oracle timed on this host (single-threaded, as it stands) on the small BASELINE configs,
next to the GPU numbers of profiles/r01_paper_tables.md.  Prints markdown.

    python scripts/oracle_times.py > profiles/r01_oracle_times.md
"""
import os
import platform
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle
from paper_2006_16465_b200.inputs import make_problem


def t(fn):
    t0 = time.perf_counter()
    r = fn()
    return r, time.perf_counter() - t0


def main():
    oracle.build()
    cpu = "unknown"
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                cpu = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    out = [f"# CPU oracle timings ({cpu}, {os.cpu_count()} logical cores; the oracle uses 1)\n",
           f"host: {platform.node()}\n",
           "| case | solver | cycles | seconds |", "|---|---|---|---|"]
    for proto in ("M", "P"):
        p = make_problem(proto, 1, 256)
        for mode, kw in (("hier", dict(tile=32, k=16)), ("classic", dict(k=1))):
            r, s = t(lambda: oracle.solve(1, 256, 1, p["h"], p["f"], p["bc"], p["x0"], mode=mode, tol=1e-8,
                                          max_cycles=10**7, history=False, **kw))
            out.append(f"| cfg1 1D N=256 protocol {proto}, tol 1e-8 | {mode} | {r['cycles']} | {s:.2f} |")
    p = make_problem("P", 2, 1024)
    r, s = t(lambda: oracle.solve(2, 1024, 1024, p["h"], p["f"], p["bc"], p["x0"], mode="hier", tile=(32, 32), k=16,
                                  tol=0.0, max_cycles=3, history=False))
    out.append(f"| cfg3 2D 1024², k=16 (3 cycles; 20,153 to 1e-4 ⇒ ≈ {s / 3 * 20153 / 60:.0f} min projected) "
               f"| hier | 3 | {s:.2f} |")
    p = make_problem("P", 2, 1023)
    r, s = t(lambda: oracle.solve_mg(2, 1023, 1023, p["h"], p["f"], p["bc"], p["x0"], tile=(32, 32), k=4,
                                     tol=1e-6, max_cycles=100, history=False))
    out.append(f"| 2D 1023² to 1e-6 | multigrid V(1,1), k=4 | {r['cycles']} | {s:.2f} |")
    print("\n".join(out))


if __name__ == "__main__":
    main()
