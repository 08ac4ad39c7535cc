"""Summarise ncu artefacts (gpurun_out/) into profiles/ (markdown + json).

    python scripts/ncu_summary.py <round-tag>
"""
import collections
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")
KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe active % (of active cycles)"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("smsp__warps_active.avg.per_cycle_active", "warps active per scheduler"),
    ("smsp__warps_eligible.avg.per_cycle_active", "warps eligible per scheduler"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__block_size", "block size"),
    ("launch__grid_size", "grid size"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
     "shared-memory pipe utilisation % (LDS/STS + SHFL wavefronts)"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak (ncu)"),
    ("smsp__inst_executed_op_shfl.sum", "SHFL executed"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (v, u) for h, u, v in zip(hdr, units, vals)}


def to_bytes(v, u):
    f = float(v.replace(",", ""))
    return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(u, 1)


def kernel_summary(rep, title, lines):
    d = raw(rep)
    lines.append(f"## {title}\n\nSource: `{os.path.basename(rep)}` (`ncu --set full --clock-control none`, one launch)\n")
    lines.append("| metric | value |\n|---|---|")
    for k, name in KEYS:
        if k in d:
            v, u = d[k]
            lines.append(f"| {name} (`{k}`) | {v} {u} |")
    stalls = []
    for k, (v, u) in d.items():
        if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
            try:
                x = float(v)
            except ValueError:
                continue
            if x >= 0.03:
                stalls.append((x, k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
    lines.append("\nWarp stall reasons (cycles per issued instruction, >= 0.03):\n")
    lines.append("| reason | per issue |\n|---|---|")
    for x, n in sorted(stalls, reverse=True):
        lines.append(f"| {n} | {x:.3f} |")
    lines.append("")
    return to_bytes(*d["dram__bytes_read.sum"]), to_bytes(*d["dram__bytes_write.sum"])


def launches(csvpath, lines):
    rows = [r for r in csv.reader(open(csvpath)) if len(r) > 5]
    hdr, data = rows[0], rows[1:]
    iK, iV, iU = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    scale = {"ns": 1e-3, "us": 1, "ms": 1e3, "nsecond": 1e-3, "usecond": 1, "msecond": 1e3}
    per = collections.defaultdict(list)
    for r in data:
        v = float(r[iV].replace(",", "")) * scale.get(r[iU], 1)
        per[r[iK].split("(")[0].replace("void ", "")[:70]].append(v)
    lines.append("## Launch list of the bench step (`ncu --metrics gpu__time_duration.sum --clock-control none`)\n")
    lines.append("Cold-cache, serialised per-launch times: compare shares, not absolutes.  Cycle-kernel launches")
    lines.append("far below the median are post-convergence no-ops / residual-only passes of the e2e calls.\n")
    lines.append("| kernel | launches | median µs | share of listed time |\n|---|---|---|---|")
    tot = sum(sum(v) for v in per.values())
    for k, v in sorted(per.items(), key=lambda x: -sum(x[1])):
        v2 = sorted(v)
        lines.append(f"| `{k}` | {len(v)} | {v2[len(v2) // 2]:.1f} | {sum(v) / tot * 100:.1f}% |")
    lines.append("")
    # the bench step itself (k = 16): cycle kernel + rowsum + finalize
    import statistics as st
    vals = []
    for r in data:
        vals.append((r[iK], float(r[iV].replace(",", "")) * scale.get(r[iU], 1)))
    k16 = [v for k, v in vals if "reg2d_kernel" in k and v > 1500]
    rs = [v for k, v in vals if "rowsum_kernel" in k]
    fz = [v for k, v in vals if "finalize_kernel" in k]
    if k16 and rs and fz:
        a, b, c = st.median(k16), st.median(rs), st.median(fz)
        lines.append(f"Bench step (k = 16; the launch list also holds the k = 1 / k = 4 load-store probes, the classic "
                     f"comparison and the multigrid leg): cycle kernel {a:.1f} µs + rowsum {b:.1f} µs + finalize "
                     f"{c:.1f} µs — the cycle kernel is {100 * a / (a + b + c):.1f}% of the step.\n")


if __name__ == "__main__":
    tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
    os.makedirs(P, exist_ok=True)
    lines = [f"# ncu summary — {tag}\n",
             "Workload: bench.py default (2D Poisson 16384², fp64, 32×32 tiles, k = 16, paper protocol).\n"]
    j = {}
    if os.path.exists(os.path.join(G, "launches.csv")):
        launches(os.path.join(G, "launches.csv"), lines)
        subprocess.run(["cp", os.path.join(G, "launches.csv"), os.path.join(P, f"{tag}_launches.csv")])
    for rep, title, key in [("prof_reg2d.ncu-rep", "Cycle kernel `reg2d_kernel<double>` (hot path)", "cycle"),
                            ("prof_classic2d.ncu-rep", "Classic sweep `classic2d_kernel<double>` (comparison)", "classic")]:
        p = os.path.join(G, rep)
        if os.path.exists(p):
            rd, wr = kernel_summary(p, title, lines)
            j[key] = {"dram_bytes_read": rd, "dram_bytes_write": wr, "dram_bytes_per_launch": rd + wr,
                      "algorithmic_bytes_per_launch": 24 * 16384 * 16384, "source": rep}
    open(os.path.join(P, f"{tag}_ncu_summary.md"), "w").write("\n".join(lines) + "\n")
    if "cycle" in j:
        json.dump(dict(j["cycle"], round=tag), open(os.path.join(P, "ncu_cycle_kernel.json"), "w"), indent=1)
    json.dump(j, open(os.path.join(P, f"{tag}_ncu_kernels.json"), "w"), indent=1)
    print("\n".join(lines))
