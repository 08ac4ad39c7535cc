"""Split a kernel's warp-stall samples by code region, from an ncu report's SASS source page.

usage: python scripts/ncu_regions.py REPORT.ncu-rep [out.md]

Regions are runs of consecutive SASS instructions with the same execution count: in reg2d the
sub-iteration loop body runs (k - 2) / 2 times per tile, everything else once per tile, so the
loop stands out as the block with the largest count.  Prints samples and the top stall reasons
per region, and the top stalled instructions outside the loop.
"""
import csv
import io
import subprocess
import sys

REASONS = ["stall_barrier", "stall_branch_resolving", "stall_dispatch", "stall_drain", "stall_lg",
           "stall_long_sb", "stall_math", "stall_membar", "stall_mio", "stall_misc", "stall_no_inst",
           "stall_not_selected", "stall_selected", "stall_short_sb", "stall_sleep", "stall_tex",
           "stall_wait"]


def main(rep, out=None):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, data = rows[1], rows[2:]
    i_s, i_e, i_src = (hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed"),
                       hdr.index("Source"))
    ir = {r: hdr.index(r) for r in REASONS if r in hdr}
    total = sum(int(r[i_s] or 0) for r in data)
    groups = []  # [exec count, samples, first, last]
    for idx, r in enumerate(data):
        e, s = int(r[i_e] or 0), int(r[i_s] or 0)
        if groups and groups[-1][0] == e:
            groups[-1][1] += s
            groups[-1][3] = idx
        else:
            groups.append([e, s, idx, idx])
    loop = max(groups, key=lambda g: (g[0], g[1]))
    lines = [f"# Warp-stall samples by code region — `{rep.split('/')[-1]}`", "",
             f"{total} samples, {len(data)} SASS instructions.  Loop body = instructions {loop[2]}–{loop[3]} "
             f"(executed {loop[0]} times).", "",
             "| region (exec count, SASS index range) | samples | share | top stall reasons (samples) |",
             "|---|---|---|---|"]
    for g in groups:
        if g[1] < 0.005 * total:
            continue
        tot = {r: sum(int(x[ir[r]] or 0) for x in data[g[2]:g[3] + 1]) for r in ir}
        top = ", ".join(f"{k[6:]} {v}" for k, v in sorted(tot.items(), key=lambda t: -t[1])[:4])
        tag = " **loop**" if g is loop else ""
        lines.append(f"| {g[0]} ({g[2]}–{g[3]}, {g[3] - g[2] + 1} instr){tag} | {g[1]} | "
                     f"{100 * g[1] / total:.1f}% | {top} |")
    lines += ["", "Top stalled instructions outside the loop:", "", "| samples | index | SASS | top reason |",
              "|---|---|---|---|"]
    outside = sorted(((int(x[i_s] or 0), i, x[i_src].strip()) for i, x in enumerate(data)
                      if not loop[2] <= i <= loop[3]), reverse=True)[:15]
    for s, i, src in outside:
        top = max(ir, key=lambda r: int(data[i][ir[r]] or 0))
        lines.append(f"| {s} | {i} | `{src[:60]}` | {top[6:]} |")
    text = "\n".join(lines) + "\n"
    print(text)
    if out:
        with open(out, "w") as fh:
            fh.write(text)


if __name__ == "__main__":
    main(*sys.argv[1:])
