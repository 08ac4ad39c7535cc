"""Summarise the multigrid ncu captures (gpurun_out/prof_mg_*.ncu-rep) into profiles/<tag>_ncu_mg.md.

    python scripts/ncu_mg_summary.py r01
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_summary import G, P, kernel_summary  # noqa: E402

tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
lines = [f"# ncu summary — multigrid kernels ({tag})\n",
         "Workload: `scripts/mg_launches.py` (2D Poisson 16383², fp64, V(1,1), 32×32 smoother tiles, k = 4).\n",
         "Algorithmic bytes: restriction 16 B per fine cell read (x, q) + 2 B written (coarse q) = 4.83 GB;",
         "fused post-smoothing cycle 24 B per fine cell + 2 B coarse patch = 6.98 GB.\n"]
for rep, title in [("prof_mg_restrict.ncu-rep", "Fine-level restriction `mg_restrict2d_stream<double>`"),
                   ("prof_mg_post.ncu-rep", "Fine-level post-smoothing with the fused correction `reg2d_kernel<double, …, SK=2, COR=1>`")]:
    p = os.path.join(G, rep)
    if os.path.exists(p):
        rd, wr = kernel_summary(p, title, lines)
        lines.append(f"DRAM bytes per launch: {(rd + wr) / 1e9:.3f} GB\n")
open(os.path.join(P, f"{tag}_ncu_mg.md"), "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
