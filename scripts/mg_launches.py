"""Run a few multigrid V-cycles at 16383^2 (for an ncu launch list / full capture).

    ncu --metrics gpu__time_duration.sum --clock-control none --csv python scripts/mg_launches.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2006_16465_b200 import hj
from paper_2006_16465_b200.inputs import make_problem

n = int(os.environ.get("HJ_N", "16383"))
k = int(os.environ.get("HJ_K", "4"))
p = make_problem("P", 2, n)
dev = torch.device("cuda", 0)
t = lambda a: torch.as_tensor(a, device=dev)
plan = hj.Plan(2, n, n, p["h"], t(p["f"]), t(p["bc"]), t(p["x0"]), mode="mg", tile=(32, 32), k=k, tol=0.0,
               max_cycles=100)
plan.run(int(os.environ.get("HJ_VC", "2")), timed=True)
torch.cuda.synchronize()
print("launches per V-cycle", plan.launches_per_cycle())
