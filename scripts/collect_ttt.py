"""Collect the time-to-1e-6 chain's per-call logs (gpurun_out/ttt_1e-06_16384_<time>.jsonl, one per lease)
into profiles/: the summary (ttt_1e-06_16384.json, written by scripts/ttt_1e6.py when the solve
converges) and the merged per-segment trajectory of the chain that produced it (the calls that resumed
from one another, newest back to the call that started at cycle 0).
    python scripts/collect_ttt.py"""
import glob
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "gpurun_out")
calls = []
for f in sorted(glob.glob(os.path.join(G, "ttt_1e-06_16384_*.jsonl"))):
    L = [json.loads(l) for l in open(f) if l.strip()]
    head = next((d for d in L if "resumed_at" in d), {})
    recs = [d for d in L if "cycles" in d]
    if recs:
        calls.append((os.path.basename(f), head.get("resumed_at", 0), recs))
# walk back from the newest call along resumed_at == previous call's last cycle count
chain = [calls[-1]]
while chain[0][1] != 0:
    prev = [c for c in calls if c[2][-1]["cycles"] == chain[0][1] and c[0] < chain[0][0]]
    if not prev:
        break
    chain.insert(0, prev[-1])
traj = [r for c in chain for r in c[2]]
out = {"calls": [c[0] for c in chain], "complete_from_zero": chain[0][1] == 0, "trajectory": traj}
summ = os.path.join(G, "ttt_1e-06_16384.json")
if os.path.exists(summ):
    out["summary"] = json.load(open(summ))
json.dump(out, open(os.path.join(ROOT, "profiles", "r02_ttt_1e-6_16384_chain.json"), "w"), indent=1)
if "summary" in out and out["summary"].get("converged"):
    s = dict(out["summary"])
    s["chain_calls"] = out["calls"]
    s["trajectory_file"] = "profiles/r02_ttt_1e-6_16384_chain.json"
    json.dump(s, open(os.path.join(ROOT, "profiles", "r02_ttt_1e-6_16384.json"), "w"), indent=1)
print(out["calls"], out["complete_from_zero"], traj[-1], "summary" in out)
