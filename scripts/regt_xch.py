"""A/B of the large REGT tiles' exchange mode (HJ_REGT_XCH: 0 mbarriers + branchy sends, 2 one named
barrier per sub-iteration + predicated sends, 3 mbarriers + predicated sends): per-cycle time at
16384^2 and 32768^2, f64, k in {1, 4, 16}, and the iterate after 3 cycles compared with mode 0.
Each mode in a fresh process (the library reads the variable once).  -> gpurun_out/regt_xch.json"""
import json, os, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CODE = r'''
import json, os, sys, hashlib, torch
sys.path.insert(0, os.environ["ROOT"])
from paper_2006_16465_b200 import hj
dev = torch.device("cuda:0"); s = torch.cuda.Stream(dev)
out = {}
for N in (16384, 32768):
    g = torch.Generator(device=dev); g.manual_seed(7)
    f = torch.rand(N * N, dtype=torch.float64, device=dev, generator=g)
    x0 = torch.rand(N * N, dtype=torch.float64, device=dev, generator=g)
    for tile in ((64, 32), (32, 64), (64, 64), (128, 32)):
        for k in (1, 4, 16):
            p = hj.Plan(2, N, N, 1.0 / (N + 1), f, None, x0, stream=s.cuda_stream, tile=tile, k=k, tol=0.0,
                        max_cycles=1 << 62)
            p.run(3, timed=True)
            ms = p.run(10, timed=True) / 10
            d = None
            if N == 16384 and k == 4:
                q = hj.Plan(2, N, N, 1.0 / (N + 1), f, None, x0, stream=s.cuda_stream, tile=tile, k=k, tol=0.0,
                            max_cycles=3)
                r = q.solve()
                d = hashlib.sha1(r["x"].cpu().numpy().tobytes()).hexdigest()[:16]
                q.close()
            p.close()
            out[f"{N} {tile[0]}x{tile[1]} k={k}"] = [round(ms, 4), round(24 * N * N / (ms * 1e-3) / 1e9, 1), d]
print(json.dumps(out))
'''
res = {}
for m in ("0", "2", "3"):
    env = dict(os.environ, ROOT=ROOT, HJ_REGT_XCH=m)
    r = subprocess.run([sys.executable, "-c", CODE], env=env, capture_output=True, text=True, timeout=900)
    try:
        res[m] = json.loads(r.stdout.strip().splitlines()[-1])
    except Exception:
        print(m, "failed", r.stderr[-800:], flush=True)
        continue
    print("mode", m, json.dumps(res[m]), flush=True)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/regt_xch.json", "w"), indent=1)
if "0" in res:
    for key in res["0"]:
        print(key, " | ".join(f"m{m} {res[m][key][0]} ms {res[m][key][1]} GB/s" + (" same" if res[m][key][2] == res["0"][key][2] else " DIFF")
                             for m in res if key in res[m]))
