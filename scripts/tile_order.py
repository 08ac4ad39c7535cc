"""Experiment: REG2D's tile traversal order (HJ_TILE_STRIP = column strips of S tiles; 0 = row-major) vs the
cycle time at 16384^2 and 32768^2, k in {1, 4, 16} (f64, 32x32).  Each setting in a fresh process (the
library reads the variable once).  Prints one line per setting."""
import json, os, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CODE = r'''
import json, os, sys, torch
sys.path.insert(0, os.environ["ROOT"])
from paper_2006_16465_b200 import hj
N = int(os.environ["N"]); dev = torch.device("cuda:0"); s = torch.cuda.Stream(dev)
f = torch.ones(N * N, dtype=torch.float64, device=dev); x0 = torch.ones(N * N, dtype=torch.float64, device=dev)
out = {}
for k in (1, 4, 16):
    p = hj.Plan(2, N, N, 1.0 / (N + 1), f, None, x0, stream=s.cuda_stream, tile=(32, 32), k=k, tol=0.0, max_cycles=1 << 62)
    p.run(3, timed=True)
    out[k] = p.run(12, timed=True) / 12
    p.close()
print(json.dumps(out))
'''
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
for N in (16384, 32768):
    for S in (0, 4, 16, 64):
        env = dict(os.environ, ROOT=ROOT, N=str(N), HJ_TILE_STRIP=str(S))
        r = subprocess.run([sys.executable, "-c", CODE], env=env, capture_output=True, text=True, timeout=600)
        try:
            d = json.loads(r.stdout.strip().splitlines()[-1])
        except Exception:
            print(N, S, "failed", r.stderr[-500:]); continue
        fr = {k: round(24 * N * N / (v * 1e-3) / 1e9 / peak, 3) for k, v in d.items()}
        print(f"N={N} strip={S}: ms {d}  HBM frac {fr}", flush=True)
