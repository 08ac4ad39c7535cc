"""Quick kernel timing: ms per cycle of the cycle kernel at a given size / k / variant."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2006_16465_b200 import hj

def run(n=16384, k=16, mode="hier", dtype="f64", kernel="auto", steps=20):
    dev = torch.device("cuda:0")
    f = torch.ones(n * n, dtype=torch.float64, device=dev)
    x0 = torch.ones(n * n, dtype=torch.float64, device=dev)
    s = torch.cuda.Stream(dev)
    p = hj.Plan(2, n, n, 1.0 / (n + 1), f, None, x0, stream=s.cuda_stream, mode=mode, tile=(32, 32),
                k=k if mode == "hier" else 1, tol=0.0, max_cycles=1 << 62, kernel=kernel, dtype=dtype)
    p.run(4, timed=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    km = p.run(steps, timed=True)
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    kms = km / steps
    cells = n * n
    out = dict(n=n, k=k, mode=mode, dtype=dtype, kernel=kernel,
               ms_cycle=round(ms, 4), ms_kernel=round(kms, 4),
               gbs=round((24 if dtype == "f64" else 12) * cells / kms / 1e6, 1),
               gupd=round(cells * (k if mode == "hier" else 1) / kms / 1e6, 1))
    print(json.dumps(out), flush=True)
    p.close()

if __name__ == "__main__":
    for spec in sys.argv[1:]:
        kw = dict(kv.split("=") for kv in spec.split(","))
        for key in ("n", "k", "steps"):
            if key in kw: kw[key] = int(kw[key])
        run(**kw)
