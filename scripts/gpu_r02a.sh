#!/bin/bash
# round 2: full GPU suite (the streamed-head REG2D kernel is now the default path), A/B of the cycle
# kernel, the L2 roofline of configs 2/3, a small-size check of the time-to-1e-6 script
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log; tail -3 gpurun_out/pytest_gpu.log
for v in 1 0 1 0; do
  HJ_REG2D_STREAM=$v timeout 300 python bench.py --ttt 0 --no-cpu --no-mg --steps 100 > gpurun_out/ab_stream$v.log 2>&1
  python - "$v" <<'PY'
import json, sys
l = [x for x in open(f"gpurun_out/ab_stream{sys.argv[1]}.log") if x.startswith("{")]
d = json.loads(l[-1]) if l else {}
r = d.get("roofline", {})
print("stream", sys.argv[1], "ms/step", round(d.get("ms_per_step", 0), 4), "kernel_ms", round(r.get("kernel_ms", 0), 4), "frac", round(r.get("frac", 0), 3), "ls", {k: round(v["kernel_ms"], 3) for k, v in (r.get("load_store_phase") or {}).items()})
PY
done
timeout 600 python scripts/l2_roofline.py > gpurun_out/l2_roofline.log 2>&1; tail -8 gpurun_out/l2_roofline.log
TTT_N=256 TTT_SEG=700 timeout 300 python scripts/ttt_1e6.py > gpurun_out/ttt_small.log 2>&1; tail -2 gpurun_out/ttt_small.log
python - <<'PY'
import numpy as np
from paper_2006_16465_b200 import hj
from paper_2006_16465_b200.inputs import make_problem
p = make_problem("P", 2, 256)
r = hj.jacobi_solve(2, 256, 256, p["h"], p["f"], p["bc"], p["x0"], tile=(32, 32), k=16, tol=1e-6, max_cycles=10**7, history=False)
print("unsegmented 256^2 cycles to 1e-6:", r["cycles"])
PY
