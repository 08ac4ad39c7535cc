"""The bench's N > 1 path (torchrun, one process per rank, row slabs, peer-memory transport, max over
ranks, one JSON line from rank 0) exercised on a one-GPU box: HJ_BENCH_ONE_GPU=1 puts both ranks on
cuda:0 with a gloo process group (bench.py).  Timings of this mode are meaningless; the test checks
that the path runs end to end and that the line keeps the contract."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

pytestmark = pytest.mark.gpu


def test_bench_two_ranks_one_gpu():
    env = dict(os.environ, HJ_BENCH_ONE_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29531", os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "5", "--warmup", "3", "--grid", "2048", "--ttt", "1e-2",
           "--no-cpu", "--no-mg"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["steps"] == 5 and d["warmup"] == 3 and d["value"] > 0
    assert d["config"]["parallelism"] == "row-slab x2"
    assert "peer" in d["config"]["transport"]
    assert d["gpu_launches"] > 0
    assert d["roofline"]["bound"] == "hbm" and d["roofline"]["traffic"] is None  # not the ncu config
    assert d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0
    # the N > 1 self-check: both transports' slabs vs the oracle and the one-GPU solve (NCCL cannot run
    # with two ranks on one GPU and reports itself skipped)
    pc = d["parity_check"]
    assert pc["peer"] is True, pc
    assert isinstance(pc["nccl"], str) and pc["nccl"].startswith("skipped")
