"""The bench's reference arm (the CPU oracle, this tier's reference) prints one JSON line with the
contract's keys — CPU only, on a small grid so it runs in seconds."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "2",
                          "--warmup", "1", "--grid", "512"], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["value"] > 0 and d["steps"] == 2
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] == 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert "workload" in d["config"]


def test_ncu_traffic_scales_to_the_rank_slab():
    """roofline.traffic is the committed ncu figure of one full 16384^2 launch; a row slab's launch
    (N > 1) reports its share of it, other configurations report none."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    b = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(b)
    full = json.load(open(os.path.join(ROOT, "profiles", "ncu_cycle_kernel.json")))["dram_bytes_per_launch"]
    n = b.N_GRID
    t1, basis1 = b.ncu_traffic(n, b.K_SUB, "hier", n * n)
    assert t1 == full and "scaled" not in basis1
    t2, basis2 = b.ncu_traffic(n, b.K_SUB, "hier", n * n // 2)
    assert t2 == full / 2 and "scaled" in basis2
    assert b.ncu_traffic(2048, b.K_SUB, "hier", 2048 * 2048) == (None, None)
    assert b.ncu_traffic(n, 4, "hier", n * n) == (None, None)
    assert b.ncu_traffic(n, b.K_SUB, "classic", n * n) == (None, None)
