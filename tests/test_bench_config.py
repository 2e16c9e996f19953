"""bench.py's workload table is the paper's budget rule as the oracle computes it,
and the reference arm runs (CPU, tiny sample)."""
import json
import os
import subprocess
import sys

import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def test_bench_k_follows_budget_rule():
    dims = [(M, K) for _, M, K, _ in bench.LAYERS]
    assert [k for *_, k in bench.LAYERS] == O.budget_to_k(0.01, dims, 3, "latency")


def test_bench_algorithmic_bytes():
    # 12288^2 3-bit + scale/zero + 15 weak columns + x + y (57.1 MB)
    assert abs(bench.algorithmic_bytes(12288, 12288, 15, 1) / 1e6 - 57.1) < 0.1
    total = sum(bench.algorithmic_bytes(M, K, k, 1) for _, M, K, k in bench.LAYERS)
    assert abs(total / 1e6 - 682.5) < 0.5


def test_reference_arm_prints_one_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--steps", "2", "--warmup", "3", "--ref-rows", "4"],
                       capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr
    lines = [l for l in r.stdout.splitlines() if l.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["unit"] == "GB/s" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["e2e"]["h2d_bytes_per_step"] == 0
