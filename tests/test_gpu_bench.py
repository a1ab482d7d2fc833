"""bench.py contract on the GPU: the JSON line's keys (task contract + roofline / cpu_baseline / e2e /
clocks / gpu_launches), and the multi-rank path (barrier, max-over-ranks timing, eigenvalue all-gather)
exercised with two ranks sharing the box's GPU over gloo (functional test, not a scaling number)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"]


def _last_json(out):
    return json.loads(out.strip().splitlines()[-1])


def test_bench_json_contract_small_workload():
    r = subprocess.run([sys.executable, "bench.py", "--workload", "C3", "--steps", "3", "--warmup", "3",
                        "--e2e-steps", "1"], cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    d = _last_json(r.stdout)
    for k in KEYS:
        assert k in d, k
    assert d["value"] > 0 and d["n_gpus"] == 1 and d["dtype"] == "f64"
    roof = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in roof
    assert 0 < roof["frac"] < 1.5
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0
    assert all(s == 0 for s in d["status"])


def test_bench_two_ranks_shared_gpu_gloo():
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29533", "bench.py", "--gpus", "2", "--workload", "C3",
           "--steps", "2", "--warmup", "3", "--dist-backend", "gloo", "--e2e-steps", "1", "--no-cpu-baseline"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    d = _last_json(r.stdout)
    assert d["n_gpus"] == 2 and d["gathered_rows"] == 4
    assert d["value"] > 0 and d["e2e"]["value"] > 0
