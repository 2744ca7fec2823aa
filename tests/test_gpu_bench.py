"""The bench arms run end to end on one GPU and print the contract's JSON line:
the single-GPU arm, the row-partitioned arm with one rank (NCCL identity), and
two ranks on one GPU through the host-staged communicator (--comm host)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, timeout=600):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True, text=True,
                       timeout=timeout, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


KEYS = ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "e2e", "gpu_launches", "roofline", "clocks")


def test_bench_single_gpu_line():
    d = _run(["--workload", "0", "--steps", "3", "--warmup", "3", "--no-cpu"])
    for k in KEYS:
        assert k in d, k
    assert d["n_gpus"] == 1 and d["value"] > 0 and d["gpu_launches"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0


def test_bench_dist_one_rank():
    d = _run(["--dist", "--workload", "0", "--steps", "2", "--warmup", "3"])
    for k in KEYS:
        assert k in d, k
    assert d["scaling"] == "strong" and d["config"]["mode"].startswith("row-partitioned")
    assert d["roofline"]["nvlink"]["bytes_per_step_received"] == 0.0


def test_bench_two_ranks_host_comm():
    d = _run(["--gpus", "2", "--comm", "host", "--workload", "0", "--steps", "1", "--warmup", "3"])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong"
    assert len(d["per_rank"]) == 2 and all(r["bytes"] > 0 for r in d["per_rank"])
    b = d["config"]["bounds"]
    assert b[0] == 0 and b[-1] == d["config"]["n"] and b[0] < b[1] < b[2]
