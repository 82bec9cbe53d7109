"""Functional check of bench.py's multi-rank path (the driver's N-GPU scaling run): two
ranks launched by torch.distributed.run exactly as the driver does, sharing the one GPU of
the test box through the PLT_BENCH_SHARE_GPU knob (gloo film all-reduce; the ranks'
kernels never wait on each other).  Only the contract of the JSON line is checked --
numbers from ranks sharing a GPU are not measurements."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_bench_two_ranks_json_contract():
    env = dict(os.environ, PLT_BENCH_SHARE_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "3", "--warmup", "3", "--rays", str(1 << 20)]
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]          # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["steps"] == 3 and d["warmup"] == 3 and d["scaling"] == "weak"
    assert d["config"]["parallelism"] == "dp2 over rays" and "2^20 rays per GPU" in d["config"]["workload"]
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and "cpu_baseline" not in d
