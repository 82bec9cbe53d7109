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


def _bench(args, ranks, tmp_env=None):
    env = dict(os.environ, PLT_BENCH_SHARE_GPU="1", **(tmp_env or {}))
    if ranks == 1:
        cmd = [sys.executable, os.path.join(ROOT, "bench.py")] + args
    else:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(ranks),
               "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "bench.py")] + args
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=1200)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


@pytest.mark.parametrize("cfg", ["C4_22", "C4_59"])
def test_flare_image_two_ranks_equals_one_rank_bitwise(tmp_path, cfg):
    """the flare image sharded over (channel, ghost, ray) ranges on two ranks
    and all-reduced (int64 SUM, Eq. 8) is bit-identical to the one-rank image -- through the
    product path (plt_trace_paths fp64 + plt_eval_map_splat, bench.py --config)."""
    import numpy as np
    f1, f2 = tmp_path / "one.npy", tmp_path / "two.npy"
    d1 = _bench(["--config", cfg, "--steps", "1", "--warmup", "3", "--no-cpu-baseline", "--dump-film", str(f1)], 1)
    d2 = _bench(["--gpus", "2", "--config", cfg, "--steps", "1", "--warmup", "3", "--dump-film", str(f2)], 2)
    a, b = np.load(f1), np.load(f2)
    assert a.shape == b.shape and int(a.sum()) > 0
    assert np.array_equal(a, b)
    assert d1["scaling"] == d2["scaling"] == "strong" and d2["n_gpus"] == 2
    assert d1["config"]["rays_total"] == d2["config"]["rays_total"] == d2["config"]["rays_per_gpu"] * 2
    assert d2["kernels"]["film_allreduce"]["bytes"] == a.size * 8


def test_c3_two_ranks_json_contract():
    """C3 strong scaling by pixel rows: two ranks each own 64 of the 128 rows."""
    d = _bench(["--gpus", "2", "--config", "C3", "--steps", "1", "--warmup", "3"], 2)
    assert d["scaling"] == "strong" and d["config"]["rays_total"] == 805_306_368
    assert d["config"]["rays_per_gpu"] == 805_306_368 // 2 and "64 pixel rows" in d["config"]["parallelism"]
    assert d["value"] > 0 and d["roofline"]["kernel"] in ("trace_rays", "eval_map")
