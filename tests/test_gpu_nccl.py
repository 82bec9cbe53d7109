"""The film all-reduce (Eq. 8) over NCCL on the test box: a
one-rank NCCL communicator on the one GPU (NCCL forbids two ranks on one device, so the
multi-rank tests share the GPU over gloo; this one runs the real backend).  A product film
(trace + fitted map, fused splat) all-reduced in int64 SUM is unchanged, twice the film
reduced from a second buffer is exactly twice it, and NCCL's init log names the
communicator (nRanks 1) -- the same calls bench.py makes at N > 1."""
import os
import socket
import subprocess
import sys
import textwrap

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = textwrap.dedent("""
    import os, sys, torch
    import torch.distributed as dist
    sys.path.insert(0, {root!r})
    import paper_2605_04017_b200 as plt
    from plt_inputs import configs as C
    from plt_inputs import rays as R
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", init_method="tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    assert dist.get_backend() == "nccl"
    cfg = C.CONFIGS["C2"]
    n = (1 << 18) + 77
    rays = R.gen_rays(cfg["law"], 7, 0, n)
    lens = plt.Lens(C.lens_text("C2"), **cfg["opts"])
    pid = lens.all_t_id()
    m = plt.Map(C.fitted_map_blob("C2"), lens=lens)
    d = plt.rays_to_device(rays, with_dz=False)
    fd = {{"width_px": 768, "height_px": 512, "channels": 1, "sensor_w_mm": 36.0, "sensor_h_mm": 24.0,
           "center_x_mm": 0.0, "center_y_mm": 0.0}}
    film = torch.zeros(768 * 512, dtype=torch.int64, device="cuda")
    spl = {{"film_desc": fd, "film": film, "weight_scale": 1.0 / n}}
    plt.trace_rays(lens, pid, d, plt.alloc_hits(n), splat=spl)
    plt.eval_map(m, d, plt.alloc_hits(n), splat=spl)
    torch.cuda.synchronize()
    ref = film.clone()
    assert int(ref.sum()) > 0
    dist.all_reduce(film)                       # int64 SUM over the one rank
    twice = torch.zeros_like(film)
    twice.copy_(ref)
    twice.add_(ref)
    dist.all_reduce(twice)
    torch.cuda.synchronize()
    assert torch.equal(film, ref), "NCCL all-reduce changed a one-rank film"
    assert torch.equal(twice, 2 * ref)
    dist.destroy_process_group()
    print("NCCL_FILM_OK", int(ref.sum()))
""")


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_nccl_film_allreduce_one_rank():
    env = dict(os.environ, NCCL_DEBUG="INFO", NCCL_DEBUG_SUBSYS="INIT")
    code = CHILD.format(root=ROOT, port=_port())
    out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0, (out.stdout[-2000:], out.stderr[-3000:])
    assert "NCCL_FILM_OK" in out.stdout
    log = out.stdout + out.stderr
    assert "NCCL INFO" in log and "nRanks 1" in log, log[-3000:]
