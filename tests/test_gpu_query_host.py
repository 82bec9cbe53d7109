"""plt_query_host (the C-ABI host-buffer query: chunked host -> device copies on the
library's copy stream overlapping the kernels, hits and film back to host memory)
produces exactly the hits and film of the device-resident calls on the same rays
(plt_trace_rays_splat / plt_eval_map_splat): int64 film and float hits bit-identical."""
import numpy as np
import pytest

from plt_inputs import configs as C
from plt_inputs import rays as R

pytestmark = pytest.mark.gpu

FILM = {"width_px": 768, "height_px": 512, "channels": 1, "sensor_w_mm": 36.0, "sensor_h_mm": 24.0,
        "center_x_mm": 0.0, "center_y_mm": 0.0}


def _device_reference(plt, lens, pid, m, rays, scale, with_dz):
    import torch
    n = rays["ox"].size
    d = plt.rays_to_device(rays, with_dz=with_dz)
    ht, hm = plt.alloc_hits(n), plt.alloc_hits(n)
    film = torch.zeros(512 * 768, dtype=torch.int64, device="cuda")
    spl = {"film_desc": FILM, "film": film, "weight_scale": scale}
    if lens is not None:
        plt.trace_rays(lens, pid, d, ht, splat=spl)
    if m is not None:
        plt.eval_map(m, d, hm, splat=spl)
    torch.cuda.synchronize()
    return ht, hm, film


@pytest.mark.parametrize("with_dz", [False, True], ids=["20B", "24B"])
@pytest.mark.parametrize("n,chunk", [((1 << 20) + 77, 1 << 18), (5000, 1024), (64, 32), (1000, 1 << 21)])
def test_query_host_matches_device_path(gpu_lib, n, chunk, with_dz):
    import torch
    plt = gpu_lib
    cfg = C.CONFIGS["C2"]
    lens = plt.Lens(C.lens_text("C2"), **cfg["opts"])
    pid = lens.all_t_id()
    m = plt.Map(C.fitted_map_blob("C2"), lens=lens)
    rays = R.gen_rays(cfg["law"], 77, 0, n)
    ht, hm, film_ref = _device_reference(plt, lens, pid, m, rays, 0.5, with_dz)
    host = {k: torch.from_numpy(rays[k]).pin_memory() for k in plt.RAY_KEYS if with_dz or k != "dz"}
    host["plane_z"] = rays["plane_z"]
    out_t, out_m = plt.alloc_host_hits(n), plt.alloc_host_hits(n)
    film = torch.zeros_like(film_ref)
    film_host = torch.empty(film.numel(), dtype=torch.int64).pin_memory()
    plt.query_host(lens, pid, m, host, FILM, film, film_host, host_trace=out_t, host_map=out_m, weight_scale=0.5,
                   chunk=chunk)
    torch.cuda.synchronize()
    assert torch.equal(film_host, film_ref.cpu()) and int(film_host.sum()) > 0
    nw = (n + 31) // 32
    for a, b in ((ht, out_t), (hm, out_m)):
        assert torch.equal(a["mask_bits"][:nw].cpu(), b["mask_bits"][:nw])
        for k in plt.HIT_KEYS:
            assert torch.equal(a[k].cpu(), b[k]), k


def test_query_host_trace_only_map_only_pageable(gpu_lib):
    """Either query alone; pageable (not pinned) host memory; hits without a film."""
    import torch
    plt = gpu_lib
    cfg = C.CONFIGS["C3"]
    lens = plt.Lens(C.lens_text("C3"), **cfg["opts"])
    pid = lens.all_t_id()
    m = plt.Map(C.fitted_map_blob("C3"), lens=lens)
    n = 70_001
    rays = R.gen_rays(cfg["law"], 5, 0, n)
    d = plt.rays_to_device(rays, with_dz=False)
    ht, hm = plt.alloc_hits(n), plt.alloc_hits(n)
    plt.trace_rays(lens, pid, d, ht, direction=plt.BACKWARD)
    plt.eval_map(m, d, hm)
    host = {k: torch.from_numpy(rays[k]) for k in plt.RAY_KEYS if k != "dz"}
    host["plane_z"] = rays["plane_z"]
    out_t, out_m = plt.alloc_host_hits(n, pin=False), plt.alloc_host_hits(n, pin=False)
    plt.query_host(lens, pid, None, host, host_trace=out_t, chunk=4096, direction=plt.BACKWARD)
    plt.query_host(None, 0, m, host, host_map=out_m, chunk=8192)
    torch.cuda.synchronize()
    nw = (n + 31) // 32
    for a, b in ((ht, out_t), (hm, out_m)):
        assert torch.equal(a["mask_bits"][:nw].cpu(), b["mask_bits"][:nw])
        for k in plt.HIT_KEYS:
            assert torch.equal(a[k].cpu(), b[k]), k


def test_query_host_flare_channels(gpu_lib):
    """A flare ghost in fp64 over three channels: the device channel array is indexed like
    the host rays across chunks."""
    import torch
    plt = gpu_lib
    cfg = C.CONFIGS["C4_22"]
    lens = plt.Lens(C.lens_text("C4_22"), **cfg["opts"])
    fd = cfg["film"]
    per = 40_000
    parts = [C.flare_rays("C4_22", c, 0, per) for c in range(3)]
    rays = {k: np.concatenate([p[k] for p in parts]) for k in plt.RAY_KEYS}
    rays["plane_z"] = parts[0]["plane_z"]
    n = 3 * per
    ch = torch.from_numpy(np.repeat(np.arange(3, dtype=np.uint8), per)).cuda()
    d = plt.rays_to_device(rays)
    h = plt.alloc_hits(n)
    ref = torch.zeros(3 * 512 * 768, dtype=torch.int64, device="cuda")
    plt.trace_rays(lens, 65616, d, h, precision=plt.FP64,
                   splat={"film_desc": fd, "film": ref, "channel": ch, "weight_scale": 1.0 / per})
    host = {k: torch.from_numpy(rays[k]).pin_memory() for k in plt.RAY_KEYS}
    host["plane_z"] = rays["plane_z"]
    film = torch.zeros_like(ref)
    fh = torch.empty(film.numel(), dtype=torch.int64).pin_memory()
    plt.query_host(lens, 65616, None, host, fd, film, fh, weight_scale=1.0 / per, chunk=1 << 15,
                   precision=plt.FP64, channel=ch)
    torch.cuda.synchronize()
    assert torch.equal(fh, ref.cpu()) and int(fh.sum()) > 0
