"""Determinism and sharding invariance on the GPU: identical inputs give
bit-identical outputs across runs; processing a batch in chunk-aligned shards (what each
rank does under torchrun) gives exactly the bytes of the unsharded launch; the int64 film
of a sharded flare equals the unsharded film bit for bit (so the NCCL all-reduce of
per-rank films is exact)."""
import numpy as np
import pytest

from plt_inputs import configs as C
from plt_inputs import rays as R

pytestmark = pytest.mark.gpu


def _run(plt, fn, rays_np, n):
    import torch
    d = plt.rays_to_device(rays_np)
    h = plt.alloc_hits(n)
    fn(d, h)
    torch.cuda.synchronize()
    return {k: (v.cpu().numpy().copy() if v is not None else None) for k, v in h.items()}


def test_trace_and_map_bit_identical_reruns(gpu_lib):
    plt = gpu_lib
    cfg = C.CONFIGS["C2"]
    n = (1 << 20) + 77
    rays = R.gen_rays(cfg["law"], 13, 0, n)
    lens = plt.Lens(C.lens_text("C2"), **cfg["opts"])
    pid = lens.all_t_id()
    m = plt.Map(C.map_blob("C2", pid))
    for fn in (lambda d, h: plt.trace_rays(lens, pid, d, h),
               lambda d, h: plt.trace_rays(lens, pid, d, h, precision=plt.FP64),
               lambda d, h: plt.eval_map(m, d, h)):
        a = _run(plt, fn, rays, n)
        b = _run(plt, fn, rays, n)
        for k in a:
            if a[k] is not None:
                assert np.array_equal(a[k], b[k]), k


def test_sharded_equals_unsharded(gpu_lib):
    """Chunk-aligned shards (ranks) reproduce the unsharded outputs exactly."""
    import torch
    plt = gpu_lib
    cfg = C.CONFIGS["C2"]
    n = 4 << 20
    rays = R.gen_rays(cfg["law"], cfg["seed"], 0, n)
    lens = plt.Lens(C.lens_text("C2"), **cfg["opts"])
    pid = lens.all_t_id()
    m = plt.Map(C.map_blob("C2", pid))
    for fn in (lambda d, h: plt.trace_rays(lens, pid, d, h), lambda d, h: plt.eval_map(m, d, h)):
        whole = _run(plt, fn, rays, n)
        for ws in (2, 4):
            per = n // ws
            for r in range(ws):
                part = R.gen_rays(cfg["law"], cfg["seed"], r * per, per)
                got = _run(plt, fn, part, per)
                for k in ("px", "py", "dx", "dy", "dz", "throughput"):
                    assert np.array_equal(got[k], whole[k][r * per:(r + 1) * per]), (k, ws, r)
                assert np.array_equal(got["mask_bits"], whole["mask_bits"][r * per // 32:(r + 1) * per // 32])


def test_flare_film_sharding_is_exact(gpu_lib):
    """Sum of per-shard int64 films == unsharded film (the all-reduce is exact)."""
    import torch
    plt = gpu_lib
    cfg = C.CONFIGS["C4_22"]
    lens = plt.Lens(C.lens_text("C4_22"), **cfg["opts"])
    fd = cfg["film"]
    npx = 3 * fd["height_px"] * fd["width_px"]
    n = 1 << 20
    ghosts = lens.enumerate_ghosts(2)[0][1:6]

    def film_of(start, count):
        film = torch.zeros(npx, dtype=torch.int64, device="cuda")
        for c in range(3):
            rays = plt.rays_to_device(C.flare_rays("C4_22", c, start, count))
            ch = torch.full((count,), c, dtype=torch.uint8, device="cuda")
            h = plt.alloc_hits(count)
            for g in ghosts:
                plt.trace_rays(lens, int(g), rays, h, precision=plt.FP64)
                plt.splat_sensor(fd, film, h, channel=ch, weight_scale=1.0 / n)
        torch.cuda.synchronize()
        return film.cpu().numpy()

    whole = film_of(0, n)
    half = n // 2
    assert np.array_equal(film_of(0, half) + film_of(half, half), whole)
    assert whole.sum() > 0
