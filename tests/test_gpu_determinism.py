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


@pytest.mark.parametrize("name,prec", [("C2", 0), ("C3", 0), ("C3", 1)])
def test_results_do_not_depend_on_the_compaction_point(gpu_lib, tmp_path, name, prec):
    """The block compaction only moves rays between lanes: moving it
    (PLT_TRACE_SPLIT_DELTA, read when a path program is compiled -- so in a subprocess) leaves
    every output bit, mask bit and guard-band flag unchanged, fp32 (JIT) and fp64."""
    import os
    import subprocess
    import sys
    import torch
    plt = gpu_lib
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = tmp_path / "moved.npz"
    n = (1 << 17) + 3
    code = f"""
import sys; sys.path.insert(0, {root!r})
import numpy as np, torch
import paper_2605_04017_b200 as plt
from plt_inputs import configs as C, rays as R
cfg = C.CONFIGS[{name!r}]
lens = plt.Lens(C.lens_text({name!r}), **cfg["opts"])
d = plt.rays_to_device(R.gen_rays(cfg["law"], 29, 0, {n}))
h = plt.alloc_hits({n}, flags=True)
plt.trace_rays(lens, lens.all_t_id(), d, h, direction=cfg["direction"], precision={prec})
torch.cuda.synchronize()
np.savez({str(out)!r}, **{{k: h[k].cpu().numpy() for k in plt.HIT_KEYS + ("mask_bits", "flags")}})
"""
    for delta in ("-3", "1"):
        subprocess.run([sys.executable, "-c", code], check=True, env=dict(os.environ, PLT_TRACE_SPLIT_DELTA=delta),
                       timeout=600)
        g = np.load(out)
        cfg = C.CONFIGS[name]
        lens = plt.Lens(C.lens_text(name), **cfg["opts"])
        d = plt.rays_to_device(R.gen_rays(cfg["law"], 29, 0, n))
        h = plt.alloc_hits(n, flags=True)
        plt.trace_rays(lens, lens.all_t_id(), d, h, direction=cfg["direction"], precision=prec)
        torch.cuda.synchronize()
        for k in plt.HIT_KEYS + ("mask_bits", "flags"):
            a = h[k].cpu().numpy()
            assert np.array_equal(a.view(np.uint8), g[k].view(np.uint8)), (delta, k)
