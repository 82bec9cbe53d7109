"""Fused query + splat (plt_trace_rays_splat / plt_eval_map_splat): the film splatted inside
the trace / regressor epilogues is bit-identical to the query followed by plt_splat_sensor
on its hits, and the hits are unchanged; covers the fp32 trace with its fp64 guard-band
refine, the fp64 ghost trace with channels, and eval_map with fitted weights."""
import numpy as np
import pytest

from plt_inputs import configs as C
from plt_inputs import rays as R

pytestmark = pytest.mark.gpu

FILM = C.CONFIGS["C4_22"]["film"]     # 768 x 512 x 3 over 24 x 16 mm


def _films(plt, run, n, channel=None, scale=1.0, flags=True):
    import torch
    npx = FILM["channels"] * FILM["height_px"] * FILM["width_px"]
    f_sep = torch.zeros(npx, dtype=torch.int64, device="cuda")
    f_fused = torch.zeros(npx, dtype=torch.int64, device="cuda")
    d_sep = torch.zeros(1, dtype=torch.int64, device="cuda")
    d_fused = torch.zeros(1, dtype=torch.int64, device="cuda")
    h1, h2 = plt.alloc_hits(n, flags=flags), plt.alloc_hits(n, flags=flags)
    run(h1, None)
    plt.splat_sensor(FILM, f_sep, h1, channel=channel, weight_scale=scale, dropped=d_sep)
    run(h2, {"film_desc": FILM, "film": f_fused, "channel": channel, "weight_scale": scale, "dropped": d_fused})
    torch.cuda.synchronize()
    for k in plt.HIT_KEYS + (("mask_bits", "flags") if flags else ("mask_bits",)):
        assert torch.equal(h1[k], h2[k]), k
    return f_sep.cpu().numpy(), f_fused.cpu().numpy(), int(d_sep.item()), int(d_fused.item())


@pytest.mark.parametrize("n", [1, 1000, (1 << 20) + 3])
def test_trace_splat_fp32_matches_separate(gpu_lib, n):
    plt = gpu_lib
    cfg = C.CONFIGS["C2"]
    lens = plt.Lens(C.lens_text("C2"), **cfg["opts"])
    d = plt.rays_to_device(R.gen_rays(cfg["law"], 5, 0, n))
    a, b, da, db = _films(plt, lambda h, sp: plt.trace_rays(lens, lens.all_t_id(), d, h, splat=sp), n,
                          scale=2.0 ** -10)
    assert np.array_equal(a, b) and da == db
    assert n < 1000 or a.sum() > 0


def test_trace_splat_fp64_ghost_channels(gpu_lib):
    import torch
    plt = gpu_lib
    cfg = C.CONFIGS["C4_22"]
    lens = plt.Lens(C.lens_text("C4_22"), **cfg["opts"])
    n = 1 << 19
    law = dict(cfg["law"], lam=(400.0, 700.0))
    d = plt.rays_to_device(R.gen_rays(law, 9, 0, n))
    ch = torch.from_numpy(np.random.default_rng(1).integers(0, 4, n).astype(np.uint8)).cuda()   # 3 = dropped
    a, b, da, db = _films(plt, lambda h, sp: plt.trace_rays(lens, 65616, d, h, precision=plt.FP64, splat=sp), n,
                          channel=ch, scale=1.0 / 3.0)
    assert np.array_equal(a, b) and da == db and a.sum() > 0 and da > 0


@pytest.mark.parametrize("name,tag", [("C2", 0), ("C4_59", 16404)])
def test_eval_map_splat_matches_separate(gpu_lib, name, tag):
    plt = gpu_lib
    cfg = C.CONFIGS[name]
    m = plt.Map(C.fitted_map_blob(name, tag))
    law = dict(cfg["law"])
    if "channels" in cfg:
        law["lam"] = (400.0, 700.0)
    n = (1 << 20) + 129
    d = plt.rays_to_device(R.gen_rays(law, 13, 0, n))
    a, b, da, db = _films(plt, lambda h, sp: plt.eval_map(m, d, h, splat=sp), n, scale=1.0, flags=False)
    assert np.array_equal(a, b) and da == db and a.sum() > 0
