"""Accuracy of the committed fitted maps (maps/*.pltmap, tests/fit_map.py) evaluated by the
library's eval_map kernel against the library's exact trace (itself parity-pinned to the
oracle in test_gpu_trace.py) on held-out seeded rays: the paper's claim that the
classifier-regressor reproduces the lens transport.  This is an
ACCURACY check of trained weights, not a parity test (no oracle input comes from here)."""
import glob
import os

import pytest

from plt_inputs import configs as C
from plt_inputs import rays as R

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
MAPS = sorted(glob.glob(os.path.join(ROOT, "maps", "*.pltmap")))
EVAL_SEED = 7_000_003        # disjoint from fit_map's training (7_000_001) and report (7_000_002) seeds


def _unpack(words, n):
    import torch
    w = words.view(torch.int32).to(torch.int64) & 0xFFFFFFFF
    return ((w[:, None] >> torch.arange(32, device=w.device)) & 1).reshape(-1)[:n].bool()


def _setup(plt, path):
    cfg_name, pid = os.path.basename(path)[:-7].rsplit("_", 1)
    cfg = C.CONFIGS[cfg_name]
    lens = plt.Lens(C.lens_text(cfg_name), **cfg["opts"])
    pid = lens.all_t_id() if int(pid) == 0 else int(pid)
    m = plt.Map(open(path, "rb").read(), lens=lens)
    return cfg_name, cfg, lens, pid, m


@pytest.mark.parametrize("path", MAPS, ids=[os.path.basename(p) for p in MAPS])
def test_fitted_map_matches_exact_trace(gpu_lib, path):
    import torch
    plt = gpu_lib
    cfg_name, cfg, lens, pid, m = _setup(plt, path)
    law = dict(cfg["law"])
    if "channels" in cfg:
        law["lam"] = (400.0, 700.0)
    n = 1 << 20
    d = plt.rays_to_device(R.gen_rays(law, EVAL_SEED, 0, n))
    ht, hm = plt.alloc_hits(n), plt.alloc_hits(n)
    prec = plt.FP32 if pid == lens.all_t_id() else plt.FP64
    plt.trace_rays(lens, pid, d, ht, direction=cfg["direction"], precision=prec)
    plt.eval_map(m, d, hm)
    torch.cuda.synchronize()
    vt, vm = _unpack(ht["mask_bits"], n), _unpack(hm["mask_bits"], n)
    both = vt & vm
    agree = float((vt == vm).float().mean())
    dp = torch.hypot(hm["px"] - ht["px"], hm["py"] - ht["py"])[both]
    dw = torch.sqrt(sum((hm[k] - ht[k]) ** 2 for k in ("dx", "dy", "dz")))[both]
    dI = (hm["throughput"] - ht["throughput"]).abs()[both]
    q = lambda t: float(torch.quantile(t.float(), 0.99))
    stats = {"valid": float(vt.float().mean()), "agree": agree, "dp99": q(dp), "dw99": q(dw), "dI99": q(dI)}
    print(os.path.basename(path), stats)
    assert both.sum() > 1000
    assert agree >= 0.996, stats
    assert stats["dp99"] <= 0.08 and stats["dw99"] <= 4e-3 and stats["dI99"] <= 5e-4, stats


@pytest.mark.parametrize("path", [p for p in MAPS if "C4_" in p], ids=lambda p: os.path.basename(p))
def test_fitted_ghost_map_flare_film(gpu_lib, path):
    """RGB flare film of one ghost path (2^20 rays per channel) from the map vs
    from the exact float64 trace on the same rays: energy within 2 %, rel-L1 on 16x16-pixel
    bins (reading A30) far below the Monte-Carlo difference of two independent ray sets."""
    import torch
    plt = gpu_lib
    cfg_name, cfg, lens, pid, m = _setup(plt, path)
    fd, n = cfg["film"], cfg["n_per_channel"]
    npx = fd["channels"] * fd["height_px"] * fd["width_px"]

    def films(shift):
        f = {k: torch.zeros(npx, dtype=torch.int64, device="cuda") for k in ("trace", "map")}
        for c, lam in enumerate(cfg["channels"]):
            law = dict(cfg["law"])
            law["lam"] = lam
            d = plt.rays_to_device(R.gen_rays(law, 1000 + cfg["seed"] * 16 + c + shift, 0, n))
            ch = torch.full((n,), c, dtype=torch.uint8, device="cuda")
            h = plt.alloc_hits(n)
            plt.trace_rays(lens, pid, d, h, direction=cfg["direction"], precision=plt.FP64)
            plt.splat_sensor(fd, f["trace"], h, channel=ch, weight_scale=1.0 / n)
            h = plt.alloc_hits(n)
            plt.eval_map(m, d, h)
            plt.splat_sensor(fd, f["map"], h, channel=ch, weight_scale=1.0 / n)
        torch.cuda.synchronize()
        return {k: v.double().view(fd["channels"], fd["height_px"] // 16, 16, fd["width_px"] // 16, 16).sum((2, 4))
                for k, v in f.items()}

    a, b = films(0), films(8)
    rel = lambda x, y: float((x - y).abs().sum() / y.sum())
    same, mc = rel(a["map"], a["trace"]), rel(b["trace"], a["trace"])
    energy = float(a["map"].sum() / a["trace"].sum())
    print(os.path.basename(path), {"rel_l1_bin16": same, "mc_floor": mc, "energy": energy})
    assert abs(energy - 1.0) <= 0.02
    assert same <= 0.06 and same <= 0.5 * mc


FLARE_MAPS = sorted(glob.glob(os.path.join(ROOT, "maps", "flare", "*", "*.pltmap")))
MCMC_MAPS = [os.path.join(ROOT, "maps", "flare", "C4_59", "16810240.pltmap")]   # trained on MCMC samples


@pytest.mark.parametrize("path", MAPS + FLARE_MAPS[::12] + MCMC_MAPS,
                         ids=[os.path.relpath(p, os.path.join(ROOT, "maps")) for p in MAPS + FLARE_MAPS[::12] + MCMC_MAPS])
def test_fitted_map_kernel_parity(gpu_lib, path):
    """PARITY of the eval_map kernel on trained weights (the bench's map and the flare
    maps) against the float64 oracle's O10 on the same blob: raw logit and regressor
    outputs within the 2e-3 north-star tolerance (A18), masks equal where |logit| > 2e-3.
    Trained classifiers amplify activation error (A31); this pins the kernel's tanh
    choices (accurate on the most logit-influential h1 units, map.cpp) on real weights."""
    import numpy as np
    import oracle
    from test_gpu_map_splat import compare_map, gpu_map
    plt = gpu_lib
    rel = os.path.relpath(path, os.path.join(ROOT, "maps"))
    cfg_name = rel.split(os.sep)[1] if rel.startswith("flare") else os.path.basename(path)[:-7].rsplit("_", 1)[0]
    blob = open(path, "rb").read()
    m = plt.Map(blob)
    rays = R.gen_rays(C.CONFIGS[cfg_name]["law"], EVAL_SEED + 1, 0, (1 << 17) + 3)
    g = gpu_map(plt, m, rays)
    o = oracle.map_eval(blob, rays, threads=oracle.host_threads())
    compare_map(g, o, blob)
    print(rel, "max logit err", float(np.abs(g["raw"][:, 0] - o["raw"][:, 0]).max()))
