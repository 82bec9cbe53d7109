"""Probe: eval_map time on the bench workload (C2 fitted map, 2^24 dz-less rays, splat fused
as in bench.py), median of 30 launches after 5 warm-ups, CUDA events on the stream.
Run with PLT_LIB pointing at a variant library (A/B of kernel arithmetic choices).

    PLT_LIB=... python tools/map_time_probe.py [--rays 16777216] [--tag name]
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2605_04017_b200 as plt  # noqa: E402
from plt_inputs import configs as C  # noqa: E402
from plt_inputs import rays as R  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rays", type=int, default=1 << 24)
    ap.add_argument("--tag", default=os.path.basename(os.environ.get("PLT_LIB", "libplt.so")))
    ap.add_argument("--map", default="C2")
    ap.add_argument("--coherent", action="store_true",
                    help="sort the rays by input position (rows, then columns): a pixel-ordered batch "
                         "whose valid fraction varies coherently along the index range")
    ap.add_argument("--ghost", type=int, default=0, help="(C4 configs) a ghost's fitted flare map and channel-1 rays")
    a = ap.parse_args()
    cfg = C.CONFIGS[a.map]
    lens = plt.Lens(C.lens_text(a.map), **cfg["opts"])
    n = a.rays
    if a.ghost:
        m = plt.Map(open(os.path.join(ROOT, "maps", "flare", a.map, f"{a.ghost}.pltmap"), "rb").read(), lens=lens)
        rays = C.flare_rays(a.map, 1, 0, n)
    else:
        m = plt.Map(C.fitted_map_blob(a.map), lens=lens)
        rays = R.gen_rays(cfg["law"], cfg["seed"], 0, n)
    if a.coherent:
        import numpy as np
        order = np.lexsort((rays["ox"], np.round(rays["oy"], 1)))
        rays = {k: (v[order] if hasattr(v, "shape") and getattr(v, "shape", ()) == (n,) else v) for k, v in rays.items()}
    d = plt.rays_to_device(rays, with_dz=False)
    h = plt.alloc_hits(n)
    fd = {"width_px": 768, "height_px": 512, "channels": 1, "sensor_w_mm": 36.0, "sensor_h_mm": 24.0,
          "center_x_mm": 0.0, "center_y_mm": 0.0}
    film = torch.zeros(768 * 512, dtype=torch.int64, device="cuda")
    spl = {"film_desc": fd, "film": film, "weight_scale": 1.0 / n}
    for _ in range(5):
        plt.eval_map(m, d, h, splat=spl)
    torch.cuda.synchronize()
    ts = []
    for _ in range(30):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        plt.eval_map(m, d, h, splat=spl)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    w = h["mask_bits"].view(torch.int32)
    valid = float(sum(bin(x & 0xFFFFFFFF).count("1") for x in w[:4096].tolist())) / (4096 * 32)
    ms = statistics.median(ts)
    print(json.dumps({"tag": a.tag, "map": a.map, "ghost": a.ghost, "coherent": a.coherent, "rays": n, "ms": ms, "M_rays_s": n / ms / 1e3,
                      "valid_sample": valid, "min_ms": min(ts)}), flush=True)


if __name__ == "__main__":
    main()
