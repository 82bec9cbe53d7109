"""Flare image: fitted per-path maps vs the exact trace (the paper's
lens-flare comparison).

    python tools/flare_compare.py --config C4_22 [--maps maps/flare] [--out profiles/r01_flare_C4_22.json]
                                  [--png profiles/r01_flare_C4_22]

Both images are rendered from the SAME rays (2^20 per RGB channel) with
paper_2605_04017_b200.render.render_flare: every ghost path traced in float64, and every
ghost path with a fitted map evaluated by eval_map (paths without a map are traced in
both images).  Reported (reading A30): energy ratio, relative L1 on the film and on 4x4 /
16x16-pixel bins, MAPE over lit 16x16 bins -- for the total image and per path -- next to
the Monte-Carlo difference of two independent ray sets.  Optional PNG images (tone-mapped).
"""
import argparse
import glob
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2605_04017_b200 as plt  # noqa: E402
from paper_2605_04017_b200.render import render_flare  # noqa: E402
from plt_inputs import configs as C  # noqa: E402
from plt_inputs import rays as R  # noqa: E402


def diff(img, ref, fd, bins=(1, 4, 16)):
    out = {}
    Ch, H, W = fd["channels"], fd["height_px"], fd["width_px"]
    for b in bins:
        i = img.view(Ch, H // b, b, W // b, b).sum((2, 4))
        r = ref.view(Ch, H // b, b, W // b, b).sum((2, 4))
        out[f"rel_l1_bin{b}"] = float((i - r).abs().sum() / r.sum().clamp_min(1e-300))
        if b == bins[-1]:
            lit = r > 0
            out[f"mape_lit_bin{b}"] = float(((i - r).abs()[lit] / r[lit]).mean()) if lit.any() else 0.0
    out["energy_ratio"] = float(img.sum() / ref.sum().clamp_min(1e-300))
    return out


def write_png(path, film, fd, exposure):
    """Tone-mapped 8-bit PNG of the film (zlib only; no imaging dependency)."""
    import struct
    import zlib
    Ch, H, W = fd["channels"], fd["height_px"] // 2, fd["width_px"] // 2     # 2x2-binned image
    x = film.view(Ch, H, 2, W, 2).sum((2, 4)).permute(1, 2, 0).double().cpu().numpy() * exposure / 4
    img = np.clip(255.0 * (1.0 - np.exp(-x)) ** (1 / 2.2), 0, 255).astype(np.uint8)
    raw = b"".join(b"\x00" + img[y].tobytes() for y in range(H))

    def chunk(t, d):
        return struct.pack(">I", len(d)) + t + d + struct.pack(">I", zlib.crc32(t + d) & 0xFFFFFFFF)
    png = (b"\x89PNG\r\n\x1a\n" + chunk(b"IHDR", struct.pack(">IIBBBBB", W, H, 8, 2, 0, 0, 0)) +
           chunk(b"IDAT", zlib.compress(raw, 9)) + chunk(b"IEND", b""))
    with open(path, "wb") as f:
        f.write(png)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C4_22")
    ap.add_argument("--maps", default=os.path.join(ROOT, "maps", "flare"))
    ap.add_argument("--out", default=None)
    ap.add_argument("--png", default=None, help="prefix: writes <prefix>_trace.png and <prefix>_map.png")
    a = ap.parse_args()
    cfg = C.CONFIGS[a.config]
    fd, npc = cfg["film"], cfg["n_per_channel"]
    lens = plt.Lens(C.lens_text(a.config), **cfg["opts"])
    ids, _ = lens.enumerate_ghosts(2)
    ghosts = [int(g) for g in ids if int(g) != lens.all_t_id()]
    maps = {}
    for f in glob.glob(os.path.join(a.maps, a.config, "*.pltmap")):
        maps[int(os.path.basename(f)[:-7])] = plt.Map(open(f, "rb").read(), lens=lens)
    rays = [plt.rays_to_device(C.flare_rays(a.config, c, 0, npc)) for c in range(3)]
    rays_b = [plt.rays_to_device(R.gen_rays(
        dict(cfg["law"], lam=cfg["channels"][c]), cfg["seed"] * 16 + c + 8, 0, npc)) for c in range(3)]
    npx = fd["channels"] * fd["height_px"] * fd["width_px"]
    per_t = {g: torch.zeros(npx, dtype=torch.int64, device="cuda") for g in ghosts}
    per_m = {g: torch.zeros(npx, dtype=torch.int64, device="cuda") for g in ghosts}
    scratch = {g: torch.zeros(npx, dtype=torch.int64, device="cuda") for g in ghosts}
    render_flare(lens, ghosts, rays, fd, None, per_path=scratch, weight_scale=1.0 / npc)             # warm-up
    render_flare(lens, ghosts, rays, fd, None, maps=maps, per_path=scratch, weight_scale=1.0 / npc)  # (weights up)
    del scratch
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    ev[0].record()
    render_flare(lens, ghosts, rays, fd, None, per_path=per_t, weight_scale=1.0 / npc)
    ev[1].record()
    used = render_flare(lens, ghosts, rays, fd, None, maps=maps, per_path=per_m, weight_scale=1.0 / npc)
    ev[2].record()
    torch.cuda.synchronize()
    t_trace, t_map = ev[0].elapsed_time(ev[1]) / 1e3, ev[1].elapsed_time(ev[2]) / 1e3
    mc = torch.zeros(npx, dtype=torch.int64, device="cuda")
    render_flare(lens, ghosts, rays_b, fd, mc, weight_scale=1.0 / npc)
    tot_t = sum(f.double() for f in per_t.values()) * 2.0 ** -32
    tot_m = sum(f.double() for f in per_m.values()) * 2.0 ** -32
    rep = {"config": a.config, "ghosts": len(ghosts), "with_map": len(maps), "rays_per_channel": npc,
           "total": {"map_vs_trace": diff(tot_m, tot_t, fd), "mc_floor_trace_vs_trace": diff(mc.double() * 2.0 ** -32,
                                                                                             tot_t, fd)},
           "render_s": {"trace_fp64": t_trace, "maps": t_map, "note": "CUDA events around each full render (warm)"}, "per_path": {}}
    energy = {g: float(per_t[g].sum()) for g in ghosts}
    tot_e = sum(energy.values())
    for g in sorted(ghosts, key=lambda g: -energy[g]):
        if g in maps:
            d = diff(per_m[g].double(), per_t[g].double(), fd)
            rep["per_path"][str(g)] = {"energy_share": energy[g] / tot_e, **d}
    shares = [v["energy_share"] for v in rep["per_path"].values()]
    rep["mapped_energy_share"] = float(sum(shares))
    print(json.dumps({k: v for k, v in rep.items() if k != "per_path"}, indent=1))
    top = list(rep["per_path"].items())[:5]
    print("brightest mapped paths:", json.dumps(top, indent=0)[:1500])
    if a.out:
        with open(a.out, "w") as f:
            json.dump(rep, f, indent=1)
    if a.png:
        expo = 4.0 / float(tot_t.view(3, -1).max(1).values.mean())
        write_png(a.png + "_trace.png", tot_t, fd, expo)
        write_png(a.png + "_map.png", tot_m, fd, expo)


if __name__ == "__main__":
    main()
