"""Depth-of-field camera: the fitted C3 map vs the exact trace (the
camera integrator of PAPER.md:422-431 and the sensor-shift focusing of P:425-427).

    python tools/dof_compare.py [--spp 64] [--out profiles/r01_dof.json] [--png profiles/r01_dof]

For each sensor shift of C3_DOF the same pixel-stratified rays are rendered through the
24 mm lens twice -- by the float32 exact trace, and by the fitted all-T map after
free-space propagation to the map's input plane (one precomputed map for every focus
setting) -- and shaded on the checkerboard scene plane (plt_shade_plane).
Reported: MAPE over pixels (the paper's image metric; reading A30 for the
normalisation), relative L1, a sharpness score (mean |gradient|) and the valid fraction
per shift.  By default the sensor rays aim at the paraxial exit pupil (plt_lens_pupils,
radius x1.1) instead of the rear clear aperture (--sampling rear), which wastes far
fewer samples; images are the unnormalised mean of I L over each pixel's samples.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2605_04017_b200 as plt  # noqa: E402
from paper_2605_04017_b200.render import render_dof  # noqa: E402
from plt_inputs import configs as C  # noqa: E402
from plt_inputs import rays as R  # noqa: E402


def sharpness(img):
    gx = np.abs(np.diff(img, axis=1)).mean()
    gy = np.abs(np.diff(img, axis=0)).mean()
    return float(gx + gy) / max(float(img.mean()), 1e-30)


def write_png(path, img):
    import struct
    import zlib
    H, W = img.shape
    g = np.clip(255.0 * (img / max(img.max(), 1e-30)) ** (1 / 2.2), 0, 255).astype(np.uint8)
    raw = b"".join(b"\x00" + g[y].tobytes() for y in range(H))

    def chunk(t, d):
        return struct.pack(">I", len(d)) + t + d + struct.pack(">I", zlib.crc32(t + d) & 0xFFFFFFFF)
    png = (b"\x89PNG\r\n\x1a\n" + chunk(b"IHDR", struct.pack(">IIBBBBB", W, H, 8, 0, 0, 0, 0)) +
           chunk(b"IDAT", zlib.compress(raw, 9)) + chunk(b"IEND", b""))
    with open(path, "wb") as f:
        f.write(png)


def render_pair(lens, m, shift, spp, cfg, pupil=None):
    law = C.dof_law(shift, spp, pupil)
    n = cfg["width_px"] * cfg["height_px"] * spp
    d = plt.rays_to_device(R.gen_rays(law, cfg["seed"], 0, n))
    pixels = cfg["width_px"] * cfg["height_px"]
    out = {}
    h = plt.alloc_hits(n)
    plt.trace_rays(lens, lens.all_t_id(), d, h, direction=plt.BACKWARD)
    torch.cuda.synchronize()
    w = h["mask_bits"].cpu().numpy().view(np.uint8)
    out["valid_fraction"] = float(np.unpackbits(w).sum()) / n
    for key, mm in (("trace", None), ("map", m)):
        film = torch.zeros(pixels, dtype=torch.int64, device="cuda")
        render_dof(lens, d, cfg["scene"], film, spp, cfg["opts"]["backward_exit_z_mm"], m=mm,
                   map_plane_z=C.CONFIGS["C3"]["law"]["plane_z"], weight_scale=1.0 / spp)
        torch.cuda.synchronize()
        out[key] = (film.double() * 2.0 ** -32).view(cfg["height_px"], cfg["width_px"]).cpu().numpy()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--spp", type=int, default=None)
    ap.add_argument("--out", default=None)
    ap.add_argument("--png", default=None)
    ap.add_argument("--sampling", choices=["exit", "rear"], default="exit",
                    help="aim the sensor rays at the paraxial exit pupil (x1.1) or at the rear clear aperture")
    a = ap.parse_args()
    cfg = C.CONFIGS["C3_DOF"]
    spp = a.spp or cfg["spp"]
    lens = plt.Lens(C.lens_text("C3_DOF"), **cfg["opts"])
    m = plt.Map(C.fitted_map_blob("C3"), lens=lens)
    pp = lens.pupils()
    pupil = (pp["exit_z_mm"], 1.1 * pp["exit_r_mm"]) if a.sampling == "exit" else None
    rep = {"config": "C3_DOF", "spp": spp, "image": [cfg["width_px"], cfg["height_px"]], "scene": cfg["scene"],
           "sampling": a.sampling, "pupil": pupil or (cfg["law"]["pupil_z"], cfg["law"]["pupil_r"]), "shifts": {}}
    for shift in cfg["sensor_shifts_mm"]:
        imgs = render_pair(lens, m, shift, spp, cfg, pupil)
        t, mp = imgs["trace"], imgs["map"]
        lit = t > 0
        rep["shifts"][str(shift)] = {
            "sensor_z_mm": C.CONFIGS["C3"]["law"]["plane_z"] + shift,
            "valid_fraction": imgs["valid_fraction"],
            "mape": float(np.mean(np.abs(mp[lit] - t[lit]) / t[lit])),
            "rel_l1": float(np.abs(mp - t).sum() / t.sum()),
            "energy_ratio": float(mp.sum() / t.sum()),
            "sharpness_trace": sharpness(t), "sharpness_map": sharpness(mp)}
        if a.png:
            write_png(f"{a.png}_{shift:+.1f}mm_trace.png", t)
            write_png(f"{a.png}_{shift:+.1f}mm_map.png", mp)
    print(json.dumps(rep, indent=1))
    if a.out:
        with open(a.out, "w") as f:
            json.dump(rep, f, indent=1)


if __name__ == "__main__":
    main()
