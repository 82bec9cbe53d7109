"""Classifier ablation (the paper's Fig. "Importance of Classifier Network", PAPER.md:448-465;
SURVEY E7): render the depth-of-field image and a flare path with the fitted maps as they
are, and with the classifier disabled (its output bias raised so every ray is "valid"),
against the exact trace on the same rays.

    python tools/classifier_ablation.py [--out profiles/r01_classifier_ablation.json]
"""
import argparse
import json
import os
import struct
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2605_04017_b200 as plt  # noqa: E402
from paper_2605_04017_b200.render import render_dof, render_flare  # noqa: E402
from plt_inputs import configs as C  # noqa: E402
from plt_inputs import rays as R  # noqa: E402


def disable_classifier(blob: bytes) -> bytes:
    """Raise the classifier's output bias to +1e4 (PLTMAP01 layout, plt_inputs.rays)."""
    b = bytearray(blob)
    off = 8 + struct.calcsize("<IIQII") + 80
    for _ in range(3):                                   # classifier layers 4-32, 32-32, 32-1
        fo, fi = struct.unpack_from("<II", b, off)
        off += 8 + 2 * fo * fi
        if fo == 1:
            struct.pack_into("<f", b, off, 1.0e4)
        off += 4 * fo
    return bytes(b)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    rep = {}
    # depth of field (C3_DOF at the in-focus shift, 256 spp)
    cfg = C.CONFIGS["C3_DOF"]
    lens = plt.Lens(C.lens_text("C3_DOF"), **cfg["opts"])
    spp, W, H = 256, cfg["width_px"], cfg["height_px"]
    d = plt.rays_to_device(R.gen_rays(C.dof_law(0.6, spp), cfg["seed"], 0, W * H * spp))
    imgs = {}
    for key, blob in (("trace", None), ("map", C.fitted_map_blob("C3")),
                      ("map_no_classifier", disable_classifier(C.fitted_map_blob("C3")))):
        m = plt.Map(blob, lens=lens) if blob else None
        film = torch.zeros(W * H, dtype=torch.int64, device="cuda")
        render_dof(lens, d, cfg["scene"], film, spp, cfg["opts"]["backward_exit_z_mm"], m=m,
                   map_plane_z=C.CONFIGS["C3"]["law"]["plane_z"], weight_scale=1.0 / spp)
        torch.cuda.synchronize()
        imgs[key] = film.double().cpu().numpy()
    t = imgs["trace"]
    lit = t > 0
    rep["dof"] = {k: {"energy_ratio": float(v.sum() / t.sum()),
                      "mape": float(np.mean(np.abs(v[lit] - t[lit]) / t[lit]))}
                  for k, v in imgs.items() if k != "trace"}
    # flare: the 22 mm ghost 65616 (3 channels x 2^20 rays)
    fc = C.CONFIGS["C4_22"]
    gl = plt.Lens(C.lens_text("C4_22"), **fc["opts"])
    fd, npc = fc["film"], fc["n_per_channel"]
    rays = [plt.rays_to_device(C.flare_rays("C4_22", c, 0, npc)) for c in range(3)]
    blob = C.fitted_map_blob("C4_22", 65616)
    films = {}
    for key, mp in (("trace", None), ("map", plt.Map(blob, lens=gl)),
                    ("map_no_classifier", plt.Map(disable_classifier(blob), lens=gl))):
        film = torch.zeros(3 * fd["height_px"] * fd["width_px"], dtype=torch.int64, device="cuda")
        render_flare(gl, [65616], rays, fd, film, maps={65616: mp} if mp else None, weight_scale=1.0 / npc)
        torch.cuda.synchronize()
        films[key] = film.double().view(3, fd["height_px"] // 16, 16, fd["width_px"] // 16, 16).sum((2, 4))
    ft = films["trace"]
    rep["flare_65616"] = {k: {"energy_ratio": float(v.sum() / ft.sum()),
                              "rel_l1_bin16": float((v - ft).abs().sum() / ft.sum())}
                          for k, v in films.items() if k != "trace"}
    print(json.dumps(rep, indent=1))
    if a.out:
        with open(a.out, "w") as f:
            json.dump(rep, f, indent=1)


if __name__ == "__main__":
    main()
