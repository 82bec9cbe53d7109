"""Probe: eval_map's raw-output error against the float64 oracle for every fitted map
(maps/*.pltmap and, with --flare, every per-ghost map), on 2^18 rays of the map's config.
Prints one JSON line per map: max |logit error|, max regressor-output error (normalised
units, rays valid in both with |logit| > 2e-3), mask disagreements on decided rays.
Run with PLT_LIB pointing at a variant library to compare kernel arithmetic choices.

    PLT_LIB=... python tools/logit_err_probe.py [--flare] [--rays 262144]
"""
import argparse
import glob
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

import oracle  # noqa: E402
import paper_2605_04017_b200 as plt  # noqa: E402
from plt_inputs import configs as C  # noqa: E402
from plt_inputs import rays as R  # noqa: E402
from test_gpu_map_splat import gpu_map  # noqa: E402


def probe(blob, cfg_name, n, seed):
    cfg = C.CONFIGS[cfg_name]
    rays = R.gen_rays(cfg["law"], seed, 0, n)
    m = plt.Map(blob)
    g = gpu_map(plt, m, rays)
    o = oracle.map_eval(blob, rays, threads=oracle.host_threads())
    lo = o["raw"][:, 0]
    dec = np.abs(lo) > 2e-3
    both = g["valid"] & o["valid"] & dec
    return {"max_logit_err": float(np.abs(g["raw"][:, 0] - lo).max()),
            "p999_logit_err": float(np.quantile(np.abs(g["raw"][:, 0] - lo), 0.999)),
            "max_reg_err": float(np.abs(g["raw"][both, 1:] - o["raw"][both, 1:]).max()) if both.any() else 0.0,
            "mask_mismatch_decided": int((g["valid"] != o["valid"])[dec].sum()), "valid": float(o["valid"].mean())}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rays", type=int, default=1 << 18)
    ap.add_argument("--flare", action="store_true")
    a = ap.parse_args()
    plt.load()
    jobs = [("C2_0", "C2"), ("C3_0", "C3"), ("C4_22_65616", "C4_22"), ("C4_59_16404", "C4_59")]
    for tag, cfg in jobs:
        with open(os.path.join(ROOT, "maps", tag + ".pltmap"), "rb") as f:
            blob = f.read()
        print(json.dumps({"map": tag, **probe(blob, cfg, a.rays, 7)}), flush=True)
    if a.flare:
        worst = {}
        for cfg in ("C4_22", "C4_59"):
            for path in sorted(glob.glob(os.path.join(ROOT, "maps", "flare", cfg, "*.pltmap"))):
                with open(path, "rb") as f:
                    r = probe(f.read(), cfg, a.rays // 4, 8)
                for k, v in r.items():
                    if k != "valid":
                        worst[k] = max(worst.get(k, 0), v)
        print(json.dumps({"map": "flare (worst over all)", **worst}), flush=True)


if __name__ == "__main__":
    main()
