"""Probe (CPU, numpy): how much regressor-output error each choice of activation precision
in eval_map's stored hidden layers would cost, on the committed fitted maps.

The kernel stores each hidden activation h = tanh(z) as the A operand of the next
tcgen05.mma.  Variants emulated here, per stored regressor layer (1..4):
  hilo  -- bf16 hi + bf16 lo pair (shipped; ~2^-17 relative)
  f16   -- one fp16 value (round to nearest even; weights converted exactly bf16 -> fp16)
  bf16  -- one bf16 value
The pre-activations are computed in float64 from the quantised activations; tanh is exact;
the inputs are the canonical inputs of Eq. 10 in float64 (the kernel's 3-term input split is
exact to ~2^-24).  Prints max / p999 |Δy| in normalised output units over rays valid in the
exact forward, per variant string (one letter per stored layer: H = hilo, F = f16, B = bf16).

    python tools/act_precision_probe.py [--rays 262144] [--flare]
"""
import argparse
import glob
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import oracle  # noqa: E402
from plt_inputs import configs as C  # noqa: E402
from plt_inputs import rays as R  # noqa: E402


def bf16(a):
    b = np.asarray(a, np.float32).view(np.uint32).astype(np.uint64)
    b = (b + 0x7FFF + ((b >> 16) & 1)) & 0xFFFF0000
    return b.astype(np.uint32).view(np.float32).astype(np.float64)


def quant(h, mode):
    if mode == "H":
        h32 = h.astype(np.float32)
        hi = bf16(h32)
        return hi + bf16((h32 - hi).astype(np.float32))
    if mode == "F":
        return h.astype(np.float16).astype(np.float64)
    if mode == "B":
        return bf16(h.astype(np.float32))
    return h


def canon(m, rays):
    lo, hi = m["norm"][:4], m["norm"][4:8]
    px, py, wx, wy = (rays[k].astype(np.float64) for k in ("ox", "oy", "dx", "dy"))
    r = np.hypot(px, py)
    with np.errstate(invalid="ignore", divide="ignore"):
        c = np.where(r > 0, px / r, 1.0)
        s = np.where(r > 0, py / r, 0.0)
    wpx = c * wx + s * wy
    wpy = np.abs(-s * wx + c * wy)
    xin = np.stack([r, wpx, wpy, rays["lambda_nm"].astype(np.float64)], 1)
    return np.clip(2 * (xin - lo) / (hi - lo) - 1, -1, 1)


def forward(head, x, modes=None):
    """modes[k] = precision of the k-th stored hidden activation (None: exact)."""
    h = x
    nl = len(head["W"])
    for li in range(nl):
        z = h @ head["W"][li].T + head["b"][li]
        if li == nl - 1:
            return z
        h = np.tanh(z)
        if modes is not None and li < nl - 2:   # the last hidden layer feeds the fp32 output dot product
            h = quant(h, modes[li])


def probe(blob, cfg_name, n, seed, variants):
    m = oracle.parse_map_blob(blob)
    cfg = C.CONFIGS[cfg_name]
    law = dict(cfg["law"])
    if "channels" in cfg:
        law["lam"] = (400.0, 700.0)
    rays = R.gen_rays(law, seed, 0, n)
    x = canon(m, rays)
    valid = forward(m["classifier"], x)[:, 0] >= 0
    xv = x[valid]
    exact = forward(m["regressor"], xv)
    out = {"valid": float(valid.mean())}
    for v in variants:
        e = np.abs(forward(m["regressor"], xv, v) - exact)
        out[v] = [float(e.max()), float(np.quantile(e, 0.999))] if e.size else [0.0, 0.0]
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rays", type=int, default=1 << 18)
    ap.add_argument("--flare", action="store_true")
    ap.add_argument("--variants", default="HHHH,FFFF,BBBB,FHHH,HFFF,FFHH,HHFF,FHFH,HFHF,FFFH,HFFH")
    a = ap.parse_args()
    variants = a.variants.split(",")
    jobs = [("C2_0", "C2"), ("C3_0", "C3"), ("C4_22_65616", "C4_22"), ("C4_59_16404", "C4_59")]
    for tag, cfg in jobs:
        with open(os.path.join(ROOT, "maps", tag + ".pltmap"), "rb") as f:
            print(json.dumps({"map": tag, **probe(f.read(), cfg, a.rays, 7, variants)}), flush=True)
    if a.flare:
        worst = {}
        for cfg in ("C4_22", "C4_59"):
            for path in sorted(glob.glob(os.path.join(ROOT, "maps", "flare", cfg, "*.pltmap"))):
                with open(path, "rb") as f:
                    r = probe(f.read(), cfg, a.rays // 4, 8, variants)
                for v in variants:
                    worst[v] = max(worst.get(v, 0.0), r[v][0])
        print(json.dumps({"map": "flare (worst max over all)", **worst}), flush=True)


if __name__ == "__main__":
    main()
