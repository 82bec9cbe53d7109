"""Probe: the C4 flare trace of one channel (2^20 rays, every ghost, fp64, fused splat)
as one plt_trace_paths call (shared all-T prefix) vs one plt_trace_rays_splat per path;
median of 10 after 3 warm-ups, CUDA events.  Checks that the films agree bit for bit.

    python tools/trace_paths_probe.py [--config C4_22] [--rays 1048576]
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
from plt_inputs import philox as PX  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C4_22")
    ap.add_argument("--rays", type=int, default=1 << 20)
    ap.add_argument("--once", action="store_true", help="one trace_paths call only (for ncu launch lists)")
    a = ap.parse_args()
    cfg = C.CONFIGS[a.config]
    lens = plt.Lens(C.lens_text(a.config), **cfg["opts"])
    ids = [int(g) for g in lens.enumerate_ghosts(2)[0][1:]]
    n = a.rays
    d = plt.gen_rays(PX.law_constants(dict(cfg["law"], lam=cfg["channels"][1])), cfg["seed"] * 16 + 1, 0, n)
    fd = cfg["film"]
    film = torch.zeros(fd["channels"] * fd["height_px"] * fd["width_px"], dtype=torch.int64, device="cuda")
    spl = {"film_desc": fd, "film": film, "weight_scale": 1.0 / n}
    hs = [plt.alloc_hits(n) for _ in ids]
    h1 = plt.alloc_hits(n)

    def per_path():
        for g in ids:
            plt.trace_rays(lens, g, d, h1, precision=plt.FP64, splat=spl)

    def shared():
        plt.trace_paths(lens, ids, d, hs, precision=plt.FP64, splat=spl)

    def shared_one_buffer():
        plt.trace_paths(lens, ids, d, [h1] * len(ids), precision=plt.FP64, splat=spl)

    if a.once:
        shared()
        torch.cuda.synchronize()
        return
    out = {"config": a.config, "rays": n, "paths": len(ids)}
    films = {}
    for name, fn in (("per_path", per_path), ("trace_paths", shared), ("trace_paths_one_buffer", shared_one_buffer)):
        for _ in range(3):
            fn()
        ts = []
        for _ in range(10):
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        out[name + "_ms"] = statistics.median(ts)
        film.zero_()
        fn()
        torch.cuda.synchronize()
        films[name] = film.clone()
    out["films_identical"] = bool(torch.equal(films["per_path"], films["trace_paths"]) and
                                  torch.equal(films["per_path"], films["trace_paths_one_buffer"]))
    out["speedup"] = out["per_path_ms"] / out["trace_paths_ms"]
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
