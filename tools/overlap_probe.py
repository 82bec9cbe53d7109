"""Probe: the C2 bench step with trace_rays and eval_map run back to back (one stream) vs
concurrently (two streams, eval_map launched first so its persistent CTAs take their SM
share and the trace blocks fill the rest).  PLT_MAP_GROUPS selects the eval_map variant.
Measured (profiles/r01_overlap_probe.jsonl): no gain -- both kernels load the MUFU pipe;
the half-SM eval_map variant ("42": 4 pipelines at <= 64 registers) used for that
measurement was removed again.

    PLT_MAP_GROUPS=8 python tools/overlap_probe.py [--rays 2^24] [--steps 20]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2605_04017_b200 as plt  # noqa: E402
from plt_inputs import configs as C  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rays", type=int, default=1 << 24)
    ap.add_argument("--steps", type=int, default=20)
    a = ap.parse_args()
    plt.load()
    dev = torch.device("cuda", 0)
    n = a.rays
    cfg, rays_np = bench.make_workload(0, n)
    lens = plt.Lens(C.lens_text("C2"), **cfg["opts"])
    pid = lens.all_t_id()
    m = plt.Map(C.fitted_map_blob("C2"), lens=lens)
    d = {k: torch.from_numpy(rays_np[k]).to(dev) for k in plt.RAY_KEYS if k in rays_np}
    d["plane_z"] = rays_np["plane_z"]
    ht, hm = plt.alloc_hits(n, dev), plt.alloc_hits(n, dev)
    F = bench.FILM
    film = torch.zeros(F["channels"] * F["height_px"] * F["width_px"], dtype=torch.int64, device=dev)
    sa = torch.cuda.current_stream()
    sb = torch.cuda.Stream(device=dev)
    spl = {"film_desc": F, "film": film, "weight_scale": 1.0 / n}

    def seq():
        plt.trace_rays(lens, pid, d, ht, stream=sa, splat=spl)
        plt.eval_map(m, d, hm, stream=sa, splat=spl)

    def ovl():
        fork = torch.cuda.Event()
        fork.record(sa)
        sb.wait_event(fork)
        plt.eval_map(m, d, hm, stream=sa, splat=spl)
        plt.trace_rays(lens, pid, d, ht, stream=sb, splat=spl)
        join = torch.cuda.Event()
        join.record(sb)
        sa.wait_event(join)

    def only_map():
        plt.eval_map(m, d, hm, stream=sa, splat=spl)

    def only_trace():
        plt.trace_rays(lens, pid, d, ht, stream=sa, splat=spl)

    out = {"groups": os.environ.get("PLT_MAP_GROUPS", "8"), "rays": n}
    films = {}
    for name, fn in (("sequential", seq), ("overlap", ovl), ("eval_map", only_map), ("trace", only_trace)):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        film.zero_()
        fn()
        torch.cuda.synchronize()
        films[name] = film.clone()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record(sa)
        for _ in range(a.steps):
            fn()
        t1.record(sa)
        torch.cuda.synchronize()
        ms = t0.elapsed_time(t1) / a.steps
        out[name + "_ms"] = round(ms, 4)
    out["overlap_film_equal"] = bool(torch.equal(films["sequential"], films["overlap"]))
    out["speedup"] = round(out["sequential_ms"] / out["overlap_ms"], 3)
    out["G_rays_s_overlap"] = round(n / out["overlap_ms"] / 1e6, 3)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
