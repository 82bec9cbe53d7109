"""Algorithmic FLOPs per ray of the exact trace, per config and path, for the trace
roofline in bench.py.  Calls only the float64 oracle (test infrastructure;
this script writes a stored value, profiles/trace_flops.json, that bench.py reads -- bench
never executes the oracle outside its cpu_baseline / reference legs).

The work a ray needs is the formulas of O1-O8 for every surface step it BEGINS before it
terminates (a ray blocked at surface k does not need steps k+1...): oracle.trace reports
that count per ray (`steps`).  FLOPs per step (add / mul / div / sqrt = 1):
spherical interaction 77, planar interaction 56 (no quadratic root: 16 fewer in the
intersection, 5 fewer in the normal), stop crossing 13, output plane 6, input
normalisation 9.  FLOPs/ray = 9 + sum_k P(steps >= k) * flops(step k) (the output plane
counts as the step after the last surface).

    python tools/trace_flops.py [--rays 65536] [--out profiles/trace_flops.json]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import oracle  # noqa: E402
from oracle.lens import decode_path, mirrored  # noqa: E402
from plt_inputs import configs as C  # noqa: E402
from plt_inputs import rays as R  # noqa: E402

FLOPS = {"sphere": 77, "plane": 56, "stop": 13, "output": 6, "init": 9}


def step_kinds(lens, path_id, direction, first_r=False):
    """Kinds of the surface steps along a path in the traversal frame, then 'output'
    (first_r: also the index of the path's first reflection step, None for all-T)."""
    surfs = lens.surfaces if direction == oracle.FORWARD else mirrored(lens)
    seq = decode_path(path_id)
    kinds, s, d, k, fr = [], 0, +1, 0, None
    while 0 <= s < len(surfs):
        sf = surfs[s]
        if sf.is_stop:
            kinds.append("stop")
        else:
            kinds.append("plane" if sf.R == 0.0 else "sphere")
            if seq[k] == "R":
                d = -d
                if fr is None:
                    fr = len(kinds) - 1
            k += 1
        s += d
    return (kinds + ["output"], fr) if first_r else kinds + ["output"]


def path_flops(lens, path_id, direction, rays):
    t = oracle.trace(lens, path_id, direction, rays, threads=oracle.host_threads())
    kinds, fr = step_kinds(lens, path_id, direction, first_r=True)
    st = t["steps"]
    alive = [float((st >= k + 1).mean()) for k in range(len(kinds))]
    f = FLOPS["init"] + sum(a * FLOPS[kd] for a, kd in zip(alive, kinds))
    out = {"flops_per_ray": f, "valid": float(t["valid"].mean()), "steps": kinds, "alive_before_step": alive}
    if fr is not None:
        # plt_trace_paths (fp64) shares steps [0, first_R) with the all-T path: the work left
        # to the path itself is the steps from its first reflection on
        out["first_R_step"] = fr
        out["suffix_flops_per_ray"] = sum(a * FLOPS[kd] for a, kd in list(zip(alive, kinds))[fr:])
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rays", type=int, default=1 << 16)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "trace_flops.json"))
    a = ap.parse_args()
    res = {"_doc": __doc__.strip().splitlines()[0], "flops_per_step": FLOPS, "rays": a.rays, "configs": {}}
    for name in ("C1", "C2", "C3", "C5"):
        cfg = C.CONFIGS[name]
        lens = oracle.load_lens(C.lens_text(name), cfg["opts"])
        rays = C.c1_rays() if name == "C1" else R.gen_rays(cfg["law"], cfg["seed"], 0, a.rays)
        pid = 1 << lens.n_optical
        res["configs"][name] = {str(pid): path_flops(lens, pid, cfg["direction"], rays)}
        print(name, res["configs"][name][str(pid)]["flops_per_ray"], flush=True)
    for name in ("C4_22", "C4_59"):
        cfg = C.CONFIGS[name]
        lens = oracle.load_lens(C.lens_text(name), cfg["opts"])
        ids, _ = oracle.enumerate_ghosts(lens, 2)
        rays = C.flare_rays(name, 1, 0, a.rays)
        per = {str(pid): path_flops(lens, pid, cfg["direction"], rays) for pid in ids}
        res["configs"][name] = per
        ghosts = [v["flops_per_ray"] for k, v in per.items() if int(k) != ids[0]]
        print(name, "ghost mean flops/ray", float(np.mean(ghosts)), flush=True)
    with open(a.out, "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
