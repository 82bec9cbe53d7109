"""Probe: trace_rays time on a config's rays (device-generated, dz-less), median of 20 after
5 warm-ups, CUDA events.  For A/B of kernel variants / developer knobs (PLT_LIB,
PLT_TRACE_SPLIT_DELTA, PLT_TRACE_JIT, ...).

    python tools/trace_time_probe.py --config C3 [--rays 67108864] [--path 0] [--fp64]
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
    ap.add_argument("--config", default="C2")
    ap.add_argument("--rays", type=int, default=1 << 24)
    ap.add_argument("--path", type=int, default=0, help="path id (0: all-T)")
    ap.add_argument("--fp64", action="store_true")
    ap.add_argument("--tag", default="")
    a = ap.parse_args()
    cfg = C.CONFIGS[a.config]
    lens = plt.Lens(C.lens_text(a.config), **cfg["opts"])
    pid = a.path or lens.all_t_id()
    law = dict(cfg["law"])
    if "channels" in cfg:
        law["lam"] = cfg["channels"][1]
    d = plt.gen_rays(PX.law_constants(law), 12345, 0, a.rays, with_dz=False)
    h = plt.alloc_hits(a.rays)
    prec = plt.FP64 if a.fp64 else plt.FP32
    run = lambda: plt.trace_rays(lens, pid, d, h, direction=cfg["direction"], precision=prec)
    for _ in range(5):
        run()
    torch.cuda.synchronize()
    ts = []
    for _ in range(20):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        run()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = statistics.median(ts)
    hf = plt.alloc_hits(a.rays, flags=True)   # guard-band rays = the float64 re-trace list
    plt.trace_rays(lens, pid, d, hf, direction=cfg["direction"], precision=prec)
    torch.cuda.synchronize()
    flagged = float(hf["flags"].float().mean())
    print(json.dumps({"tag": a.tag, "config": a.config, "path": pid, "rays": a.rays, "fp64": a.fp64, "ms": ms,
                      "M_rays_s": a.rays / ms / 1e3, "kernel": plt.trace_kernel(lens, pid, cfg["direction"], prec),
                      "split_delta": os.environ.get("PLT_TRACE_SPLIT_DELTA", "0"), "flagged_frac": flagged,
                      "jit_defines": os.environ.get("PLT_JIT_DEFINES", "")}), flush=True)


if __name__ == "__main__":
    main()
