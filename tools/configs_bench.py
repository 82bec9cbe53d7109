"""Per-configuration throughput and roofline fractions of the CUDA path on one B200
(BASELINE.json configs C1-C5).

    python tools/configs_bench.py [--out profiles/r02_configs.json] [--quick]

C2, C3, C4_22, C4_59 and every C5 sweep size run through `bench.py --config ...` (the
driver's contract: W warm-ups, K timed steps, CUDA events on the launching stream, NVML
clocks) -- each JSON line carries the per-kernel times, the roofline of every kernel and of
the dominant one.  C3 (805 M rays) and C5 (up to 2^30 rays) are generated on the device at
full size by plt_gen_rays (no tiled inputs).  C1 (12,288 rays) is launch-bound; it is timed
eagerly and as a CUDA-graph replay.  Not part of the driver's bench contract.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def bench_line(args: list) -> dict:
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--no-cpu-baseline"] + args
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=1800)
    if out.returncode != 0:
        return {"error": out.stderr[-1500:], "args": args}
    return json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][-1])


def timed(fn, reps=5, warm=2):
    import torch
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) / 1e3)
    return statistics.median(ts)


def c1():
    import torch
    import paper_2605_04017_b200 as plt
    from plt_inputs import configs as C
    cfg = C.CONFIGS["C1"]
    lens = plt.Lens(C.lens_text("C1"), **cfg["opts"])
    d = plt.rays_to_device(C.c1_rays())
    n = d["ox"].numel()
    h = plt.alloc_hits(n)
    flops = json.load(open(os.path.join(ROOT, "profiles", "trace_flops.json")))["configs"]["C1"]["4"]["flops_per_ray"]
    t = timed(lambda: plt.trace_rays(lens, lens.all_t_id(), d, h), reps=20)
    out = [{"config": "C1", "kernel": "trace_rays fp32", "rays": n, "ms": t * 1e3, "M_rays_s": n / t / 1e6,
            "TFLOPs": n * flops / t / 1e12, "note": "launch-latency bound at 12,288 rays (per-call Python + launch)"}]
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            plt.trace_rays(lens, lens.all_t_id(), d, h, stream=s)
    reps = 100
    tg = timed(lambda: [g.replay() for _ in range(reps)], reps=5) / reps
    out.append({"config": "C1", "kernel": "trace_rays fp32, CUDA-graph replay", "rays": n, "ms": tg * 1e3,
                "M_rays_s": n / tg / 1e6, "TFLOPs": n * flops / tg / 1e12,
                "note": "trace + fp64 refine launches replayed from one graph; 12,288 rays cannot fill 148 SMs"})
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--steps", type=int, default=10)
    a = ap.parse_args()
    import torch
    import paper_2605_04017_b200 as plt
    plt.load()
    res = {"gpu": torch.cuda.get_device_name(), "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())}
    res["C1"] = c1()
    st = ["--steps", str(a.steps), "--warmup", "3"]
    for name in ("C2", "C3", "C4_22", "C4_59"):
        if a.quick and name == "C4_59":
            continue
        res[name] = bench_line(["--config", name] + (st if name != "C3" else ["--steps", "3", "--warmup", "3"]))
        print(name, json.dumps({k: res[name].get(k) for k in ("value", "ms_per_step", "roofline")}), flush=True)
    sizes = (20, 24) if a.quick else (20, 22, 24, 26, 28, 30)
    res["C5"] = []
    for k in sizes:
        line = bench_line(["--config", "C5", "--rays", str(1 << k)] + st)
        res["C5"].append(line)
        print("C5 2^%d" % k, json.dumps({x: line.get(x) for x in ("value", "ms_per_step")}), flush=True)
    txt = json.dumps(res, indent=1)
    if a.out:
        with open(a.out, "w") as f:
            f.write(txt + "\n")
    else:
        print(txt)


if __name__ == "__main__":
    main()
