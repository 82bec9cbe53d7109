"""Probe: the C2 bench step (trace + map of the same 2^24 rays, both splatted in-kernel) with
the two kernels back to back on one stream vs forked onto two streams (eval_map first, the
trace filling SMs as eval_map's persistent CTAs drain), median of 30 after 5 warm-ups."""
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

cfg = C.CONFIGS["C2"]
lens = plt.Lens(C.lens_text("C2"), **cfg["opts"])
m = plt.Map(C.fitted_map_blob("C2"), lens=lens)
n = 1 << 24
d = plt.gen_rays(PX.law_constants(cfg["law"]), 2, 0, n, with_dz=False)
ht, hm = plt.alloc_hits(n), plt.alloc_hits(n)
fd = {"width_px": 768, "height_px": 512, "channels": 1, "sensor_w_mm": 36.0, "sensor_h_mm": 24.0,
      "center_x_mm": 0.0, "center_y_mm": 0.0}
film = torch.zeros(768 * 512, dtype=torch.int64, device="cuda")
spl = {"film_desc": fd, "film": film, "weight_scale": 1.0 / n}
pid = lens.all_t_id()
main = torch.cuda.current_stream()
side = torch.cuda.Stream()


def seq():
    plt.trace_rays(lens, pid, d, ht, splat=spl)
    plt.eval_map(m, d, hm, splat=spl)


def par(map_first=True):
    f = torch.cuda.Event()
    f.record(main)
    side.wait_event(f)
    if map_first:
        plt.eval_map(m, d, hm, splat=spl)
        plt.trace_rays(lens, pid, d, ht, splat=spl, stream=side)
    else:
        plt.trace_rays(lens, pid, d, ht, splat=spl)
        plt.eval_map(m, d, hm, splat=spl, stream=side)
    j = torch.cuda.Event()
    j.record(side)
    main.wait_event(j)


def t(fn):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(30):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


res = {"sequential": t(seq), "map_first_trace_side": t(lambda: par(True)), "trace_first_map_side": t(lambda: par(False))}
print(json.dumps({k: round(v, 4) for k, v in res.items()}))
