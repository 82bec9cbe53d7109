"""Dev probe: fp64 trace (C2 all-T) and fp64 flare ghost trace + fused splat timings."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2605_04017_b200 as plt  # noqa: E402
from plt_inputs import configs as C  # noqa: E402
from plt_inputs import rays as R  # noqa: E402


def timed(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


cfg = C.CONFIGS["C2"]
lens = plt.Lens(C.lens_text("C2"), **cfg["opts"])
n = 1 << 24
d = plt.rays_to_device(R.gen_rays(cfg["law"], 2, 0, n))
h = plt.alloc_hits(n)
t64 = timed(lambda: plt.trace_rays(lens, lens.all_t_id(), d, h, precision=plt.FP64))
c4 = C.CONFIGS["C4_22"]
gl = plt.Lens(C.lens_text("C4_22"), **c4["opts"])
fd = c4["film"]
npc = 1 << 20
dd = plt.rays_to_device(C.flare_rays("C4_22", 0, 0, npc))
hh = plt.alloc_hits(npc)
film = torch.zeros(3 * 512 * 768, dtype=torch.int64, device="cuda")
ids, _ = gl.enumerate_ghosts(2)
g = ids[1:9]
tf = timed(lambda: [plt.trace_rays(gl, int(x), dd, hh, precision=plt.FP64,
                                   splat={"film_desc": fd, "film": film, "weight_scale": 1.0 / npc}) for x in g], reps=3)
ts = timed(lambda: [(plt.trace_rays(gl, int(x), dd, hh, precision=plt.FP64),
                     plt.splat_sensor(fd, film, hh, weight_scale=1.0 / npc)) for x in g], reps=3)
print(os.path.basename(plt.LIB_PATH), f"C2 fp64 trace {t64:.3f} ms | 8 ghosts fp64 fused {tf:.3f} ms, separate {ts:.3f} ms")
