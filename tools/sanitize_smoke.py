"""Small exercise of every kernel for compute-sanitizer (memcheck / racecheck / synccheck)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2605_04017_b200 as plt  # noqa: E402
from plt_inputs import configs as C  # noqa: E402
from plt_inputs import rays as R  # noqa: E402

cfg = C.CONFIGS["C2"]
lens = plt.Lens(C.lens_text("C2"), **cfg["opts"])
pid = lens.all_t_id()
m = plt.Map(C.map_blob("C2", pid))
for n in (1, 37, 4096 + 37):
    rays = plt.rays_to_device(R.gen_rays(cfg["law"], 5, 0, n))
    h = plt.alloc_hits(n, flags=True)
    plt.trace_rays(lens, pid, rays, h)
    plt.trace_rays(lens, pid, rays, h, precision=plt.FP64)
    raw = torch.empty(7 * n, device="cuda")
    plt.eval_map(m, rays, h, raw=raw)
    fd = {"width_px": 64, "height_px": 48, "channels": 1, "sensor_w_mm": 36.0, "sensor_h_mm": 24.0}
    film = torch.zeros(64 * 48, dtype=torch.int64, device="cuda")
    plt.splat_sensor(fd, film, h, weight_scale=1.0)
    out = torch.empty(64 * 48, device="cuda")
    plt.film_resolve(fd, film, out)
    # fused query + splat, camera shading and propagation
    spl = {"film_desc": fd, "film": film, "weight_scale": 1.0}
    plt.trace_rays(lens, pid, rays, h, splat=spl)
    plt.trace_rays(lens, pid, rays, h, precision=plt.FP64, splat=spl)
    plt.eval_map(m, rays, h, splat=spl)
    plt.shade_plane({"z_mm": -1000.0, "period_mm": 50.0, "contrast": 0.1}, -5.0, h, film, 3)
    dst = {k: torch.empty_like(rays[k]) for k in plt.RAY_KEYS}
    plt.propagate_rays(rays, dst, -4.0, direction=plt.BACKWARD)
torch.cuda.synchronize()
print("sanitize smoke done")
