"""Dev probe: time splat_sensor on the C2 trace hits (bench film, scale 1.0 and 2^-24)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2605_04017_b200 as plt  # noqa: E402
from plt_inputs import configs as C  # noqa: E402
from plt_inputs import rays as R  # noqa: E402

FILM = {"width_px": 768, "height_px": 512, "channels": 1, "sensor_w_mm": 36.0, "sensor_h_mm": 24.0,
        "center_x_mm": 0.0, "center_y_mm": 0.0}


def main():
    n = 1 << 24
    cfg = C.CONFIGS["C2"]
    lens = plt.Lens(C.lens_text("C2"), **cfg["opts"])
    d = plt.rays_to_device(R.gen_rays(cfg["law"], cfg["seed"], 0, n))
    h = plt.alloc_hits(n)
    plt.trace_rays(lens, lens.all_t_id(), d, h)
    film = torch.zeros(512 * 768, dtype=torch.int64, device="cuda")
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    out = []
    for scale in (1.0, 2.0 ** -24, 1.0 / 3.0):
        for _ in range(3):
            plt.splat_sensor(FILM, film, h, weight_scale=scale)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(20):
            plt.splat_sensor(FILM, film, h, weight_scale=scale)
        e1.record()
        torch.cuda.synchronize()
        out.append(f"scale {scale:.3g}: {e0.elapsed_time(e1) / 20 * 1e3:.1f} us")
    print(os.path.basename(plt.LIB_PATH), os.environ.get("PLT_SPLAT_NOPOW2", ""), " | ".join(out))


if __name__ == "__main__":
    main()
