"""The host-batch path (paper_2605_04017_b200.pipeline.query_host_batch: chunked H2D on a
copy stream overlapping the kernels) produces exactly the film and hits of the
device-resident path on the same rays (int64 film: bit-identical)."""
import numpy as np
import pytest

from plt_inputs import configs as C
from plt_inputs import rays as R

pytestmark = pytest.mark.gpu

FILM = {"width_px": 768, "height_px": 512, "channels": 1, "sensor_w_mm": 36.0, "sensor_h_mm": 24.0,
        "center_x_mm": 0.0, "center_y_mm": 0.0}


@pytest.mark.parametrize("fused", [True, False], ids=["fused", "separate"])
@pytest.mark.parametrize("n,chunk", [((1 << 20) + 77, 1 << 18), (5000, 1024), (64, 32)])
def test_host_batch_matches_device_path(gpu_lib, n, chunk, fused):
    import torch
    from paper_2605_04017_b200.pipeline import query_host_batch
    plt = gpu_lib
    cfg = C.CONFIGS["C2"]
    lens = plt.Lens(C.lens_text("C2"), **cfg["opts"])
    pid = lens.all_t_id()
    m = plt.Map(C.fitted_map_blob("C2"), lens=lens)
    rays = R.gen_rays(cfg["law"], 77, 0, n)
    # device-resident reference
    d = plt.rays_to_device(rays)
    ht, hm = plt.alloc_hits(n), plt.alloc_hits(n)
    film_ref = torch.zeros(512 * 768, dtype=torch.int64, device="cuda")
    plt.trace_rays(lens, pid, d, ht)
    plt.eval_map(m, d, hm)
    plt.splat_sensor(FILM, film_ref, ht, weight_scale=0.5)
    plt.splat_sensor(FILM, film_ref, hm, weight_scale=0.5)
    # host batch
    host = {k: torch.from_numpy(rays[k]).pin_memory() for k in plt.RAY_KEYS}
    host["plane_z"] = rays["plane_z"]
    d2 = {k: torch.full((n,), float("nan"), device="cuda") for k in plt.RAY_KEYS}
    ht2, hm2 = plt.alloc_hits(n), plt.alloc_hits(n)
    film = torch.zeros_like(film_ref)
    film_host = torch.empty(film.numel(), dtype=torch.int64).pin_memory()
    query_host_batch(lens, pid, m, host, d2, ht2, hm2, FILM, film, film_host, weight_scale=0.5, chunk=chunk,
                     fused=fused)
    torch.cuda.synchronize()
    assert torch.equal(film_host, film_ref.cpu())
    for a, b in ((ht, ht2), (hm, hm2)):
        nw = (n + 31) // 32
        assert torch.equal(a["mask_bits"][:nw], b["mask_bits"][:nw])
        for k in plt.HIT_KEYS:
            assert torch.equal(a[k], b[k]), k
