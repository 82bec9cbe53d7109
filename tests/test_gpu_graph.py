"""The query is CUDA-graph capturable: trace + eval_map (+ fused splat) captured once and
replayed gives the film and hits of eager execution (launch-bound small batches, e.g. C1,
are served by graph replay instead of per-call launches)."""
import numpy as np
import pytest

from plt_inputs import configs as C
from plt_inputs import rays as R

pytestmark = pytest.mark.gpu

FILM = {"width_px": 768, "height_px": 512, "channels": 1, "sensor_w_mm": 36.0, "sensor_h_mm": 24.0,
        "center_x_mm": 0.0, "center_y_mm": 0.0}


@pytest.mark.parametrize("n", [4096 + 17, 1 << 18])
def test_graph_replay_matches_eager(gpu_lib, n):
    import torch
    plt = gpu_lib
    cfg = C.CONFIGS["C2"]
    lens = plt.Lens(C.lens_text("C2"), **cfg["opts"])
    pid = lens.all_t_id()
    m = plt.Map(C.fitted_map_blob("C2"), lens=lens)
    d = plt.rays_to_device(R.gen_rays(cfg["law"], 23, 0, n))
    ht, hm = plt.alloc_hits(n), plt.alloc_hits(n)
    film = torch.zeros(512 * 768, dtype=torch.int64, device="cuda")
    spl = {"film_desc": FILM, "film": film, "weight_scale": 0.25}

    def step(stream):
        film.zero_()
        plt.trace_rays(lens, pid, d, ht, stream=stream, splat=spl)
        plt.eval_map(m, d, hm, stream=stream, splat=spl)

    step(None)                                   # eager (also JIT-compiles / configures kernels)
    torch.cuda.synchronize()
    ref_film = film.clone()
    ref = {k: (ht[k].clone(), hm[k].clone()) for k in plt.HIT_KEYS + ("mask_bits",)}
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        for k in plt.HIT_KEYS:
            ht[k].zero_(); hm[k].zero_()
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            step(s)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    assert torch.equal(film, ref_film)
    for k, (a, b) in ref.items():
        assert torch.equal(ht[k], a) and torch.equal(hm[k], b), k
