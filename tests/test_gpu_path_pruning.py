"""GPU ghost pruning by measured path flux (render.path_energies / prune_paths, SURVEY §8(f)
NEXT-4): per-path energies from the fused one-pixel splat of the float64 trace against the
oracle's trace + splat on the same rays, for two- and four-bounce paths."""
import numpy as np
import pytest

import oracle
from plt_inputs import configs as C
from plt_inputs import rays as R

pytestmark = pytest.mark.gpu


def test_path_energies_and_prune_match_oracle(gpu_lib):
    from paper_2605_04017_b200.render import path_energies, prune_paths
    plt = gpu_lib
    cfg = C.CONFIGS["C4_59"]
    gl = plt.Lens(C.lens_text("C4_59"), **cfg["opts"])
    ol = oracle.load_lens(C.lens_text("C4_59"), cfg["opts"])
    rays = C.flare_rays("C4_59", 0, 0, 1 << 14)
    d = plt.rays_to_device(rays)
    ids2, _ = gl.enumerate_ghosts(2)
    ids4, _ = gl.enumerate_ghosts(4, 1e-7)
    four = sorted(set(ids4) - set(ids2))[:40]
    paths = [int(p) for p in ids2[1:]] + four
    e = path_energies(gl, paths, d)
    whole = {"width_px": 1, "height_px": 1, "channels": 1, "sensor_w_mm": 1e9, "sensor_h_mm": 1e9,
             "center_x_mm": 0.0, "center_y_mm": 0.0}
    eo = []
    for p in paths:
        t = oracle.trace(ol, p, 0, rays, threads=oracle.host_threads())
        f, _ = oracle.splat(whole, t["valid"], t["px"].astype(np.float32), t["py"].astype(np.float32),
                            t["dz"].astype(np.float32), t["I"].astype(np.float32), None, 1.0)
        eo.append(float(f.sum()) / 4294967296.0)
    e, eo = np.array(e), np.array(eo)
    assert np.all(eo >= 0) and eo.max() > 0
    # fp64 GPU vs oracle: same valid sets; per-ray outputs agree to output rounding
    assert np.allclose(e, eo, rtol=1e-5, atol=1e-9 * eo.max()), np.abs(e - eo).max()
    kept, en = prune_paths(gl, paths, d, 1e-3)
    ref = path_energies(gl, [gl.all_t_id()], d)[0]
    expect = [p for p, v in zip(paths, eo) if v >= 1e-3 * ref]
    near = [p for p, v in zip(paths, eo) if abs(v - 1e-3 * ref) <= 1e-4 * ref]
    assert set(kept) ^ set(expect) <= set(near)
    assert 0 < len(kept) < len(paths)
