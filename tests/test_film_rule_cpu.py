"""CPU checks of the per-pixel film rule used by the end-to-end film parity tests
(tests/gpu_helpers.film_pixel_bound; SURVEY §8(c) film rule 2): hits perturbed within the
stated tolerances always pass, a perturbation beyond them or a mirrored image fails."""
import numpy as np

import oracle
from plt_inputs import configs as C

from gpu_helpers import assert_film_within_bound, film_pixel_bound, near_edge


def _setup(n=1 << 16):
    cfg = C.CONFIGS["C4_59"]
    ol = oracle.load_lens(C.lens_text("C4_59"), cfg["opts"])
    rays = C.flare_rays("C4_59", 0, 0, n)
    o = oracle.trace(ol, 16404, 0, rays, threads=oracle.host_threads())
    fd = dict(cfg["film"], channels=1)
    return o, fd, 1.0 / n


def _film(fd, h, scale):
    f, _ = oracle.splat(fd, h["valid"], h["px"].astype(np.float32), h["py"].astype(np.float32),
                        h["dz"].astype(np.float32), h["I"].astype(np.float32), None, scale=scale)
    return f


def test_perturbation_within_tolerance_passes():
    o, fd, s = _setup()
    rng = np.random.default_rng(5)
    g = {k: o[k].copy() for k in ("valid", "px", "py", "dz", "I")}
    n = g["px"].size
    for k, t in (("px", 4e-6), ("py", 4e-6), ("dz", 2e-7), ("I", 2e-7)):
        g[k] = g[k] + rng.uniform(-t, t, n) * g["valid"]
    b = film_pixel_bound(fd, s, o, g, near_edge(o["margins"]), 4e-6, 2e-7)
    st = assert_film_within_bound(_film(fd, g, s), _film(fd, o, s), b, max_rel_bound=0.05)
    assert st["pixels_diff"] > 0        # the perturbation did flip some bins


def test_violations_fail():
    o, fd, s = _setup()
    f_o = _film(fd, o, s)
    b = film_pixel_bound(fd, s, o, o, near_edge(o["margins"]), 4e-6, 2e-7)
    for k, fn in (("py", lambda v: -v), ("px", lambda v: v + 2e-4), ("I", lambda v: v + 5e-5)):
        g = {kk: o[kk].copy() for kk in ("valid", "px", "py", "dz", "I")}
        g[k] = fn(g[k])
        d = np.abs(_film(fd, g, s).astype(np.float64) - f_o).reshape(b.shape)
        assert (d > b).any(), k
    # dropping 1 % of the valid rays
    g = {kk: o[kk].copy() for kk in ("valid", "px", "py", "dz", "I")}
    idx = np.nonzero(g["valid"])[0][::100]
    g["valid"][idx] = False
    d = np.abs(_film(fd, g, s).astype(np.float64) - f_o).reshape(b.shape)
    assert (d > b).any()
