"""Degenerate inputs on the GPU through the C ABI: empty batches are no-ops for every
compute entry point (nothing written, no launch errors), rays that miss the lens entirely
or arrive exactly along the axis behave as the oracle says."""
import numpy as np
import pytest

import oracle
from plt_inputs import configs as C

from gpu_helpers import compare_trace, gpu_trace

pytestmark = pytest.mark.gpu


def test_empty_batches_are_no_ops(gpu_lib):
    import torch
    plt = gpu_lib
    cfg = C.CONFIGS["C2"]
    lens = plt.Lens(C.lens_text("C2"), **cfg["opts"])
    m = plt.Map(C.fitted_map_blob("C2"), lens=lens)
    d = {k: torch.zeros(1, dtype=torch.float32, device="cuda") for k in plt.RAY_KEYS}
    d["plane_z"] = -5.0
    h = plt.alloc_hits(1)
    for k in plt.HIT_KEYS:
        h[k].fill_(7.0)
    film = torch.full((768 * 512,), 5, dtype=torch.int64, device="cuda")
    fd = {"width_px": 768, "height_px": 512, "channels": 1, "sensor_w_mm": 36.0, "sensor_h_mm": 24.0}
    spl = {"film_desc": fd, "film": film, "weight_scale": 1.0}
    for prec in (plt.FP32, plt.FP64):
        plt.trace_rays(lens, lens.all_t_id(), d, h, precision=prec, n=0)
        plt.trace_rays(lens, lens.all_t_id(), d, h, precision=prec, n=0, splat=spl)
    plt.eval_map(m, d, h, n=0)
    plt.eval_map(m, d, h, n=0, splat=spl)
    plt.splat_sensor(fd, film, h, n=0)
    plt.shade_plane({"z_mm": -1000.0, "period_mm": 50.0, "contrast": 0.1}, -5.0, h, film, 4, n=0)
    plt.propagate_rays(d, {k: d[k] for k in plt.RAY_KEYS}, 10.0, n=0)
    torch.cuda.synchronize()
    assert all(bool((h[k] == 7.0).all()) for k in plt.HIT_KEYS)
    assert bool((film == 5).all())


def test_rays_missing_the_lens_and_axial_rays(gpu_lib):
    """Rays far outside the front aperture are invalid with all-zero outputs; exactly axial
    rays (p = 0, w = +z) pass the all-T path undeviated (p_out = 0) with the oracle's
    throughput; a ray parallel to the input plane (w_z = 0) is invalid."""
    plt = gpu_lib
    cfg = C.CONFIGS["C2"]
    gl = plt.Lens(C.lens_text("C2"), **cfg["opts"])
    ol = oracle.load_lens(C.lens_text("C2"), cfg["opts"])
    n = 96
    ox = np.zeros(n, np.float32)
    ox[:32] = 50.0                                   # outside every aperture
    dx = np.zeros(n, np.float32)
    dz = np.ones(n, np.float32)
    dx[64:], dz[64:] = 1.0, 0.0                      # grazing: parallel to the plane
    rays = {"ox": ox, "oy": np.zeros(n, np.float32), "dx": dx, "dy": np.zeros(n, np.float32), "dz": dz,
            "lambda_nm": np.linspace(400, 700, n).astype(np.float32), "plane_z": -5.0}
    for prec in (0, 1):
        g = gpu_trace(plt, gl, gl.all_t_id(), rays, precision=prec)
        o = oracle.trace(ol, gl.all_t_id(), 0, rays)
        compare_trace(g, o, excluded_max=32)           # the 32 grazing rays have |w_z| = 0
        assert not g["valid"][:32].any() and g["valid"][32:64].all() and not g["valid"][64:].any()
        assert np.abs(g["px"][32:64]).max() == 0.0 and np.abs(g["py"][32:64]).max() == 0.0


def test_total_internal_reflection_and_sphere_misses(gpu_lib):
    """Eq. 6-7 branches the kernels take without a comparison of their own (DESIGN.md "Misses
    and TIR die through NaN"): a ray missing a spherical cap (disc < 0) and a ray totally
    internally reflected on a transmission step (A6: absorbed) are invalid with zero outputs,
    exactly as the oracle's explicit tests (pinned in test_oracle_trace) decide, in fp32 and
    fp64 (the generic packed and scalar fp32 kernels: the same test under PLT_TRACE_JIT=0 /
    PLT_TRACE_X1=1).  Lens: n = 2 front cap (R = 10 mm) + planar rear; parallel rays at
    heights 0 ... 12 mm: below 7.14 mm they transmit, higher ones are bent past the 30 deg
    critical angle at the rear face, above 10 mm they miss the cap."""
    plt = gpu_lib
    text = "name tir\n10 3.0 n:2.0 20\n0 0 air 40\n"
    opts = {"sensor_z_mm": 20.0}
    gl = plt.Lens(text, **opts)
    ol = oracle.load_lens(text, opts)
    n = 4096
    rng = np.random.default_rng(5)
    h = np.linspace(0.0, 12.0, n)
    phi = rng.uniform(0, 2 * np.pi, n)
    rays = {"ox": (h * np.cos(phi)).astype(np.float32), "oy": (h * np.sin(phi)).astype(np.float32),
            "dx": np.zeros(n, np.float32), "dy": np.zeros(n, np.float32), "dz": np.ones(n, np.float32),
            "lambda_nm": rng.uniform(400, 700, n).astype(np.float32), "plane_z": -5.0}
    pid = gl.all_t_id()
    o = oracle.trace(ol, pid, 0, rays)
    assert o["valid"][h < 7.0].all()                     # transmitted
    assert not o["valid"][(h > 7.3) & (h < 9.99)].any()   # TIR at the rear face
    assert not o["valid"][h > 10.01].any()               # misses the cap
    for prec in (plt.FP32, plt.FP64):
        compare_trace(gpu_trace(plt, gl, pid, rays, precision=prec), o)
