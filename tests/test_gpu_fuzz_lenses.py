"""Fuzz parity: seeded random air-spaced lenses (plt_inputs.lenses.random_lens_text: 2-3
singlet / cemented elements, both radius signs, Abbe / Cauchy / Sellmeier glasses, a stop
somewhere) traced by the library -- the run-time specialised fp32 kernel (whose constant
folding and fitted eta(lambda) polynomials are lens-specific), the float64 kernel, and a
ghost path -- against the float64 oracle under the same rules as tests/test_gpu_trace.py."""
import pytest

import oracle
from plt_inputs import rays as R
from plt_inputs.lenses import random_lens_text

from gpu_helpers import compare_trace, gpu_trace

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("seed", range(8))
def test_random_lens_parity(gpu_lib, seed):
    plt = gpu_lib
    text, semi, z_last = random_lens_text(seed)
    opts = {"sensor_z_mm": z_last + 40.0}
    gl, ol = plt.Lens(text, **opts), oracle.load_lens(text, opts)
    law = {"kind": "disc_cap", "plane_z": -5.0, "disc_r": 0.9 * semi, "cap_deg": 8.0, "lam": (400.0, 700.0)}
    rays = R.gen_rays(law, 1000 + seed, 0, (1 << 15) + 19)
    pid = gl.all_t_id()
    o = oracle.trace(ol, pid, 0, rays, threads=oracle.host_threads())
    st = compare_trace(gpu_trace(plt, gl, pid, rays, precision=0), o)
    assert st["n_both"] > 100, st
    compare_trace(gpu_trace(plt, gl, pid, rays, precision=1), o)
    ids, _ = gl.enumerate_ghosts(2)
    g = int(ids[1 + seed % (len(ids) - 1)])
    og = oracle.trace(ol, g, 0, rays, threads=oracle.host_threads())
    compare_trace(gpu_trace(plt, gl, g, rays, precision=1), og, tol_p=5e-5)


@pytest.mark.parametrize("seed", range(4))
def test_random_lens_backward_parity(gpu_lib, seed):
    """Backward (sensor -> object) traces of the same random lenses: rays leave the sensor
    plane along the reversed exit directions of a forward oracle trace (so most of them
    pass), library fp32 / fp64 vs the oracle's backward trace."""
    import numpy as np
    plt = gpu_lib
    text, semi, z_last = random_lens_text(seed)
    opts = {"sensor_z_mm": z_last + 40.0, "backward_exit_z_mm": -5.0}
    gl, ol = plt.Lens(text, **opts), oracle.load_lens(text, opts)
    law = {"kind": "disc_cap", "plane_z": -5.0, "disc_r": 0.9 * semi, "cap_deg": 8.0, "lam": (400.0, 700.0)}
    fw = R.gen_rays(law, 2000 + seed, 0, 1 << 15)
    pid = gl.all_t_id()
    o = oracle.trace(ol, pid, 0, fw)
    v = o["valid"]
    rays = {"ox": o["px"][v].astype(np.float32), "oy": o["py"][v].astype(np.float32),
            "dx": (-o["dx"][v]).astype(np.float32), "dy": (-o["dy"][v]).astype(np.float32),
            "dz": (-o["dz"][v]).astype(np.float32), "lambda_nm": fw["lambda_nm"][v].copy(),
            "plane_z": z_last + 40.0}
    ob = oracle.trace(ol, pid, 1, rays, threads=oracle.host_threads())
    assert ob["valid"].mean() > 0.5
    compare_trace(gpu_trace(plt, gl, pid, rays, direction=1, precision=0), ob)
    compare_trace(gpu_trace(plt, gl, pid, rays, direction=1, precision=1), ob)
