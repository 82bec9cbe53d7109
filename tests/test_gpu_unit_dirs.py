"""GPU parity for rays given without dz (plt_rays.dz == NULL: omega in S^2_+ of P:180 given
by (dx, dy); include/plt.h).  The kernels complete w_z per ray in their own precision
(fp32 passes in fp32, fp64 passes and the guard-band re-trace in fp64); the oracle
completes it in float64 (oracle.hemisphere_dz).  Same tolerances as tests/test_gpu_trace.py."""
import numpy as np
import pytest

import oracle
from plt_inputs import configs as C
from plt_inputs import rays as R

from gpu_helpers import compare_trace, gpu_trace

pytestmark = pytest.mark.gpu


def _no_dz(rays):
    return {k: v for k, v in rays.items() if k != "dz"}


@pytest.mark.parametrize("name,direction,precision", [("C2", 0, 0), ("C2", 0, 1), ("C3", 1, 0), ("C3", 1, 1)])
def test_all_t_trace_without_dz(gpu_lib, name, direction, precision):
    plt = gpu_lib
    cfg = C.CONFIGS[name]
    gl = plt.Lens(C.lens_text(name), **cfg["opts"])
    ol = oracle.load_lens(C.lens_text(name), cfg["opts"])
    rays = _no_dz(R.gen_rays(cfg["law"], 41, 0, (1 << 18) + 77))
    pid = gl.all_t_id()
    g = gpu_trace(plt, gl, pid, rays, direction=direction, precision=precision)
    o = oracle.trace(ol, pid, direction, rays, threads=oracle.host_threads())
    st = compare_trace(g, o)
    assert st["n_both"] > 1000


def test_ghost_fp64_without_dz(gpu_lib):
    plt = gpu_lib
    cfg = C.CONFIGS["C4_22"]
    gl = plt.Lens(C.lens_text("C4_22"), **cfg["opts"])
    ol = oracle.load_lens(C.lens_text("C4_22"), cfg["opts"])
    rays = _no_dz(R.gen_rays(cfg["law"], 42, 0, 1 << 17))
    g = gpu_trace(plt, gl, 65616, rays, precision=1)
    o = oracle.trace(ol, 65616, 0, rays, threads=oracle.host_threads())
    st = compare_trace(g, o, tol_p=5e-5)
    assert st["n_both"] > 100


def test_eval_map_ignores_dz(gpu_lib):
    """The map's canonical input is (r, w'_x, w'_y, lambda) (O10): dz NULL is bit-identical."""
    import torch
    plt = gpu_lib
    cfg = C.CONFIGS["C2"]
    gl = plt.Lens(C.lens_text("C2"), **cfg["opts"])
    m = plt.Map(C.fitted_map_blob("C2"), lens=gl)
    rays = R.gen_rays(cfg["law"], 43, 0, (1 << 18) + 5)
    n = rays["ox"].size
    outs = []
    for with_dz in (True, False):
        d = plt.rays_to_device(rays, with_dz=with_dz)
        h = plt.alloc_hits(n)
        plt.eval_map(m, d, h)
        torch.cuda.synchronize()
        outs.append({k: h[k].cpu() for k in ("mask_bits", "px", "py", "dx", "dy", "dz", "throughput")})
    for k in outs[0]:
        assert torch.equal(outs[0][k], outs[1][k]), k


def test_propagate_without_dz(gpu_lib):
    """plt_propagate_rays with in->dz == out->dz == NULL vs the float64 oracle: backward
    (sensor) rays moved along their lines upstream and downstream (the sensor-shift
    focusing of P:425-427; w_z takes the query direction's sign, as in the trace)."""
    import torch
    plt = gpu_lib
    cfg = C.CONFIGS["C3_DOF"] if "C3_DOF" in C.CONFIGS else C.CONFIGS["C3"]
    rays = _no_dz(R.gen_rays(cfg["law"], 44, 0, 1 << 16))
    n = rays["ox"].size
    d = plt.rays_to_device(rays)
    out = {k: torch.empty(n, dtype=torch.float32, device="cuda") for k in ("ox", "oy", "dx", "dy", "lambda_nm")}
    out["dz"] = None
    z0 = float(rays["plane_z"])
    # backward sensor rays (w_z < 0) moved both downstream and upstream of their plane
    for zt in (z0 + 1.5, z0 - 1.0):
        plt.propagate_rays(d, out, zt, direction=plt.BACKWARD)
        torch.cuda.synchronize()
        o = oracle.propagate(rays, zt, direction=oracle.BACKWARD)
        for k in ("ox", "oy"):
            err = np.abs(out[k].cpu().numpy().astype(np.float64) - o[k])
            assert err.max() < 2e-5 * (1.0 + np.abs(o[k]).max()), (zt, k, err.max())
        for k in ("dx", "dy", "lambda_nm"):
            assert np.array_equal(out[k].cpu().numpy(), rays[k]), k


def test_host_query_without_dz(gpu_lib):
    """plt_query_host moving 20 B per ray (no dz) gives the film of the device-resident
    query on the same dz-less rays, bit for bit."""
    import torch
    plt = gpu_lib
    cfg = C.CONFIGS["C2"]
    gl = plt.Lens(C.lens_text("C2"), **cfg["opts"])
    m = plt.Map(C.fitted_map_blob("C2"), lens=gl)
    n = (1 << 20) + 64
    rays = R.gen_rays(cfg["law"], 45, 0, n)
    fd = {"width_px": 256, "height_px": 128, "channels": 1, "sensor_w_mm": 36.0, "sensor_h_mm": 24.0}
    host = {k: torch.from_numpy(rays[k]).pin_memory() for k in plt.RAY_KEYS if k != "dz"}
    host["plane_z"] = rays["plane_z"]
    film = torch.zeros(256 * 128, dtype=torch.int64, device="cuda")
    fh = torch.empty_like(film, device="cpu").pin_memory()
    plt.query_host(gl, gl.all_t_id(), m, host, fd, film, fh, weight_scale=1.0 / n, chunk=1 << 18)
    torch.cuda.synchronize()
    ref = torch.zeros_like(film)
    dd = plt.rays_to_device(rays, with_dz=False)
    h2 = plt.alloc_hits(n)
    spl = {"film_desc": fd, "film": ref, "weight_scale": 1.0 / n}
    plt.trace_rays(gl, gl.all_t_id(), dd, h2, splat=spl)
    plt.eval_map(m, dd, h2, splat=spl)
    torch.cuda.synchronize()
    assert torch.equal(fh, ref.cpu())
    assert int(ref.sum()) > 0
