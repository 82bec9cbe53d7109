"""GPU parity on even-aspheric lenses against the oracle:
the run-time specialised all-T kernel, the generic packed kernel (a ghost path), and
float64, on an aspheric singlet and on the 50 mm double-Gauss with an aspheric front
surface (C2 ray law)."""
import numpy as np
import pytest

import oracle
from plt_inputs import configs as C
from plt_inputs import rays as R
from plt_inputs.lenses import LENSES

from gpu_helpers import compare_trace, gpu_trace

pytestmark = pytest.mark.gpu

ASPH_SINGLET = """name asph_singlet
0       5.0  stop                     16.0
50.0    5.0  sellmeier:1.03961212,0.231792344,1.01046945,0.00600069867,0.0200179144,103.560653  25.0  asph:-0.8,2e-6,-3e-9
-50.0   0.0  air                      25.0
"""


def _asph_dgauss():
    out, done = [], False
    for line in LENSES["dgauss50"].splitlines():
        body = line.split("#", 1)[0].split()
        if not done and len(body) >= 4 and body[0] != "name" and float(body[0]) != 0.0:
            line = line.split("#", 1)[0].rstrip() + "  asph:-0.3,-4e-6,2e-9"
            done = True
        out.append(line)
    return "\n".join(out) + "\n"


@pytest.mark.parametrize("which", ["singlet", "dgauss50"])
def test_aspheric_lens_parity(gpu_lib, which):
    plt = gpu_lib
    if which == "singlet":
        text, cfg = ASPH_SINGLET, C.CONFIGS["C1"]
        rays = R.gen_rays(cfg["law"], 21, 0, (1 << 16) + 11)
        rays["lambda_nm"] = np.random.default_rng(2).uniform(400, 700, rays["ox"].size).astype(np.float32)
    else:
        text, cfg = _asph_dgauss(), C.CONFIGS["C2"]
        rays = R.gen_rays(cfg["law"], 21, 0, (1 << 17) + 11)
    gl, ol = plt.Lens(text, **cfg["opts"]), oracle.load_lens(text, cfg["opts"])
    assert abs(gl.info()["sensor_z_mm"] - ol.opts["sensor_z_mm"]) < 1e-9
    pid = gl.all_t_id()
    o = oracle.trace(ol, pid, 0, rays, threads=oracle.host_threads())
    st = compare_trace(gpu_trace(plt, gl, pid, rays, precision=0), o)            # JIT-specialised fp32
    assert st["n_both"] > 1000 and st["max_dp"] <= 1e-4 and st["max_dw"] <= 1e-5 and st["max_dI"] <= 1e-5
    compare_trace(gpu_trace(plt, gl, pid, rays, precision=1), o, tol_p=4e-6, tol_w=2e-7, tol_i=2e-7)
    ids, _ = gl.enumerate_ghosts(2)
    g = int(ids[len(ids) // 2])
    og = oracle.trace(ol, g, 0, rays, threads=oracle.host_threads())
    # ghost exits land up to ~330 mm off-axis on the unbounded C1 sensor: float32 storage of
    # the position rounds at ~3e-5 mm there
    compare_trace(gpu_trace(plt, gl, g, rays, precision=1), og, tol_p=5e-5, tol_w=2e-7, tol_i=2e-7)
    s32 = compare_trace(gpu_trace(plt, gl, g, rays, precision=0), og, assert_ok=False)   # generic packed
    assert s32["mask_mismatch"] <= max(2, int(1e-3 * og["valid"].sum()))


def test_coated_lens_parity(gpu_lib):
    """Single-layer AR coatings (NEXT-4) on every air-glass surface of the double-Gauss and
    an aspheric front: the all-T path (JIT) and a ghost (fp64, generic packed fp32) against
    the oracle; the coated ghost is much dimmer than the bare one."""
    import sys
    import os
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from test_abi_cpu import _coated
    plt = gpu_lib
    cfg = C.CONFIGS["C2"]
    text = _coated(_asph_dgauss())
    gl, ol = plt.Lens(text, **cfg["opts"]), oracle.load_lens(text, cfg["opts"])
    rays = R.gen_rays(cfg["law"], 23, 0, (1 << 17) + 7)
    pid = gl.all_t_id()
    o = oracle.trace(ol, pid, 0, rays, threads=oracle.host_threads())
    st = compare_trace(gpu_trace(plt, gl, pid, rays, precision=0), o)
    assert st["n_both"] > 1000
    ids, _ = gl.enumerate_ghosts(2)
    g = int(ids[len(ids) // 2])
    og = oracle.trace(ol, g, 0, rays, threads=oracle.host_threads())
    compare_trace(gpu_trace(plt, gl, g, rays, precision=1), og, tol_p=4e-6, tol_w=2e-7, tol_i=2e-7)
    s32 = compare_trace(gpu_trace(plt, gl, g, rays, precision=0), og, assert_ok=False)
    assert s32["mask_mismatch"] <= max(2, int(1e-3 * og["valid"].sum())) and s32["max_dI"] <= 1e-5
    bare = oracle.trace(oracle.load_lens(_asph_dgauss(), cfg["opts"]), g, 0, rays, threads=oracle.host_threads())
    v = og["valid"] & bare["valid"]
    assert v.sum() > 100 and og["I"][v].mean() < 0.5 * bare["I"][v].mean()


def test_backward_aspheric_coated_parity(gpu_lib):
    """Backward (camera) traces through the 24 mm lens with an aspheric, coated element:
    the mirrored frame negates the sag (pinned by oracle reciprocity); GPU fp32 (JIT) and
    fp64 against the oracle."""
    plt = gpu_lib
    cfg = C.CONFIGS["C3"]
    lines, k = [], 0
    for line in LENSES["wide24"].splitlines():
        body = line.split("#", 1)[0].split()
        if len(body) >= 4 and body[0] != "name" and body[2].lower() != "stop" and float(body[0]) != 0.0:
            k += 1
            if k == 3:
                line = line.split("#", 1)[0].rstrip() + " asph:-0.5,3e-5,-1e-7 coat:1.38,550"
        lines.append(line)
    text = "\n".join(lines) + "\n"
    gl, ol = plt.Lens(text, **cfg["opts"]), oracle.load_lens(text, cfg["opts"])
    rays = R.gen_rays(cfg["law"], 31, 0, (1 << 17) + 3)
    pid = gl.all_t_id()
    o = oracle.trace(ol, pid, 1, rays, threads=oracle.host_threads())
    st = compare_trace(gpu_trace(plt, gl, pid, rays, direction=1, precision=0), o)
    assert st["n_both"] > 2000
    compare_trace(gpu_trace(plt, gl, pid, rays, direction=1, precision=1), o, tol_p=4e-6, tol_w=2e-7, tol_i=2e-7)
