"""GPU parity of plt_trace_rays against the float64 oracle (SURVEY.md §8(c) rules).

fp32 mode binds for all-T paths (C1, C2, C3, C5); fp64 mode binds for ghost paths
(C4).  All calls go through the C-ABI binding."""
import numpy as np
import pytest

import oracle
from plt_inputs import configs as C
from plt_inputs import rays as R
from plt_inputs.lenses import LENSES

from gpu_helpers import compare_trace, gpu_trace, unpack_mask

pytestmark = pytest.mark.gpu


def _lenses(plt, name, opts):
    return plt.Lens(LENSES[name], **opts), oracle.load_lens(LENSES[name], opts)


def test_c1_singlet_parity_and_abcd(gpu_lib):
    plt = gpu_lib
    cfg = C.CONFIGS["C1"]
    gl, ol = _lenses(plt, "singlet", cfg["opts"])
    assert abs(gl.info()["sensor_z_mm"] - ol.opts["sensor_z_mm"]) < 1e-9
    rays = C.c1_rays()
    pid = 1 << 2
    g = gpu_trace(plt, gl, pid, rays)
    o = oracle.trace(ol, pid, 0, rays)
    st = compare_trace(g, o)
    assert 0.3 < st["valid_frac"] < 0.9
    # near-axis GPU rays follow the ABCD prediction to third order
    ab = C.c1_abcd_rays()
    g = gpu_trace(plt, gl, pid, ab)
    assert g["valid"].all()
    M = oracle.abcd_input_to_plane(ol, R.LAMBDA_D, -5.0, ol.opts["sensor_z_mm"])
    h = ab["oy"].astype(np.float64)
    u = ab["dy"].astype(np.float64) / ab["dz"].astype(np.float64)
    pred = M[0, 0] * h + M[0, 1] * u
    assert np.all(np.abs(g["py"] - pred) <= 4.2e-5 * (np.abs(h) / 0.4) ** 3 + 1e-4)


@pytest.mark.parametrize("n", [1, 31, 32, 33, 1000, 4097])
def test_ragged_sizes(gpu_lib, n):
    plt = gpu_lib
    cfg = C.CONFIGS["C2"]
    gl, ol = _lenses(plt, "dgauss50", cfg["opts"])
    rays = R.gen_rays(cfg["law"], 17, 0, n)
    g = gpu_trace(plt, gl, 1 << 10, rays)
    o = oracle.trace(ol, 1 << 10, 0, rays)
    compare_trace(g, o)


def test_c2_dgauss_parity_2e20(gpu_lib):
    plt = gpu_lib
    cfg = C.CONFIGS["C2"]
    gl, ol = _lenses(plt, "dgauss50", cfg["opts"])
    rays = R.gen_rays(cfg["law"], cfg["seed"], 0, 1 << 20)
    g = gpu_trace(plt, gl, 1 << 10, rays)
    o = oracle.trace(ol, 1 << 10, 0, rays, threads=oracle.host_threads())
    st = compare_trace(g, o)
    assert 0.3 < st["valid_frac"] < 0.45
    assert g["flags"].mean() < 0.02   # guard-band re-trace stays a small fraction


def test_c2_full_size_sampled(gpu_lib):
    """Full C2 size (2^24 rays) in the bench's launch configuration; oracle on a sample."""
    import torch
    plt = gpu_lib
    cfg = C.CONFIGS["C2"]
    gl, ol = _lenses(plt, "dgauss50", cfg["opts"])
    n = cfg["n"]
    rays = R.gen_rays(cfg["law"], cfg["seed"], 0, n)
    g = gpu_trace(plt, gl, 1 << 10, rays, flags=False)
    idx = R.sample_indices(n, 1 << 16, 123)
    sub = {k: rays[k][idx] for k in plt.RAY_KEYS}
    sub["plane_z"] = rays["plane_z"]
    o = oracle.trace(ol, 1 << 10, 0, sub, threads=oracle.host_threads())
    gs = {k: v[idx] for k, v in g.items() if k != "flags" and v is not None}
    compare_trace(gs, o)
    # invalid rays everywhere carry zeros; mask tail words beyond n untouched semantics
    assert np.count_nonzero(g["I"][~g["valid"]]) == 0


def test_c3_backward_parity(gpu_lib):
    plt = gpu_lib
    cfg = C.CONFIGS["C3"]
    gl, ol = _lenses(plt, "wide24", cfg["opts"])
    rays = R.gen_rays(cfg["law"], cfg["seed"], 0, 1 << 20)
    g = gpu_trace(plt, gl, 1 << 12, rays, direction=1)
    o = oracle.trace(ol, 1 << 12, 1, rays, threads=oracle.host_threads())
    st = compare_trace(g, o)
    assert 0.04 < st["valid_frac"] < 0.12
    assert np.all(g["dz"][g["valid"]] < 0)


@pytest.mark.parametrize("cfg_name", ["C4_22", "C4_59"])
def test_c4_ghosts_fp64_parity(gpu_lib, cfg_name):
    """Ghost paths: fp64 mode binds (A22); fp32 mode is reported, with its bounded error."""
    plt = gpu_lib
    cfg = C.CONFIGS[cfg_name]
    lens_name = cfg["lens"]
    gl, ol = _lenses(plt, lens_name, cfg["opts"])
    ids, ij = gl.enumerate_ghosts(2)
    oids, _ = oracle.enumerate_ghosts(ol, 2)
    assert ids == oids
    rays = C.flare_rays(cfg_name, 1, 0, 1 << 15)
    rng = np.random.default_rng(0)
    pick = [ids[0]] + list(rng.choice(ids[1:], 8, replace=False))
    nval = 0
    for pid in pick:
        o = oracle.trace(ol, int(pid), 0, rays, threads=oracle.host_threads())
        g64 = gpu_trace(plt, gl, int(pid), rays, precision=1)
        # fp64 arithmetic, float32 output storage: errors are output rounding only
        st = compare_trace(g64, o, tol_p=4e-6, tol_w=2e-7, tol_i=2e-7)
        nval += st["n_both"]
        g32 = gpu_trace(plt, gl, int(pid), rays, precision=0)
        s32 = compare_trace(g32, o, assert_ok=False)
        assert s32["mask_mismatch"] <= max(2, int(1e-3 * o["valid"].sum()))
    assert nval > 100


@pytest.mark.parametrize("cfg_name", ["C4_22", "C4_59"])
def test_four_bounce_paths_fp64_parity(gpu_lib, cfg_name):
    """Four-bounce paths (up to 60+ surface steps): the brightest ones
    by normal-incidence throughput, float64 trace vs the oracle, flare rays."""
    plt = gpu_lib
    cfg = C.CONFIGS[cfg_name]
    gl, ol = _lenses(plt, cfg["lens"], cfg["opts"])
    ids4, _ = gl.enumerate_ghosts(4, 1e-9)
    ids2, _ = gl.enumerate_ghosts(2)
    four = sorted(set(ids4) - set(ids2))
    thr = {p: oracle.lens._walk_normal_incidence(ol, p, 587.5618) for p in four}
    pick = sorted(four, key=lambda p: -thr[p])[:5] + [max(four)]     # brightest + the longest path
    rays = C.flare_rays(cfg_name, 1, 0, 1 << 15)
    nval = 0
    for pid in pick:
        o = oracle.trace(ol, int(pid), 0, rays, threads=oracle.host_threads())
        g64 = gpu_trace(plt, gl, int(pid), rays, precision=1)
        nval += compare_trace(g64, o, tol_p=4e-6, tol_w=2e-7, tol_i=2e-7)["n_both"]
    assert nval > 20


def test_invalid_path_id_and_empty(gpu_lib):
    plt = gpu_lib
    gl = plt.Lens(LENSES["dgauss50"])
    rays = R.gen_rays(C.CONFIGS["C2"]["law"], 1, 0, 64)
    d = plt.rays_to_device(rays)
    h = plt.alloc_hits(64)
    with pytest.raises(plt.PltError):
        plt.trace_rays(gl, (1 << 10) | 1, d, h)       # R at the first surface: exits the front
    with pytest.raises(plt.PltError):
        plt.trace_rays(gl, 1 << 9, d, h)              # too few interactions
    plt.trace_rays(gl, 1 << 10, d, h, n=0)            # n == 0 is a no-op


@pytest.mark.parametrize("housing", [11.0, 9.0])
def test_housing_cylinder_parity(gpu_lib, housing):
    """Housing absorption (A5) on the GPU: the C2 lens inside a barrel of
    radius 11 / 9 mm (smaller than the 12.6 / 11.5 / 10 mm clear apertures it crosses), fp32
    all-T (JIT), fp64 all-T and an fp64 ghost against the oracle's housing branch (pinned in
    tests/test_oracle_branches.py).  The barrel must actually decide rays: a share of
    the rays valid without it become invalid with it."""
    plt = gpu_lib
    cfg = C.CONFIGS["C2"]
    opts = dict(cfg["opts"], housing_radius_mm=housing)
    gl, ol = _lenses(plt, "dgauss50", opts)
    _, ol0 = _lenses(plt, "dgauss50", cfg["opts"])
    rays = R.gen_rays(cfg["law"], 77, 0, (1 << 18) + 5)
    o = oracle.trace(ol, 1 << 10, 0, rays, threads=oracle.host_threads())
    o0 = oracle.trace(ol0, 1 << 10, 0, rays, threads=oracle.host_threads())
    absorbed = o0["valid"] & ~o["valid"]
    assert absorbed.mean() > 0.01, absorbed.mean()
    assert not (o["valid"] & ~o0["valid"]).any()
    compare_trace(gpu_trace(plt, gl, 1 << 10, rays, precision=0), o)
    compare_trace(gpu_trace(plt, gl, 1 << 10, rays, precision=1), o, tol_p=4e-6, tol_w=2e-7, tol_i=2e-7)
    pid = oracle.ghost_id(10, 7, 3)
    og = oracle.trace(ol, pid, 0, rays, threads=oracle.host_threads())
    st = compare_trace(gpu_trace(plt, gl, pid, rays, precision=1), og, tol_p=4e-6, tol_w=2e-7, tol_i=2e-7)
    assert st["n_both"] > 100
    s32 = compare_trace(gpu_trace(plt, gl, pid, rays, precision=0), og, assert_ok=False)
    assert s32["mask_mismatch"] <= max(2, int(1e-3 * og["valid"].sum()))


def test_housing_and_rectangle_scalar_kernel_subprocess():
    """The scalar (non-packed, non-JIT) fp32 kernel through the same housing + CMOS-rectangle
    cases: PLT_TRACE_X1 / PLT_TRACE_JIT=0 are read once per process, so run a child."""
    import os
    import subprocess
    import sys
    code = r'''
import sys, numpy as np
sys.path.insert(0, "tests")
import oracle, paper_2605_04017_b200 as plt
from plt_inputs import configs as C, rays as R
from gpu_helpers import compare_trace, gpu_trace
cfg = C.CONFIGS["C4_22"]
for opts in (dict(cfg["opts"], housing_radius_mm=10.0), cfg["opts"]):
    gl = plt.Lens(C.lens_text("C4_22"), **opts); ol = oracle.load_lens(C.lens_text("C4_22"), opts)
    rays = C.flare_rays("C4_22", 1, 0, 1 << 16)
    o = oracle.trace(ol, 1 << 12, 0, rays)
    compare_trace(gpu_trace(plt, gl, 1 << 12, rays, precision=0), o)
print("ok")
'''
    env = dict(os.environ, PLT_TRACE_X1="1", PLT_TRACE_JIT="0")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]
