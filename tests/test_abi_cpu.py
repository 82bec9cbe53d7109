"""CPU-side checks of the C-ABI library: it builds for sm_100a, loads, exports every
symbol include/plt.h declares, its host-only logic (parsing, validation, ABCD,
ghost enumeration) agrees with the oracle, and compute calls fail loudly without
an sm_100a device (no CPU fallback)."""
import ctypes as C
import json
import math
import os
import re

import numpy as np
import pytest

import oracle
from plt_inputs import configs as CF
from plt_inputs.lenses import LENSES

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def plt():
    from paper_2605_04017_b200 import build
    build.build()
    import paper_2605_04017_b200 as p
    p.load()
    return p


def test_exports_every_header_symbol(plt):
    hdr = open(os.path.join(ROOT, "include", "plt.h")).read()
    declared = set(re.findall(r"PLT_API[^;(]*?\b(plt_\w+)\s*\(", hdr))
    assert len(declared) >= 12
    lib = C.CDLL(plt.LIB_PATH)
    for name in declared:
        assert hasattr(lib, name), name
    assert declared == set(plt.EXPORTED)
    assert plt.version().startswith("plt")


@pytest.mark.parametrize("name", ["singlet", "dgauss50", "wide22", "wide24", "dgauss59"])
def test_lens_info_matches_oracle_abcd(plt, name):
    L = plt.Lens(LENSES[name])
    O = oracle.load_lens(LENSES[name])
    for lam in (486.1327, 587.5618, 656.2725, 400.0, 700.0):
        info = L.info(lam)
        M = oracle.abcd_vertex_to_vertex(O, lam)
        assert np.allclose(info["abcd"], M.ravel(), rtol=1e-12, atol=1e-14)
        efl, bfl = oracle.efl_bfl(O, lam)
        assert abs(info["efl_mm"] - efl) < 1e-9 and abs(info["bfl_mm"] - bfl) < 1e-9
    assert abs(L.info()["sensor_z_mm"] - O.opts["sensor_z_mm"]) < 1e-9
    assert info["n_optical"] == O.n_optical


@pytest.mark.parametrize("name", ["dgauss50", "wide22", "singlet"])
def test_ghost_enumeration_matches_oracle(plt, name):
    L = plt.Lens(LENSES[name])
    O = oracle.load_lens(LENSES[name])
    for mb, thr in ((0, 0.0), (2, 0.0), (2, 1e-5), (2, 1e-3), (4, 0.0), (4, 1e-6)):
        ids, ij = L.enumerate_ghosts(mb, thr)
        oids, oij = oracle.enumerate_ghosts(O, mb, thr)
        assert ids == oids and ij == [tuple(x) for x in oij]


def test_two_call_capacity_pattern(plt):
    L = plt.Lens(LENSES["wide22"])
    lib = plt.load()
    cnt = C.c_int()
    st = lib.plt_enumerate_ghosts(L.handle, 2, 0.0, None, None, 0, C.byref(cnt))
    assert st == 4 and cnt.value == 67
    assert 65616 in L.enumerate_ghosts()[0]      # the paper's 22 mm path id


def test_json_prescription_equals_table(plt):
    import json
    O = oracle.load_lens(LENSES["dgauss50"])
    rows = []
    for line in LENSES["dgauss50"].splitlines():
        b = line.split("#")[0].split()
        if not b or b[0] == "name":
            continue
        rows.append({"radius_mm": float(b[0]), "thickness_mm": float(b[1]), "glass": b[2],
                     "semi_aperture_mm": float(b[3]) / 2})
    doc = json.dumps({"name": "dg", "surfaces": rows})
    Lj, Lt = plt.Lens(doc), plt.Lens(LENSES["dgauss50"])
    assert Lj.info(500.0) == Lt.info(500.0)
    assert oracle.efl_bfl(oracle.load_lens(doc), 500.0) == oracle.efl_bfl(O, 500.0)


@pytest.mark.parametrize("text,code,frag", [
    ("name x\n50 5 abbe:1.5 25\n", 2, "needs 2"),                       # parse error with field context
    ("name x\n50 5 foo:1 25\n", 2, "unknown glass"),
    ("name x\n50 5 n:1.5 oops\n", 2, "line 2"),
    ("name x\n0 5 stop 10\n0 5 stop 10\n50 0 n:1.5 20\n", 3, "more than one aperture stop"),
    ("name x\n5 2 n:1.5 20\n-50 0 air 20\n", 3, "semi-aperture"),         # |R| < a
    ("name x\n50 0 n:1.5 20\n-50 0 air 20\n", 3, "non-increasing"),
    ("name x\n50 5 n:0.9 20\n-50 0 air 20\n", 3, "index < 1"),
    ("name x\n0 5 stop 10\n", 3, "no optical surface"),
])
def test_parse_and_validation_errors(plt, text, code, frag):
    with pytest.raises(plt.PltError) as e:
        plt.Lens(text, sensor_z_mm=50.0)
    assert e.value.status == code and frag in str(e.value)


def test_map_blob_validation(plt):
    blob = CF.map_blob("C2", 1 << 10)
    plt.Map(blob)
    with pytest.raises(plt.PltError) as e:
        plt.Map(blob[:100])
    assert e.value.status == 2
    with pytest.raises(plt.PltError) as e:
        plt.Map(b"XXXXXXXX" + blob[8:])
    assert e.value.status == 2
    with pytest.raises(plt.PltError) as e:   # path 2^10 does not fit the 12-surface lens
        plt.Map(blob, lens=plt.Lens(LENSES["wide22"]))
    assert e.value.status == 3


def test_compute_calls_fail_loudly_without_gpu(plt):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    lib = plt.load()
    L = plt.Lens(LENSES["dgauss50"])
    fake = [C.c_void_p(4096 * (k + 1)) for k in range(8)]
    rays = plt.Rays(*fake[:6], -5.0)
    hits = plt.Hits(*fake[:7], None)
    st = lib.plt_trace_rays(L.handle, 1 << 10, 0, 0, C.byref(rays), C.byref(hits), 10, None)
    assert st == 6   # PLT_E_CUDA: no sm_100a device, no fallback
    assert lib.plt_trace_rays(L.handle, 1 << 10, 0, 0, C.byref(rays), C.byref(hits), 0, None) == 0
    assert lib.plt_trace_rays(L.handle, 1 << 10, 0, 0, C.byref(rays), C.byref(hits), -1, None) == 1
    m = plt.Map(CF.map_blob("C2", 1 << 10))
    assert lib.plt_eval_map(m.handle, C.byref(rays), C.byref(hits), None, 10, None) == 6


def test_fused_splat_entry_points_validate_then_fail_loudly(plt):
    """plt_trace_rays_splat / plt_eval_map_splat: a null target or a bad film description is
    PLT_E_INVALID_ARG (checked before the device); a valid call needs the GPU (PLT_E_CUDA)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    lib = plt.load()
    L = plt.Lens(LENSES["dgauss50"])
    m = plt.Map(CF.map_blob("C2", 1 << 10))
    fake = [C.c_void_p(4096 * (k + 1)) for k in range(8)]
    rays = plt.Rays(*fake[:6], -5.0)
    hits = plt.Hits(*fake[:7], None)
    good = plt.FilmDesc(768, 512, 3, 24.0, 16.0, 0.0, 0.0)
    bad = plt.FilmDesc(0, 512, 3, 24.0, 16.0, 0.0, 0.0)
    for fd, want in ((good, 6), (bad, 1)):
        t = plt.SplatTarget(C.addressof(fd), 8192, None, 1.0, None)
        assert lib.plt_trace_rays_splat(L.handle, 1 << 10, 0, 0, C.byref(rays), C.byref(hits), C.byref(t), 10,
                                        None) == want
        assert lib.plt_eval_map_splat(m.handle, C.byref(rays), C.byref(hits), None, C.byref(t), 10, None) == want
    assert lib.plt_trace_rays_splat(L.handle, 1 << 10, 0, 0, C.byref(rays), C.byref(hits), None, 10, None) == 1
    assert lib.plt_eval_map_splat(m.handle, C.byref(rays), C.byref(hits), None, None, 10, None) == 1
    t = plt.SplatTarget(C.addressof(good), None, None, 1.0, None)     # null film
    assert lib.plt_eval_map_splat(m.handle, C.byref(rays), C.byref(hits), None, C.byref(t), 10, None) == 1


@pytest.mark.parametrize("name,path,direction", [("C1", 0, 0), ("C2", 0, 0), ("C3", 0, 1), ("C4_22", 65616, 0)])
def test_trace_jit_compiles_without_gpu(plt, name, path, direction):
    """plt_trace_jit_cubin: the path-specialised trace kernel compiles with NVRTC for sm_100a
    on the build host (catches a broken JIT source before any GPU run)."""
    cfg = CF.CONFIGS[name]
    L = plt.Lens(CF.lens_text(name), **cfg["opts"])
    cubin = L.trace_jit_cubin(path or L.all_t_id(), direction)
    assert cubin[:4] == b"\x7fELF" and b"plt_trace_jit" in cubin


def test_camera_entry_points_validate_then_fail_loudly(plt):
    """plt_shade_plane / plt_propagate_rays: bad arguments are PLT_E_INVALID_ARG before the
    device is touched; valid calls need the GPU (PLT_E_CUDA)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    lib = plt.load()
    fake = [C.c_void_p(4096 * (k + 1)) for k in range(8)]
    rays = plt.Rays(*fake[:6], 52.0)
    hits = plt.Hits(*fake[:7], None)
    good = plt.ScenePlane(-1000.0, 50.0, 0.1)
    bad = plt.ScenePlane(-1000.0, 0.0, 0.1)
    film = C.c_void_p(1 << 20)
    assert lib.plt_shade_plane(C.byref(good), -5.0, C.byref(hits), 4, 100, 1.0, film, 10, None) == 6
    assert lib.plt_shade_plane(C.byref(bad), -5.0, C.byref(hits), 4, 100, 1.0, film, 10, None) == 1
    assert lib.plt_shade_plane(C.byref(good), -5.0, C.byref(hits), 0, 100, 1.0, film, 10, None) == 1
    assert lib.plt_shade_plane(C.byref(good), -5.0, C.byref(hits), 4, 100, 1.0, None, 10, None) == 1
    assert lib.plt_shade_plane(C.byref(good), -5.0, C.byref(hits), 4, 100, 1.0, film, 0, None) == 0
    assert lib.plt_propagate_rays(C.byref(rays), C.byref(rays), 50.0, 0, 10, None) == 6
    assert lib.plt_propagate_rays(C.byref(rays), C.byref(rays), float("nan"), 0, 10, None) == 1
    assert lib.plt_propagate_rays(C.byref(rays), C.byref(rays), 50.0, 0, -1, None) == 1
    assert lib.plt_propagate_rays(C.byref(rays), C.byref(rays), 50.0, 2, 10, None) == 1   # bad direction


ASPH_TABLE = """name asph_singlet
0       5.0  stop                     16.0
50.0    5.0  sellmeier:1.03961212,0.231792344,1.01046945,0.00600069867,0.0200179144,103.560653  25.0  asph:-0.8,2e-6,-3e-9
-50.0   0.0  air                      25.0
"""


def test_aspheric_lens_parse_validate_and_match_oracle(plt):
    """Even aspheres (NEXT-4): the table 'asph:' token and the JSON conic/aspheric fields
    give the same lens; paraxial data (ABCD) ignore the aspheric terms; a conic undefined
    inside the aperture is rejected; ghost enumeration unchanged."""
    L = plt.Lens(ASPH_TABLE)
    base = plt.Lens(ASPH_TABLE.replace("  asph:-0.8,2e-6,-3e-9", ""))
    assert L.info()["abcd"] == base.info()["abcd"]
    O = oracle.load_lens(ASPH_TABLE)
    assert O.surfaces[1].asph and O.surfaces[1].k == -0.8 and O.surfaces[1].A == (2e-6, -3e-9, 0.0, 0.0)
    doc = {"name": "j", "surfaces": [
        {"radius_mm": 0.0, "thickness_mm": 5.0, "glass": "stop", "semi_aperture_mm": 8.0},
        {"radius_mm": 50.0, "thickness_mm": 5.0, "semi_aperture_mm": 12.5, "conic": -0.8, "aspheric": [2e-6, -3e-9],
         "glass": "sellmeier:1.03961212,0.231792344,1.01046945,0.00600069867,0.0200179144,103.560653"},
        {"radius_mm": -50.0, "thickness_mm": 0.0, "glass": "air", "semi_aperture_mm": 12.5}]}
    J = plt.Lens(json.dumps(doc))
    assert J.info() == L.info()
    with pytest.raises(plt.PltError) as e:                 # hyperbolic domain: 1 - (1+k) c^2 a^2 < 0
        plt.Lens(ASPH_TABLE.replace("asph:-0.8", "asph:20"))
    assert e.value.status == 3
    assert L.enumerate_ghosts(2) == base.enumerate_ghosts(2)


@pytest.mark.parametrize("name", ["singlet", "dgauss50", "wide24", "wide22"])
def test_pupils_match_oracle(plt, name):
    L, O = plt.Lens(LENSES[name]), oracle.load_lens(LENSES[name])
    for lam in (486.1327, 587.5618, 656.2725):
        p = L.pupils(lam)
        o = oracle.pupils(O, lam)
        assert np.allclose([p["entrance_z_mm"], p["entrance_r_mm"], p["exit_z_mm"], p["exit_r_mm"]], o,
                           rtol=1e-12, atol=1e-12)


def _coated(text, tok="coat:1.38,550"):
    """Add a single-layer coating to every surface with air on one side."""
    lens = oracle.load_lens(text)
    out, k = [], 0
    for line in text.splitlines():
        body = line.split("#", 1)[0].split()
        if len(body) >= 4 and body[0] != "name":
            s = lens.surfaces[k]
            k += 1
            air = lambda g: g[0] == 0 and g[1][0] == 1.0
            if not s.is_stop and (air(s.glass_before) or air(s.glass_after)):
                line = line.split("#", 1)[0].rstrip() + " " + tok
        out.append(line)
    return "\n".join(out) + "\n"


def test_coated_lens_parse_validate_and_prune_match_oracle(plt):
    """AR coatings (NEXT-4): parsed in table and JSON forms, rejected on glass-glass
    surfaces, paraxial data unchanged, and the normal-incidence ghost prune (which now
    uses the film reflectance) matches the oracle's."""
    text = _coated(LENSES["dgauss50"])
    L, O = plt.Lens(text), oracle.load_lens(text)
    assert L.info()["abcd"] == plt.Lens(LENSES["dgauss50"]).info()["abcd"]
    assert sum(1 for s in O.surfaces if s.coat_n > 0) >= 6
    for thr in (0.0, 1e-6, 1e-5):
        ids, ij = L.enumerate_ghosts(2, thr)
        oids, oij = oracle.enumerate_ghosts(O, 2, thr)
        assert ids == oids
    assert len(L.enumerate_ghosts(2, 1e-5)[0]) < len(plt.Lens(LENSES["dgauss50"]).enumerate_ghosts(2, 1e-5)[0])
    with pytest.raises(plt.PltError) as e:                 # a coating on a glass-glass interface
        plt.Lens("name c\n10 2 n:1.5 10 coat:1.38,550\n-10 2 n:1.7 10 coat:1.38,550\n-30 0 air 10\n")
    assert e.value.status == 3
    doc = {"surfaces": [{"radius_mm": 0, "thickness_mm": 2, "glass": "n:1.5", "semi_aperture_mm": 5,
                         "coating": {"n": 1.38, "lambda0_nm": 550}},
                        {"radius_mm": 0, "thickness_mm": 0, "glass": "air", "semi_aperture_mm": 5}]}
    J = plt.Lens(json.dumps(doc), sensor_z_mm=10.0)
    T = plt.Lens("name t\n0 2 n:1.5 10 coat:1.38,550\n0 0 air 10\n", sensor_z_mm=10.0)
    assert J.enumerate_ghosts(2, 1e-9) == T.enumerate_ghosts(2, 1e-9)


def test_rays_without_dz_pass_validation_then_fail_loudly(plt):
    """plt_rays.dz may be NULL (directions in S^2_+ given by (dx, dy)): the call is
    not an argument error; it needs the GPU (PLT_E_CUDA).  Other null ray arrays still are
    PLT_E_INVALID_ARG.  plt_propagate_rays: out->dz may be NULL only when in->dz is."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    lib = plt.load()
    L = plt.Lens(LENSES["dgauss50"])
    m = plt.Map(CF.map_blob("C2", 1 << 10))
    fake = [C.c_void_p(4096 * (k + 1)) for k in range(8)]
    no_dz = plt.Rays(fake[0], fake[1], fake[2], fake[3], None, fake[5], -5.0)
    no_dx = plt.Rays(fake[0], fake[1], None, fake[3], fake[4], fake[5], -5.0)
    hits = plt.Hits(*fake[:7], None)
    assert lib.plt_trace_rays(L.handle, 1 << 10, 0, 0, C.byref(no_dz), C.byref(hits), 10, None) == 6
    assert lib.plt_trace_rays(L.handle, 1 << 10, 0, 0, C.byref(no_dx), C.byref(hits), 10, None) == 1
    assert lib.plt_eval_map(m.handle, C.byref(no_dz), C.byref(hits), None, 10, None) == 6
    full = plt.Rays(*fake[:6], -5.0)
    assert lib.plt_propagate_rays(C.byref(no_dz), C.byref(no_dz), 50.0, 1, 10, None) == 6
    assert lib.plt_propagate_rays(C.byref(full), C.byref(no_dz), 50.0, 1, 10, None) == 1


@pytest.mark.parametrize("kind", ["coated", "aspheric", "sellmeier"])
def test_trace_jit_compiles_for_every_feature(plt, kind):
    """The run-time specialised trace compiles for programs that use each optional feature:
    coated surfaces (no eta polynomials: the film needs both indices), aspheres (Newton
    intersection) and Sellmeier glasses (eta(lambda) fitted from the Sellmeier formula)."""
    if kind == "coated":
        L = plt.Lens(_coated(LENSES["dgauss50"]))
    elif kind == "aspheric":
        L = plt.Lens(ASPH_TABLE, sensor_z_mm=120.0)
    else:
        L = plt.Lens(LENSES["singlet"])
    cubin = L.trace_jit_cubin(L.all_t_id())
    assert cubin[:4] == b"\x7fELF" and b"plt_trace_jit" in cubin


def test_film_size_limit(plt):
    """Splat keys are 32-bit: films with channels*height*width >= 2^31 are rejected before
    any device work (PLT_E_INVALID_ARG), smaller ones pass validation (then need the GPU)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    lib = plt.load()
    fake = [C.c_void_p(4096 * (k + 1)) for k in range(8)]
    hits = plt.Hits(*fake[:7], None)
    big = plt.FilmDesc(65536, 32768, 1, 24.0, 16.0, 0.0, 0.0)      # 2^31 entries
    ok = plt.FilmDesc(65535, 32768, 1, 24.0, 16.0, 0.0, 0.0)
    film = C.c_void_p(1 << 20)
    assert lib.plt_splat_sensor(C.byref(big), film, C.byref(hits), None, 1.0, 10, None, None) == 1
    assert lib.plt_splat_sensor(C.byref(ok), film, C.byref(hits), None, 1.0, 10, None, None) == 6


@pytest.mark.parametrize("seed", range(8))
def test_random_lenses_load_and_match_oracle_paraxials(plt, seed):
    """The fuzz lenses of tests/test_gpu_fuzz_lenses.py parse in both implementations with
    the same paraxial matrix, ghost list, and a JIT-compilable all-T program."""
    from plt_inputs.lenses import random_lens_text
    text, semi, z_last = random_lens_text(seed)
    L, O = plt.Lens(text, sensor_z_mm=z_last + 40.0), oracle.load_lens(text, {"sensor_z_mm": z_last + 40.0})
    for lam in (400.0, 587.5618, 700.0):
        M = oracle.abcd_vertex_to_vertex(O, lam)
        assert np.allclose(L.info(lam)["abcd"], M.ravel(), rtol=1e-12, atol=1e-14)
    ids, _ = L.enumerate_ghosts(2)
    oids, _ = oracle.enumerate_ghosts(O, 2)
    assert list(ids) == list(oids)
    assert L.trace_jit_cubin(L.all_t_id())[:4] == b"\x7fELF"


def test_pupil_weight_and_new_entry_points_validate(plt):
    """plt_pupil_weight is the closed form pi r^2 / dz^2 (host); plt_gen_rays / plt_query_host /
    plt_trace_kernel validate their arguments before touching the device."""
    import math
    import torch
    assert abs(plt.pupil_weight(52.0, 36.0, 9.8) - math.pi * 9.8 ** 2 / 16.0 ** 2) < 1e-15
    assert abs(plt.pupil_weight(20.0, 36.0, 2.0) - math.pi * 4.0 / 256.0) < 1e-15
    with pytest.raises(plt.PltError):
        plt.pupil_weight(36.0, 36.0, 1.0)
    with pytest.raises(plt.PltError):
        plt.pupil_weight(50.0, 36.0, 0.0)
    lib = plt.load()
    fake = [C.c_void_p(4096 * (k + 1)) for k in range(8)]
    rays = plt.Rays(*fake[:6], -5.0)
    law = plt.RayLaw(0, 0, 0, 0, -5.0, 10.0, 0.0, 0.9, 0.0, 1.0, 0, 0, 0, 0, 400.0, 700.0)
    bad = plt.RayLaw(7, 0, 0, 0, -5.0, 10.0, 0.0, 0.9, 0.0, 1.0, 0, 0, 0, 0, 400.0, 700.0)
    grid = plt.RayLaw(3, 0, 16, 4, -5.0, 0, 0, 0, 0, 0, 24.0, 16.0, 36.0, 9.0, 400.0, 700.0)
    if not torch.cuda.is_available():
        assert lib.plt_gen_rays(C.byref(law), 1, 0, C.byref(rays), 10, None) == 6
    assert lib.plt_gen_rays(C.byref(bad), 1, 0, C.byref(rays), 10, None) == 1
    assert lib.plt_gen_rays(C.byref(grid), 1, 0, C.byref(rays), 10, None) == 1
    assert lib.plt_gen_rays(C.byref(law), 1, -1, C.byref(rays), 10, None) == 1
    assert lib.plt_gen_rays(C.byref(law), 1, 0, C.byref(rays), 0, None) == 0
    L = plt.Lens(LENSES["dgauss50"])
    assert lib.plt_query_host(L.handle, 1 << 10, 0, 0, None, C.byref(rays), None, None, None, None, 64, 33,
                              None) == 1                                  # chunk not a multiple of 32
    assert lib.plt_query_host(None, 0, 0, 0, None, C.byref(rays), None, None, None, None, 64, 32, None) == 1
    k = C.c_int()
    assert lib.plt_trace_kernel(L.handle, 1 << 10, 0, 1, C.byref(k)) == 0 and k.value == 3   # fp64
    assert lib.plt_trace_kernel(L.handle, (1 << 10) | 1, 0, 0, C.byref(k)) == 1            # bad path id


def test_jit_uses_the_toolkit_nvrtc_even_with_torch_loaded(plt):
    """The run-time specialised trace is compiled by the CUDA toolkit's NVRTC (the release
    that builds the ahead-of-time kernels), not by whichever libnvrtc.so.12 the process has
    already loaded (torch bundles an older one, whose code for the same source measured 9 %
    more instructions).  The cubin records its compiler release."""
    import re
    import subprocess
    import torch  # noqa: F401  (loads torch's libraries first, as bench.py and the tests do)
    nvcc = subprocess.run(["/usr/local/cuda/bin/nvcc", "--version"], capture_output=True, text=True).stdout
    release = re.search(r"release (\d+\.\d+)", nvcc).group(1)
    L = plt.Lens(LENSES["dgauss50"])
    cubin = L.trace_jit_cubin(L.all_t_id())
    m = re.search(rb"Cuda compilation tools, release (\d+\.\d+)", cubin)
    assert m and m.group(1).decode() == release, (m.group(0) if m else None, release)


def test_trace_paths_validates_then_fails_loudly(plt):
    """plt_trace_paths: n_paths < 0, null ids / outs, a null hit pointer or an id inconsistent
    with the lens are PLT_E_INVALID_ARG before any device work; n == 0 / n_paths == 0 are
    no-ops; a valid call needs the GPU (PLT_E_CUDA)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    lib = plt.load()
    L = plt.Lens(LENSES["wide22"])
    ids = [int(g) for g in L.enumerate_ghosts(2)[0]][:3]
    arr = (C.c_uint64 * 3)(*ids)
    fake = [C.c_void_p(4096 * (k + 1)) for k in range(8)]
    rays = plt.Rays(*fake[:6], -5.0)
    outs = (plt.Hits * 3)(*[plt.Hits(*fake[:7], None) for _ in range(3)])
    call = lambda a, k, o, n, prec=1: lib.plt_trace_paths(L.handle, a, k, 0, prec, C.byref(rays), o, None, n, None)
    assert call(arr, 3, outs, 10) == 6
    assert call(arr, 3, outs, 10, prec=0) == 6
    assert call(arr, 3, outs, 0) == 0
    assert call(arr, 0, outs, 10) == 0
    assert call(arr, -1, outs, 10) == 1
    assert call(None, 3, outs, 10) == 1
    assert call(arr, 3, None, 10) == 1
    bad = (plt.Hits * 3)(*[plt.Hits(*fake[:7], None) for _ in range(2)], plt.Hits(None, *fake[1:7], None))
    assert call(arr, 3, bad, 10) == 1
    wrong = (C.c_uint64 * 3)(ids[0], 12345678901, ids[2])
    assert call(wrong, 3, outs, 10) == 1
