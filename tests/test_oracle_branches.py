"""Pins for the oracle branches that decide validity and record margins (SURVEY §8(c)
O4-O6, O8; readings A5, A11, A12, A23):

* the housing cylinder ("rays ... absorbed by the housing"; "housing ...
  absorbed"; A5: endpoint tests on every surface),
* the CMOS rectangle on the output plane ("CMOS sized rectangle"; A11/A12),
* the margin bookkeeping that defines the parity band (north_star "1e-6 mm
  aperture-edge band"; A23): geometric edge |rho - a|, TIR |kappa|, sphere
  discriminant, |w_z|.

Every expected value is a closed form of a plane-parallel slab or a single spherical
cap (Snell's law in angle form, vertex-local sphere geometry), never the oracle's own
expressions.  CPU only."""
import math

import numpy as np
import pytest

import oracle

SLAB = "name slab\n0 2.0 n:1.5 40\n0 0.0 air 40\n"       # two planes, a = 20 mm, glass 1.5
N_GLASS = 1.5
Z_IN = -5.0


def rays_of(ox, oy, dx, dy, dz, lam, plane_z):
    a = lambda v: np.atleast_1d(np.asarray(v, dtype=np.float64))
    n = max(a(v).size for v in (ox, oy, dx, dy, dz, lam))
    b = lambda v: np.broadcast_to(a(v), (n,)).copy()
    return {"ox": b(ox), "oy": b(oy), "dx": b(dx), "dy": b(dy), "dz": b(dz), "lambda_nm": b(lam),
            "plane_z": plane_z}


def slab_landing(x0, theta, z_out):
    """x of a meridional ray (angle theta in x-z) through the slab: entry plane z=0, exit z=2,
    Snell sin(theta_t) = sin(theta)/1.5; x at z=0, z=2 and the output plane."""
    tt = math.asin(math.sin(theta) / N_GLASS)
    x1 = x0 + (0.0 - Z_IN) * math.tan(theta)
    x2 = x1 + 2.0 * math.tan(tt)
    x3 = x2 + (z_out - 2.0) * math.tan(theta)
    return x1, x2, x3


# ---------------------------------------------------------------------------
# housing cylinder
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("delta", [1e-3, 1e-5, 3e-7])
def test_housing_exit_face(delta):
    """A ray leaving the slab's rear face at rho = H + delta is absorbed, at H - delta it
    passes with geometric margin exactly delta (the front face is 2 tan(theta_t) inside)."""
    H = 10.0
    lens = oracle.load_lens(SLAB, {"sensor_z_mm": 12.0, "housing_radius_mm": H})
    th = math.radians(20.0)
    tt = math.asin(math.sin(th) / N_GLASS)
    xs = []
    for target in (H - delta, H + delta):
        # choose x0 so that the rear-face hit lands at `target`
        x0 = target - 2.0 * math.tan(tt) - 5.0 * math.tan(th)
        xs.append(x0)
    r = rays_of(xs, 0.0, math.sin(th), 0.0, math.cos(th), 550.0, Z_IN)
    t = oracle.trace(lens, 1 << 2, 0, r)
    assert t["valid"][0] and not t["valid"][1]
    assert abs(t["margins"][0, 0] - delta) < 1e-12
    assert abs(t["margins"][1, 0] - delta) < 1e-12
    # without the housing both pass (the clear aperture is 20 mm)
    free = oracle.trace(oracle.load_lens(SLAB, {"sensor_z_mm": 12.0}), 1 << 2, 0, r)
    assert free["valid"].all()
    assert np.all(free["margins"][:, 0] > 9.0)


def test_housing_entry_face_and_inward_ray():
    """Entering at rho = H + delta is absorbed even when the ray then heads inwards (the
    endpoint test at the front face); a ray that starts outside H on the input plane but
    enters inside passes (the input plane is not a surface)."""
    H = 10.0
    lens = oracle.load_lens(SLAB, {"sensor_z_mm": 12.0, "housing_radius_mm": H})
    th = math.radians(-15.0)
    d = 1e-4
    x0_in = (H + d) - 5.0 * math.tan(th)       # front-face hit at H + d, moving inwards
    x0_ok = (H - d) - 5.0 * math.tan(th)       # front-face hit at H - d
    r = rays_of([x0_in, x0_ok], 0.0, math.sin(th), 0.0, math.cos(th), 550.0, Z_IN)
    t = oracle.trace(lens, 1 << 2, 0, r)
    assert not t["valid"][0] and t["valid"][1]
    assert x0_ok > H                            # started outside the cylinder
    assert abs(t["margins"][1, 0] - d) < 1e-12


def test_housing_applies_along_ghost_paths():
    """On the ghost (2,1) the ray crosses the slab three times; the housing test applies at
    every hit.  A normal-incidence ray at rho = H - delta passes (margin delta) and at
    H + delta is absorbed -- the throughput T R R T of the slab is unchanged."""
    H = 7.5
    delta = 2e-4
    lens = oracle.load_lens(SLAB, {"sensor_z_mm": 12.0, "housing_radius_mm": H})
    pid = oracle.ghost_id(2, 2, 1)
    r = rays_of([0.0, 0.0], [H - delta, H + delta], 0.0, 0.0, 1.0, 550.0, Z_IN)
    t = oracle.trace(lens, pid, 0, r)
    assert t["valid"][0] and not t["valid"][1]
    R0 = ((N_GLASS - 1.0) / (N_GLASS + 1.0)) ** 2
    assert abs(t["I"][0] - (1 - R0) * R0 * R0 * (1 - R0)) < 1e-15
    assert abs(t["margins"][0, 0] - delta) < 1e-12


# ---------------------------------------------------------------------------
# CMOS rectangle on the output plane
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("axis", ["x", "y"])
@pytest.mark.parametrize("delta", [1e-2, 1e-6])
def test_sensor_rectangle_edges(axis, delta):
    """A ray landing at W/2 - delta (resp. H/2 - delta) passes with margin delta, one at
    W/2 + delta is dropped at trace time; the landing point is the slab closed form."""
    W, Hh, z_out = 8.0, 6.0, 12.0
    lens = oracle.load_lens(SLAB, {"sensor_z_mm": z_out, "sensor_w_mm": W, "sensor_h_mm": Hh})
    half = W / 2 if axis == "x" else Hh / 2
    th = math.radians(12.0)
    _, _, x3_per0 = slab_landing(0.0, th, z_out)      # landing of x0 = 0
    starts = [(half - delta) - x3_per0, (half + delta) - x3_per0]
    if axis == "x":
        r = rays_of(starts, 0.0, math.sin(th), 0.0, math.cos(th), 550.0, Z_IN)
        key = "px"
    else:
        r = rays_of(0.0, starts, 0.0, math.sin(th), math.cos(th), 550.0, Z_IN)
        key = "py"
    t = oracle.trace(lens, 1 << 2, 0, r)
    assert t["valid"][0] and not t["valid"][1]
    assert abs(t[key][0] - (half - delta)) < 1e-12
    assert abs(t["margins"][0, 0] - delta) < 1e-11
    assert abs(t["margins"][1, 0] - delta) < 1e-11
    # mirrored side (negative coordinate) behaves identically (|p - c| test)
    rm = {k: (-v if k in ("ox", "oy", "dx", "dy") else v) for k, v in r.items()}
    tm = oracle.trace(lens, 1 << 2, 0, rm)
    assert tm["valid"][0] and not tm["valid"][1]
    # unbounded output plane: both pass
    free = oracle.trace(oracle.load_lens(SLAB, {"sensor_z_mm": z_out}), 1 << 2, 0, r)
    assert free["valid"].all()


def test_sensor_rectangle_corner_and_backward_unbounded():
    """Corner: inside on x but outside on y is dropped.  The backward frame has no
    rectangle on its exit plane (A11: the sensor is the input there)."""
    W, Hh, z_out = 8.0, 6.0, 12.0
    lens = oracle.load_lens(SLAB, {"sensor_z_mm": z_out, "sensor_w_mm": W, "sensor_h_mm": Hh})
    r = rays_of([3.9, 3.9, 4.1], [2.9, 3.1, 2.9], 0.0, 0.0, 1.0, 550.0, Z_IN)
    t = oracle.trace(lens, 1 << 2, 0, r)
    assert t["valid"].tolist() == [True, False, False]
    assert abs(t["margins"][0, 0] - 0.1) < 1e-12
    # backward: rays start on the sensor plane (z = 12) travelling -z, exit at z = -5
    rb = rays_of([30.0], [0.0], 0.0, 0.0, -1.0, 550.0, z_out)
    lens_b = oracle.load_lens(SLAB.replace("40\n", "80\n"), {"sensor_z_mm": z_out, "sensor_w_mm": W,
                                                              "sensor_h_mm": Hh, "backward_exit_z_mm": -5.0})
    tb = oracle.trace(lens_b, 1 << 2, 1, rb)
    assert tb["valid"][0] and abs(tb["px"][0] - 30.0) < 1e-12 and tb["dz"][0] == -1.0


# ---------------------------------------------------------------------------
# margin bookkeeping (A23): the four recorded margins are the closed-form distances
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("delta", [1e-3, 1e-6, 1e-8])
def test_aperture_margin_equals_delta(delta):
    """A ray parallel to the axis at rho = a - delta passes both faces of the slab with
    geometric margin delta; at a + delta it is blocked at the first face."""
    lens = oracle.load_lens(SLAB, {"sensor_z_mm": 12.0})
    a = 20.0
    ang = 0.7
    rho = np.array([a - delta, a + delta])
    r = rays_of(rho * math.cos(ang), rho * math.sin(ang), 0.0, 0.0, 1.0, 550.0, Z_IN)
    t = oracle.trace(lens, 1 << 2, 0, r)
    assert t["valid"][0] and not t["valid"][1]
    assert np.allclose(t["margins"][:, 0], delta, rtol=1e-6, atol=1e-14)


def test_tir_margin_and_direction_margin_closed_form():
    """Oblique ray through the slab: kappa at the front face is 1 - sin^2(th)/1.5^2, at the
    rear face 1 - 1.5^2 sin^2(th_t) = cos^2(th) (the smaller); the smallest |w_z| over the
    direction checks is cos(th) (air before and after)."""
    lens = oracle.load_lens(SLAB, {"sensor_z_mm": 12.0})
    for deg in (5.0, 40.0, 80.0):
        th = math.radians(deg)
        r = rays_of(-5.0 * math.tan(th), 0.0, math.sin(th), 0.0, math.cos(th), 550.0, Z_IN)
        t = oracle.trace(lens, 1 << 2, 0, r)
        assert t["valid"][0]
        assert abs(t["margins"][0, 1] - math.cos(th) ** 2) < 1e-14
        assert abs(t["margins"][0, 3] - math.cos(th)) < 1e-15
        assert math.isinf(t["margins"][0, 2])          # no sphere on the path


def test_tir_margin_at_the_critical_angle():
    """Glass (n=2) hemisphere front, planar back: an axis-parallel ray at height h meets the
    sphere (R = 10) at incidence asin(h/R), refracts to th_t, and reaches the back face at
    asin(h/R) - th_t to the axis (thickness 9 > the cap's sag); the recorded kappa at the rear face is 1 - 4 sin^2 of that angle;
    it changes sign exactly where the ray becomes absorbed."""
    lens = oracle.load_lens("name tir\n10 9.0 n:2.0 20\n0 0 air 40\n", {"sensor_z_mm": 20.0})
    hs = np.linspace(0.5, 9.5, 37)
    t = oracle.trace(lens, 1 << 2, 0, rays_of(0.0, hs, 0.0, 0.0, 1.0, 550.0, Z_IN))
    for i, h in enumerate(hs):
        ti = math.asin(h / 10.0)                        # incidence at the sphere
        tt = math.asin(math.sin(ti) / 2.0)              # refracted
        back = ti - tt                                  # angle to the axis inside the glass
        k_front = 1.0 - (0.5 * math.sin(ti)) ** 2
        k_back = 1.0 - (2.0 * math.sin(back)) ** 2
        assert bool(t["valid"][i]) == (k_back >= 0.0)
        if t["valid"][i]:
            assert abs(t["margins"][i, 1] - min(k_front, abs(k_back))) < 1e-12
        # disc of the vertex-local sphere for an axis-parallel ray: R^2 - h^2
        assert abs(t["margins"][i, 2] - (100.0 - h * h)) < 1e-11


def test_sphere_discriminant_margin_and_miss():
    """Single convex cap (R = 10, a = 15 so the aperture never decides): a ray parallel to
    the axis at height h has disc = R^2 - h^2 exactly; at h > R it misses the sphere."""
    lens = oracle.load_lens("name cap\n10 0 n:1.5 30\n", {"sensor_z_mm": 30.0})
    hs = np.array([0.0, 3.0, 9.99, 10.0 - 1e-6, 10.0 + 1e-6, 12.0])
    t = oracle.trace(lens, 1 << 1, 0, rays_of(hs, 0.0, 0.0, 0.0, 1.0, 550.0, Z_IN))
    for i, h in enumerate(hs):
        assert bool(t["valid"][i]) == (h < 10.0)
        assert abs(t["margins"][i, 2] - abs(100.0 - h * h)) < 1e-11 * 100.0


def test_near_edge_band_selects_the_constructed_rays():
    """The parity band (tests/gpu_helpers.near_edge) selects exactly the rays built within
    1e-6 mm of an edge: rays at a +- 1e-7 are banded, at a +- 1e-5 they are not."""
    import sys, os
    sys.path.insert(0, os.path.dirname(__file__))
    from gpu_helpers import near_edge
    lens = oracle.load_lens(SLAB, {"sensor_z_mm": 12.0})
    rho = np.array([20.0 - 1e-7, 20.0 + 1e-7, 20.0 - 1e-5, 20.0 + 1e-5, 5.0])
    t = oracle.trace(lens, 1 << 2, 0, rays_of(rho, 0.0, 0.0, 0.0, 1.0, 550.0, Z_IN))
    assert near_edge(t["margins"]).tolist() == [True, True, False, False, False]


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4_22", "C4_59"])
def test_band_excludes_few_rays_on_the_config_laws(name):
    """The 1e-6 mm band may only exclude a handful of rays from mask exactness on the
    configs' ray laws (gpu_helpers.max_excluded bounds it in every GPU comparison)."""
    import sys, os
    sys.path.insert(0, os.path.dirname(__file__))
    from gpu_helpers import max_excluded, near_edge
    from plt_inputs import configs as C
    from plt_inputs import rays as R
    cfg = C.CONFIGS[name]
    ol = oracle.load_lens(C.lens_text(name), cfg["opts"])
    n = 1 << 18
    if name == "C1":
        rays, pids = C.c1_rays(), [1 << 2]
    elif "channels" in cfg:
        rays = C.flare_rays(name, 0, 0, n)
        ids, _ = oracle.enumerate_ghosts(ol, 2)
        pids = [1 << ol.n_optical] + list(ids[::9])
    else:
        rays, pids = R.gen_rays(cfg["law"], cfg.get("seed", 1), 0, n), [1 << ol.n_optical]
    for pid in pids:
        t = oracle.trace(ol, pid, cfg["direction"], rays, threads=oracle.host_threads())
        k = int(near_edge(t["margins"]).sum())
        assert k <= max_excluded(rays["ox"].size), (name, pid, k)


def test_steps_bookkeeping():
    """`steps` counts the surface steps a ray began (stop crossings included) plus the output
    plane: the basis of the algorithmic work count of the trace roofline."""
    lens = oracle.load_lens(SLAB, {"sensor_z_mm": 12.0})
    t = oracle.trace(lens, 1 << 2, 0, rays_of([0.0, 25.0], 0.0, 0.0, 0.0, 1.0, 550.0, Z_IN))
    assert t["steps"].tolist() == [3, 1]                # through both faces + output; blocked at face 1
    g = oracle.trace(lens, oracle.ghost_id(2, 2, 1), 0, rays_of(0.0, 0.0, 0.0, 0.0, 1.0, 550.0, Z_IN))
    assert g["steps"].tolist() == [5]                   # T, R, R, T + output
    from plt_inputs.lenses import LENSES
    s = oracle.load_lens(LENSES["singlet"])             # stop at z = 0 (a = 8), two spherical faces
    t = oracle.trace(s, 1 << 2, 0, rays_of([0.0, 9.0], 0.0, 0.0, 0.0, 1.0, 550.0, Z_IN))
    assert t["steps"].tolist() == [4, 1]                # stop + 2 faces + output; blocked at the stop
