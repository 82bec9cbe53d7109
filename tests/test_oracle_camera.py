"""Pins of the oracle's backward camera integrand (O14, Eq. 9; SURVEY §8(f)
NEXT-3) and free-space propagation: closed forms on hand-made rays."""
import numpy as np

import oracle

SCENE = {"z_mm": -100.0, "period_mm": 10.0, "contrast": 0.25}


def test_axial_rays_hit_the_square_below_them():
    # straight down the axis from (x, y): hits (x, y); parity of floor(x/10) + floor(y/10)
    xs = np.array([1.0, 11.0, -1.0, -11.0, 25.0, 5.0], np.float32)
    ys = np.array([1.0, 1.0, 1.0, -1.0, 15.0, -25.0], np.float32)
    n = xs.size
    f = oracle.shade_plane(SCENE, -5.0, np.ones(n), xs, ys, np.zeros(n), np.zeros(n), -np.ones(n),
                           np.full(n, 0.5), spp=1, pixels=n, scale=1.0)
    parity = (np.floor(xs / 10.0) + np.floor(ys / 10.0)).astype(np.int64) & 1
    want = np.round(0.5 * np.where(parity == 1, 0.25, 1.0) * 2.0 ** 32).astype(np.int64)
    assert np.array_equal(f, want)


def test_oblique_ray_lands_where_the_line_meets_the_plane():
    # from (0, 0, -5) along (3, 4, -12)/13: reaches z = -100 after t = 95 * 13 / 12 -> (23.75, 31.67)
    d = np.array([3.0, 4.0, -12.0]) / 13.0
    f = oracle.shade_plane(SCENE, -5.0, [1], [0.0], [0.0], [d[0]], [d[1]], [d[2]], [1.0], spp=1, pixels=1)
    x, y = 95.0 / 12.0 * 3.0, 95.0 / 12.0 * 4.0                 # (23.75, 31.67): squares 2 + 3 -> odd
    assert (int(np.floor(x / 10)) + int(np.floor(y / 10))) % 2 == 1
    assert f[0] == round(0.25 * 2.0 ** 32)


def test_pixels_accumulate_spp_rays_and_skip_invalid_backward_and_out_of_range():
    n, spp = 12, 4
    dz = -np.ones(n)
    dz[5] = +1.0                                  # leaves away from the scene: t < 0, no contribution
    valid = np.ones(n, bool)
    valid[2] = False
    f = oracle.shade_plane(SCENE, -5.0, valid, np.full(n, 1.0), np.full(n, 1.0), np.zeros(n), np.zeros(n), dz,
                           np.full(n, 0.125), spp=spp, pixels=2, scale=2.0)   # rays 8..11 -> pixel 2 >= pixels
    one = round(0.125 * 2.0 * 2.0 ** 32)
    assert list(f) == [3 * one, 3 * one]


def test_propagation_stays_on_the_ray_and_reaches_the_plane():
    rng = np.random.default_rng(3)
    n = 1000
    w = rng.normal(size=(n, 3))
    w[:, 2] = -np.abs(w[:, 2]) - 0.2
    w /= np.linalg.norm(w, axis=1, keepdims=True)
    rays = {"ox": rng.uniform(-10, 10, n), "oy": rng.uniform(-10, 10, n), "dx": w[:, 0], "dy": w[:, 1],
            "dz": w[:, 2], "lambda_nm": np.full(n, 550.0), "plane_z": 52.0}
    p = oracle.propagate(rays, 50.0)
    t = (50.0 - 52.0) / w[:, 2]
    assert np.allclose(p["ox"], rays["ox"] + t * w[:, 0], rtol=0, atol=1e-12)
    # (o' - o) is parallel to w and its z step is exactly the plane distance
    step = np.stack([p["ox"] - rays["ox"], p["oy"] - rays["oy"], np.full(n, -2.0)], 1)
    assert np.allclose(np.cross(step, w), 0.0, atol=1e-12)


def test_pupil_sampling_weight_reproduces_the_projected_solid_angle():
    """Eq. 9 with directions drawn through uniform points on a disc (radius r, axial
    distance D) parallel to the sensor: weighting each ray by (A / D^2) cos^4(theta)
    estimates the cosine-weighted solid angle of the disc seen from the on-axis sensor
    point, pi sin^2(alpha) with tan(alpha) = r / D (closed form).  A cos^3 or cos^5 weight
    misses it by several percent."""
    r, D, m = 6.0, 12.0, 1 << 18
    k = np.arange(m)
    rad = r * np.sqrt((k + 0.5) / m)                        # stratified radius x golden-angle
    phi = k * np.pi * (3.0 - np.sqrt(5.0))
    px, py = rad * np.cos(phi), rad * np.sin(phi)
    w = np.stack([px, py, np.full(m, D)], 1)
    w /= np.linalg.norm(w, axis=1, keepdims=True)
    ones, zeros = np.ones(m, np.float32), np.zeros(m, np.float32)
    scene = {"z_mm": -100.0, "period_mm": 1e6, "contrast": 1.0}     # uniform radiance L = 1
    A = np.pi * r * r
    f = oracle.shade_plane(scene, 0.0, np.ones(m, bool), zeros, zeros, zeros, zeros, -ones, ones, spp=m, pixels=1,
                           scale=A / D ** 2 / m, in_dz=w[:, 2].astype(np.float32))
    est = f[0] / 2.0 ** 32
    sin2 = r * r / (r * r + D * D)
    assert abs(est - np.pi * sin2) < 2e-3 * np.pi * sin2
    cos3 = np.mean(w[:, 2] ** 3) * A / D ** 2
    assert abs(cos3 - np.pi * sin2) > 0.03 * np.pi * sin2


def test_scene_cards_nearest_card_inside_its_rectangle():
    """O14b: straight-back rays (w = (0, 0, -1)) from z_hits = 0 through a near card
    (z = -100, |x| <= 10, y in [-5, 5], uniform L = 1) in front of a far card (z = -500,
    |x|, |y| <= 40, contrast 0.25 on every square: period huge, so x >= 0 squares are
    even (L = 1) and x < 0 odd); outside both: background 0.5.  Also: a single card
    covering the whole plane reproduces shade_plane bit for bit."""
    near = {"z_mm": -100.0, "period_mm": 1e9, "contrast": 1.0, "x0_mm": -10.0, "x1_mm": 10.0, "y0_mm": -5.0,
            "y1_mm": 5.0}
    far = {"z_mm": -500.0, "period_mm": 1e9, "contrast": 0.25, "x0_mm": -40.0, "x1_mm": 40.0, "y0_mm": -40.0,
           "y1_mm": 40.0}
    xs = np.array([0.0, 5.0, -20.0, 20.0, 0.0, 60.0, -30.0], np.float32)
    ys = np.array([0.0, 4.0, 0.0, 0.0, 20.0, 0.0, -50.0], np.float32)
    n = xs.size
    ones, zeros = np.ones(n, np.float32), np.zeros(n, np.float32)
    f = oracle.shade_cards([far, near], 0.5, 0.0, np.ones(n, bool), xs, ys, zeros, zeros, -ones, ones, spp=1,
                           pixels=n)
    L = f / 2.0 ** 32
    # x = -20 hits the far card at x < 0: floor(-20/1e9) = -1 -> odd -> contrast 0.25
    assert np.allclose(L, [1.0, 1.0, 0.25, 1.0, 1.0, 0.5, 0.5]), L
    # card order does not matter (nearest wins), single all-covering card == shade_plane
    assert np.array_equal(f, oracle.shade_cards([near, far], 0.5, 0.0, np.ones(n, bool), xs, ys, zeros, zeros,
                                                -ones, ones, spp=1, pixels=n))
    rng = np.random.default_rng(1)
    m = 4096
    px, py = rng.uniform(-30, 30, m).astype(np.float32), rng.uniform(-30, 30, m).astype(np.float32)
    dx, dy = rng.uniform(-0.2, 0.2, m).astype(np.float32), rng.uniform(-0.2, 0.2, m).astype(np.float32)
    dz = -np.sqrt(1 - dx.astype(np.float64) ** 2 - dy.astype(np.float64) ** 2).astype(np.float32)
    I = rng.uniform(0.5, 1.0, m).astype(np.float32)
    val = rng.random(m) < 0.8
    scene = {"z_mm": -300.0, "period_mm": 7.0, "contrast": 0.3}
    whole = {"z_mm": -300.0, "period_mm": 7.0, "contrast": 0.3, "x0_mm": -1e9, "x1_mm": 1e9, "y0_mm": -1e9,
             "y1_mm": 1e9}
    a = oracle.shade_plane(scene, 0.0, val, px, py, dx, dy, dz, I, spp=4, pixels=m // 4, scale=0.5)
    b = oracle.shade_cards([whole], 0.0, 0.0, val, px, py, dx, dy, dz, I, spp=4, pixels=m // 4, scale=0.5)
    assert np.array_equal(a, b)
