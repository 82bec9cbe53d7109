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
