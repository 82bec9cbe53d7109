"""Pins of the paraxial pupils (SURVEY §8(f) NEXT-3 exit-pupil sampling): with a pinhole
aperture stop, the exact (oracle) backward trace of rays from a near-axis sensor point
aimed at points of the axis passes the stop only when aimed at the paraxial exit pupil;
forward rays from an object point pass only when aimed at the entrance pupil."""
import numpy as np

import oracle
from plt_inputs import configs as C
from plt_inputs.lenses import LENSES

LD = 587.5618


def _pinhole(text, d=0.01):
    out = []
    for line in text.splitlines():
        body = line.split("#", 1)[0].split()
        if len(body) >= 4 and body[2].lower() == "stop":
            body[3] = repr(d)
            line = " ".join(body)
        out.append(line)
    return "\n".join(out) + "\n"


def _centre(z, valid):
    assert valid.sum() >= 3
    return float(z[valid].mean())


def test_exit_pupil_is_where_backward_rays_through_the_stop_aim():
    opts = C.CONFIGS["C3"]["opts"]
    lens = oracle.load_lens(_pinhole(LENSES["wide24"]), opts)
    z_ent, r_ent, z_ex, r_ex = oracle.pupils(oracle.load_lens(LENSES["wide24"], opts), LD)
    zs = opts["sensor_z_mm"]
    z = np.linspace(z_ex - 1.5, z_ex + 1.5, 6001)
    x0 = 1.0                                   # near-axis sensor point
    v = np.stack([-x0 * np.ones_like(z), np.zeros_like(z), z - zs], 1)
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    rays = {"ox": np.full(z.size, x0), "oy": np.zeros(z.size), "dx": v[:, 0], "dy": v[:, 1], "dz": v[:, 2],
            "lambda_nm": np.full(z.size, LD), "plane_z": zs}
    t = oracle.trace(lens, oracle.all_t_id(lens.n_optical), 1, rays)
    assert abs(_centre(z, t["valid"]) - z_ex) < 0.02


def test_entrance_pupil_is_where_forward_rays_through_the_stop_aim():
    lens = oracle.load_lens(_pinhole(LENSES["dgauss50"]))
    z_ent, r_ent, z_ex, r_ex = oracle.pupils(oracle.load_lens(LENSES["dgauss50"]), LD)
    z = np.linspace(z_ent - 1.5, z_ent + 1.5, 6001)
    y0, z0 = 0.3, -200.0                       # object point, near the axis
    v = np.stack([np.zeros_like(z), -y0 * np.ones_like(z), z - z0], 1)
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    # start the rays on the input plane z = -5 along the same lines
    s = (-5.0 - z0) / v[:, 2]
    rays = {"ox": np.zeros(z.size), "oy": y0 + s * v[:, 1], "dx": v[:, 0], "dy": v[:, 1], "dz": v[:, 2],
            "lambda_nm": np.full(z.size, LD), "plane_z": -5.0}
    t = oracle.trace(lens, oracle.all_t_id(lens.n_optical), 0, rays)
    assert abs(_centre(z, t["valid"]) - z_ent) < 0.02


def test_pupil_radii_scale_with_the_stop():
    base = oracle.load_lens(LENSES["wide24"])
    half = oracle.load_lens(_pinhole(LENSES["wide24"], 2 * base.surfaces[[s.is_stop for s in base.surfaces].index(True)].a * 0.5))
    a, b = oracle.pupils(base, LD), oracle.pupils(half, LD)
    assert np.allclose([b[0], b[2]], [a[0], a[2]]) and np.allclose([b[1], b[3]], [0.5 * a[1], 0.5 * a[3]])
