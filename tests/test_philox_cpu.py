"""CPU checks of the counter-based ray generator (plt_inputs/philox.py; the device twin is
plt_gen_rays): Philox4x32-10 known-answer vectors, the angle polynomial against libm, and
the ray laws' geometry and statistics (SURVEY.md §8(d) input recipe)."""
import json
import math
import os

import numpy as np
import pytest

from plt_inputs import philox as P
from plt_inputs import configs as C
from plt_inputs import rays as R

KAT = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "philox_kat.json")))


@pytest.mark.parametrize("v", KAT["vectors"], ids=range(len(KAT["vectors"])))
def test_philox_known_answers(v):
    c = [np.array([int(x, 16)], np.uint64) for x in v["ctr"]]
    k = [int(x, 16) for x in v["key"]]
    out = P.philox4x32_10(*c, *k)
    assert [int(o[0]) for o in out] == [int(x, 16) for x in v["out"]]


def test_angle_matches_libm_and_is_unit():
    u = np.concatenate([np.linspace(0, 1, 100001, endpoint=False), np.random.default_rng(1).random(100000)])
    c, s = P.angle(u)
    # (the reference itself rounds 2 pi u: ulp(2 pi) ~ 8.9e-16)
    assert np.max(np.abs(c - np.cos(2 * math.pi * u))) < 2e-15
    assert np.max(np.abs(s - np.sin(2 * math.pi * u))) < 2e-15
    assert np.max(np.abs(c * c + s * s - 1.0)) < 6e-16


def test_uniforms_are_open_unit_interval_and_uniform():
    u = P.uniforms(7, np.arange(1 << 18))
    assert u.min() > 0.0 and u.max() < 1.0
    assert np.all(np.abs(u.mean(axis=1) - 0.5) < 4 * math.sqrt(1 / 12 / (1 << 18)))
    # distinct words are uncorrelated
    cc = np.corrcoef(u)
    assert np.max(np.abs(cc - np.eye(8))) < 0.01


def test_counter_based_any_index_any_split():
    law = C.CONFIGS["C5"]["law"]
    a = R.gen_rays(law, 5, (1 << 33) - 1000, 3000)            # crosses 2^33: counter high word
    b = R.gen_rays_at(law, 5, np.arange((1 << 33) - 1000, (1 << 33) + 2000)[::-1].copy())
    for k in ("ox", "oy", "dx", "dy", "dz", "lambda_nm"):
        assert np.array_equal(a[k], b[k][::-1])


@pytest.mark.parametrize("name", ["C3", "C5"])
def test_law_geometry_and_statistics(name):
    cfg = C.CONFIGS[name]
    law = cfg["law"]
    n = 1 << 18
    r = R.gen_rays(law, cfg["seed"], 12345, n)
    d = np.stack([r[k].astype(np.float64) for k in ("dx", "dy", "dz")])
    assert np.max(np.abs(np.linalg.norm(d, axis=0) - 1.0)) < 3e-7
    lam = r["lambda_nm"].astype(np.float64)
    assert lam.min() >= 400.0 and lam.max() <= 700.0 and abs(lam.mean() - 550.0) < 1.0
    if law["kind"] == "disc_cap":
        rho = np.hypot(r["ox"], r["oy"])
        assert rho.max() <= law["disc_r"] * (1 + 1e-6)
        # uniform on the disc: P(rho < R/2) = 1/4
        assert abs((rho < law["disc_r"] / 2).mean() - 0.25) < 0.005
        assert d[2].min() >= math.cos(math.radians(law["cap_deg"])) - 1e-6
        # uniform on the cap: w_z uniform on [cos a, 1]
        assert abs(d[2].mean() - (1 + math.cos(math.radians(law["cap_deg"]))) / 2) < 5e-4
    else:
        assert np.abs(r["ox"]).max() <= law["sensor_w"] / 2 and np.abs(r["oy"]).max() <= law["sensor_h"] / 2
        # every direction aims at a point of the pupil disc
        t = (law["pupil_z"] - law["plane_z"]) / d[2]
        qx, qy = r["ox"] + t * d[0], r["oy"] + t * d[1]
        assert np.hypot(qx, qy).max() <= law["pupil_r"] * (1 + 1e-5)
        assert (d[2] < 0).all()
