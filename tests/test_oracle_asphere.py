"""Pins of the oracle's even-asphere surfaces (the paper allows
"aspheric circularly symmetric" surfaces): the Newton intersection and the
sag-gradient normal against an independent bisection tracer with finite-difference
normals, the spherical special case, the h^3 onset of the A4 term, rotational symmetry
and table/JSON equivalence.  CPU only."""
import json
import math

import numpy as np
import pytest

import oracle
from plt_inputs import configs as C
from plt_inputs import rays as R
from plt_inputs.lenses import LENSES

LD = R.LAMBDA_D
# N-BK7 singlet with a front stop (the C1 lens); front surface a strong conic + polynomial asphere
ASPH = (-0.8, 2.0e-6, -3.0e-9, 0.0, 0.0)
TEXT = LENSES["singlet"]


def _with_front_asphere(text, asph):
    out, done = [], False
    for line in text.splitlines():
        body = line.split("#", 1)[0].split()
        if not done and len(body) >= 4 and body[0] != "name" and body[2].lower() not in ("stop", "air") and \
                float(body[0]) != 0.0:
            line = line.split("#", 1)[0].rstrip() + "  asph:" + ",".join(repr(v) for v in asph)
            done = True
        out.append(line)
    return "\n".join(out) + "\n"


def _sag(R_, k, A, rho):
    c = 0.0 if R_ == 0.0 else 1.0 / R_
    q = 1.0 - (1.0 + k) * c * c * rho * rho
    if q < 0:
        return None
    return c * rho * rho / (1.0 + math.sqrt(q)) + sum(a * rho ** (4 + 2 * i) for i, a in enumerate(A))


def _bisect_hit(o, w, zs, R_, k, A, a):
    def g(t):
        p = o + t * w
        s = _sag(R_, k, A, math.hypot(p[0], p[1]))
        return None if s is None else p[2] - zs - s
    t0 = (zs - o[2]) / w[2]
    lo, hi = t0 - 10.0, t0 + 10.0          # the cap lies within 10 mm of the vertex plane here
    glo, ghi = g(lo), g(hi)
    if glo is None or ghi is None or glo * ghi > 0:
        return None
    for _ in range(200):
        m = 0.5 * (lo + hi)
        gm = g(m)
        if gm is None:
            return None
        if (gm > 0) == (glo > 0):
            lo, glo = m, gm
        else:
            hi = m
    p = o + 0.5 * (lo + hi) * w
    return p if math.hypot(p[0], p[1]) <= a else None


def _fd_normal(p, R_, k, A):
    rho = math.hypot(p[0], p[1])
    h = 1e-6
    d = (_sag(R_, k, A, rho + h) - _sag(R_, k, A, max(rho - h, 0.0))) / (rho + h - max(rho - h, 0.0))
    nv = np.array([-d * p[0] / rho, -d * p[1] / rho, 1.0]) if rho > 0 else np.array([0.0, 0.0, 1.0])
    return nv / np.linalg.norm(nv)


def _refract(w, nv, n1, n2):
    if np.dot(w, nv) > 0:
        nv = -nv
    cosi = -np.dot(w, nv)
    eta = n1 / n2
    k = 1 - eta * eta * (1 - cosi * cosi)
    if k < 0:
        return None
    return eta * w + (eta * cosi - math.sqrt(k)) * nv


def test_bisection_tracer_agrees_with_newton():
    lens = oracle.load_lens(_with_front_asphere(TEXT, ASPH))
    s1, s2 = lens.surfaces[1], lens.surfaces[2]
    assert s1.asph and not s2.asph
    n = oracle.glass_index(s1.glass_after, LD)
    rays = R.gen_rays(C.CONFIGS["C1"]["law"], 123, 0, 200)
    rays["lambda_nm"] = np.full(200, LD, np.float32)
    t = oracle.trace(lens, 1 << 2, 0, rays)
    z_out = lens.opts["sensor_z_mm"]
    nval = 0
    for i in range(200):
        o = np.array([rays["ox"][i], rays["oy"][i], -5.0], float)
        w = np.array([rays["dx"][i], rays["dy"][i], rays["dz"][i]], float)
        w /= np.linalg.norm(w)
        p = o + (0.0 - o[2]) / w[2] * w                      # stop at z = 0, a = 8
        ok = math.hypot(p[0], p[1]) <= 8.0
        if ok:
            p1 = _bisect_hit(p, w, s1.z, s1.R, s1.k, s1.A, s1.a)
            ok = p1 is not None
        if ok:
            w1 = _refract(w, _fd_normal(p1 - np.array([0, 0, s1.z]), s1.R, s1.k, s1.A), 1.0, n)
            p2 = _bisect_hit(p1, w1, s2.z, s2.R, 0.0, (0, 0, 0, 0), s2.a)
            ok = p2 is not None
        if ok:
            w2 = _refract(w1, _fd_normal(p2 - np.array([0, 0, s2.z]), s2.R, 0.0, (0, 0, 0, 0)), n, 1.0)
            tt = (z_out - p2[2]) / w2[2]
            exit_ = np.array([p2[0] + tt * w2[0], p2[1] + tt * w2[1], w2[0], w2[1], w2[2]])
        assert bool(t["valid"][i]) == ok, i
        if ok:
            nval += 1
            got = np.array([t[k][i] for k in ("px", "py", "dx", "dy", "dz")])
            assert np.max(np.abs(got[:2] - exit_[:2])) < 1e-6 and np.max(np.abs(got[2:] - exit_[2:])) < 1e-8
    assert nval > 100


def test_spherical_special_case_matches_the_quadratic_root():
    base = oracle.load_lens(TEXT)
    asph = oracle.load_lens(_with_front_asphere(TEXT, (0.0, 0.0, 0.0, 0.0, 0.0)))
    rays = R.gen_rays(C.CONFIGS["C1"]["law"], 5, 0, 2000)
    for pid in (1 << 2, oracle.ghost_id(2, 2, 1)):
        a, b = oracle.trace(base, pid, 0, rays), oracle.trace(asph, pid, 0, rays)
        assert np.array_equal(a["valid"], b["valid"])
        for k in ("px", "py", "dx", "dy", "dz", "I"):
            assert np.max(np.abs(a[k][a["valid"]] - b[k][a["valid"]])) < 1e-10


def test_a4_term_enters_at_third_order():
    """A pure A4 term leaves the paraxial (ABCD) system unchanged and perturbs a ray of
    height h at the surface by O(h^3): halving h divides the exit-slope change by ~8."""
    base = oracle.load_lens(TEXT)
    asph = oracle.load_lens(_with_front_asphere(TEXT, (0.0, 1e-5, 0.0, 0.0, 0.0)))
    z_out = base.opts["sensor_z_mm"]
    assert np.allclose(oracle.lens.abcd_input_to_plane(base, LD, -5.0, z_out),
                       oracle.lens.abcd_input_to_plane(asph, LD, -5.0, z_out), rtol=0, atol=0)
    d = []
    for h in (0.8, 0.4, 0.2):
        r = {"ox": np.array([0.0]), "oy": np.array([h]), "dx": np.zeros(1), "dy": np.zeros(1), "dz": np.ones(1),
             "lambda_nm": np.array([LD]), "plane_z": -5.0}
        a, b = oracle.trace(base, 1 << 2, 0, r), oracle.trace(asph, 1 << 2, 0, r)
        d.append(abs(b["dy"][0] - a["dy"][0]))
    assert 7.0 < d[0] / d[1] < 9.0 and 7.0 < d[1] / d[2] < 9.0


def test_rotational_symmetry_and_json_equivalence():
    text = _with_front_asphere(TEXT, ASPH)
    lens = oracle.load_lens(text)
    rays = R.gen_rays(C.CONFIGS["C1"]["law"], 8, 0, 500)
    phi = 0.7
    c, s = math.cos(phi), math.sin(phi)
    rot = dict(rays, ox=c * rays["ox"] - s * rays["oy"], oy=s * rays["ox"] + c * rays["oy"],
               dx=c * rays["dx"] - s * rays["dy"], dy=s * rays["dx"] + c * rays["dy"])
    a, b = oracle.trace(lens, 1 << 2, 0, rays), oracle.trace(lens, 1 << 2, 0, rot)
    v = a["valid"] & b["valid"]
    assert v.sum() > 100
    assert np.allclose(b["px"][v], c * a["px"][v] - s * a["py"][v], atol=2e-6)   # float32 ray inputs
    doc = {"name": "s", "surfaces": []}
    for sf, nxt in zip(lens.surfaces, lens.surfaces[1:] + [None]):
        e = {"radius_mm": sf.R, "thickness_mm": (nxt.z - sf.z) if nxt else 0.0,
             "glass": "stop" if sf.is_stop else "sellmeier:" + ",".join(map(repr, sf.glass_after[1]))
             if sf.glass_after[0] == 3 else "air", "semi_aperture_mm": sf.a}
        if sf.asph:
            e["conic"], e["aspheric"] = sf.k, list(sf.A)
        doc["surfaces"].append(e)
    lj = oracle.load_lens(json.dumps(doc))
    assert [(x.asph, x.k, x.A) for x in lj.surfaces] == [(x.asph, x.k, x.A) for x in lens.surfaces]


def test_backward_forward_reciprocity_with_aspheres_and_coatings():
    """The mirrored (backward) frame negates the aspheric sag (A' = -A, k unchanged) and
    keeps coatings: backward exit rays of the 24 mm lens with an aspheric, coated element,
    reversed and traced forward, land back on the sensor points they started from."""
    cfg = C.CONFIGS["C3"]
    text = LENSES["wide24"]
    lines, k = [], 0
    for line in text.splitlines():
        body = line.split("#", 1)[0].split()
        if len(body) >= 4 and body[0] != "name" and body[2].lower() != "stop" and float(body[0]) != 0.0:
            k += 1
            if k == 3:
                line = line.split("#", 1)[0].rstrip() + " asph:-0.5,3e-5,-1e-7 coat:1.38,550"
        lines.append(line)
    lens = oracle.load_lens("\n".join(lines) + "\n", cfg["opts"])
    assert sum(s.asph for s in lens.surfaces) == 1
    r = R.gen_rays(cfg["law"], 3, 0, 20000)
    pid = oracle.all_t_id(lens.n_optical)
    b = oracle.trace(lens, pid, 1, r)
    v = b["valid"]
    assert v.sum() > 500
    back = {"ox": b["px"][v], "oy": b["py"][v], "dx": -b["dx"][v], "dy": -b["dy"][v], "dz": -b["dz"][v],
            "lambda_nm": np.asarray(r["lambda_nm"][v], np.float64), "plane_z": cfg["opts"]["backward_exit_z_mm"]}
    f = oracle.trace(lens, pid, 0, back)
    # forward output plane = the sensor plane of the backward rays
    assert f["valid"].all()
    assert np.max(np.abs(f["px"] - r["ox"][v])) < 1e-9 and np.max(np.abs(f["py"] - r["oy"][v])) < 1e-9
    assert np.max(np.abs(f["I"] - b["I"][v])) < 1e-12                 # reciprocity of the film too
