"""Pins for the oracle trace (O2-O8): closed forms, an independent brute-force
singlet tracer, Eq. 10 symmetry, backward/forward reciprocity, ABCD
third-order convergence and sum_P I <= 1.  CPU only."""
import json
import math
import os

import numpy as np
import pytest

import oracle
from oracle.lens import ghost_id
from plt_inputs import configs as C
from plt_inputs import rays as R
from plt_inputs.lenses import LENSES

G = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_values.json")))
LF, LD, LC = R.LAMBDA_F, R.LAMBDA_D, R.LAMBDA_C


def rays_of(ox, oy, dx, dy, dz, lam, plane_z):
    a = lambda v: np.atleast_1d(np.asarray(v, dtype=np.float64))
    n = max(a(v).size for v in (ox, oy, dx, dy, dz, lam))
    b = lambda v: np.broadcast_to(a(v), (n,)).copy()
    return {"ox": b(ox), "oy": b(oy), "dx": b(dx), "dy": b(dy), "dz": b(dz), "lambda_nm": b(lam),
            "plane_z": plane_z}


def fresnel_angle_form(n1, n2, ti):
    """Independent textbook form: Rs = sin^2(ti-tt)/sin^2(ti+tt), Rp = tan^2(ti-tt)/tan^2(ti+tt)."""
    if ti == 0.0:
        return ((n1 - n2) / (n1 + n2)) ** 2
    tt = math.asin(n1 / n2 * math.sin(ti))
    rs = math.sin(ti - tt) ** 2 / math.sin(ti + tt) ** 2
    rp = math.tan(ti - tt) ** 2 / math.tan(ti + tt) ** 2
    return 0.5 * (rs + rp)


SLAB = "name slab\n0 2.0 n:1.5 40\n0 0.0 air 40\n"


def test_normal_incidence_slab_fresnel_and_ghost():
    lens = oracle.load_lens(SLAB, {"sensor_z_mm": 10.0})
    r = rays_of(0.0, 0.0, 0.0, 0.0, 1.0, 550.0, -5.0)
    t = oracle.trace(lens, 1 << 2, 0, r)
    g = G["fresnel_normal_1_to_1p5"]
    assert t["valid"][0] and abs(t["I"][0] - g["T"] ** 2) < 1e-15
    gh = oracle.trace(lens, ghost_id(2, 2, 1), 0, r)
    assert gh["valid"][0] and abs(gh["I"][0] - g["T"] * g["R"] * g["R"] * g["T"]) < 1e-15
    assert gh["px"][0] == 0.0 and gh["dz"][0] == 1.0


def test_oblique_slab_snell_fresnel_displacement():
    lens = oracle.load_lens(SLAB, {"sensor_z_mm": 10.0})
    ti = math.radians(30.0)
    r = rays_of(0.0, 0.0, math.sin(ti), 0.0, math.cos(ti), 550.0, -5.0)
    t = oracle.trace(lens, 1 << 2, 0, r)
    tt = math.radians(G["snell_30deg_1_to_1p5_theta_t_deg"]["value"])
    assert abs(math.asin(math.sin(ti) / 1.5) - tt) < 1e-14
    Rf = fresnel_angle_form(1.0, 1.5, ti)
    assert abs(t["I"][0] - (1 - Rf) ** 2) < 1e-14
    x = 5.0 * math.tan(ti) + 2.0 * math.tan(tt) + 8.0 * math.tan(ti)
    assert abs(t["px"][0] - x) < 1e-12
    assert abs(t["dx"][0] - math.sin(ti)) < 1e-15 and abs(t["dz"][0] - math.cos(ti)) < 1e-15


def test_tir_on_transmission_step_is_absorbed():
    # n = 2 hemisphere-ish front (R=10) + planar rear; a ray at 75 deg incidence is bent to
    # ~46 deg inside, beyond the 30 deg critical angle of 2 -> 1 at the rear face.
    lens = oracle.load_lens("name tir\n10 3.0 n:2.0 20\n0 0 air 40\n", {"sensor_z_mm": 20.0})
    h = 10.0 * math.sin(math.radians(75.0))
    r = rays_of(0.0, h, 0.0, 0.0, 1.0, 550.0, -5.0)
    t = oracle.trace(lens, 1 << 2, 0, r)
    assert not t["valid"][0]
    # the same geometry at small height transmits and satisfies R+T=1 bookkeeping
    r2 = rays_of(0.0, 0.5, 0.0, 0.0, 1.0, 550.0, -5.0)
    assert oracle.trace(lens, 1 << 2, 0, r2)["valid"][0]


def test_axial_throughput_product_and_sum_le_one():
    lens = oracle.load_lens(LENSES["singlet"])
    for lam in (LF, LD, LC):
        n = oracle.glass_index(lens.surfaces[1].glass_after, lam)
        R0 = ((1 - n) / (1 + n)) ** 2
        t = oracle.trace(lens, 1 << 2, 0, rays_of(0, 0, 0, 0, 1, lam, -5.0))
        assert abs(t["I"][0] - (1 - R0) ** 2) < 1e-15
    # sum over all paths of I_out <= 1, dGauss, random rays
    d = oracle.load_lens(LENSES["dgauss50"])
    rays = R.gen_rays(C.CONFIGS["C2"]["law"], 7, 0, 3000)
    ids, _ = oracle.enumerate_ghosts(d, 2)
    tot = np.zeros(3000)
    for pid in ids:
        t = oracle.trace(d, pid, 0, rays)
        assert np.all(t["I"][t["valid"]] > 0) and np.all(t["I"] <= 1.0)
        tot += np.where(t["valid"], t["I"], 0.0)
    assert tot.max() <= 1.0 + 1e-12


# ---------------------------------------------------------------------------
# Independent brute-force singlet tracer (T1): bisection on the sag z(rho),
# normal from the sag derivative, angle-form Snell and Fresnel.
# ---------------------------------------------------------------------------
def _sag(R, zs, rho):
    return zs + R - math.copysign(math.sqrt(R * R - rho * rho), R)


def _bf_intersect(o, w, zs, R, a):
    if R == 0.0:
        t = (zs - o[2]) / w[2]
    else:
        zext = _sag(R, zs, min(a, abs(R)) * 0.999999)
        z0, z1 = min(zs, zext) - 1e-3, max(zs, zext) + 1e-3
        ta, tb = (z0 - o[2]) / w[2], (z1 - o[2]) / w[2]
        ta, tb = min(ta, tb), max(ta, tb)

        def g(t):
            p = o + t * w
            rho = math.hypot(p[0], p[1])
            if rho >= abs(R):
                return None
            return p[2] - _sag(R, zs, rho)
        ga, gb = g(ta), g(tb)
        if ga is None or gb is None or ga * gb > 0:
            return None
        for _ in range(200):
            tm = 0.5 * (ta + tb)
            gm = g(tm)
            if gm is None:
                return None
            if (gm > 0) == (ga > 0):
                ta, ga = tm, gm
            else:
                tb = tm
            if tb - ta < 1e-15:
                break
        t = 0.5 * (ta + tb)
    p = o + t * w
    if math.hypot(p[0], p[1]) > a:
        return None
    return p


def _bf_normal(p, zs, R):
    if R == 0.0:
        return np.array([0.0, 0.0, 1.0])
    rho = math.hypot(p[0], p[1])
    dz = math.copysign(1.0, R) * rho / math.sqrt(R * R - rho * rho)  # d sag / d rho
    if rho == 0:
        nv = np.array([0.0, 0.0, 1.0])
    else:
        nv = np.array([-dz * p[0] / rho, -dz * p[1] / rho, 1.0])
    return nv / np.linalg.norm(nv)


def _bf_interact(w, nv, n1, n2, kind):
    c = float(np.dot(w, nv))
    s = math.copysign(1.0, c)              # w = cos(ti) (s nv) + sin(ti) e
    ti = math.acos(min(1.0, abs(c)))
    tang = w - c * nv
    tn = np.linalg.norm(tang)
    e = tang / tn if tn > 0 else np.zeros(3)
    sin_t = n1 / n2 * math.sin(ti)
    if sin_t > 1.0:
        if kind == "T":
            return None, None
        return -math.cos(ti) * s * nv + math.sin(ti) * e, 1.0
    tt = math.asin(sin_t)
    Rf = fresnel_angle_form(n1, n2, ti)
    if kind == "T":
        return math.cos(tt) * s * nv + sin_t * e, 1.0 - Rf
    return -math.cos(ti) * s * nv + math.sin(ti) * e, Rf


def bruteforce_singlet(ray, lam, seq, z_out):
    stop_a, zs1, zs2, Rr, a = 8.0, 5.0, 10.0, 50.0, 12.5
    n = oracle.glass_index(oracle.load_lens(LENSES["singlet"]).surfaces[1].glass_after, lam)
    o = np.array(ray[:3], float)
    w = np.array(ray[3:], float)
    w = w / np.linalg.norm(w)
    # stop plane
    p = o + (0.0 - o[2]) / w[2] * w
    if math.hypot(p[0], p[1]) > stop_a:
        return None
    o = p
    surf = [(zs1, Rr, 1.0, n), (zs2, -Rr, n, 1.0)]
    idx, d, I = 0, +1, 1.0
    for kind in seq:
        zs, Rs, nb, na = surf[idx]
        p = _bf_intersect(o, w, zs, Rs, a)
        if p is None:
            return None
        nv = _bf_normal(p, zs, Rs)
        n1, n2 = (nb, na) if d > 0 else (na, nb)
        w, f = _bf_interact(w, nv, n1, n2, kind)
        if w is None:
            return None
        I *= f
        o = p
        if kind == "R":
            d = -d
        idx += d
    if d < 0 or idx != 2:
        return None
    t = (z_out - o[2]) / w[2]
    return np.array([o[0] + t * w[0], o[1] + t * w[1], w[0], w[1], w[2], I])


@pytest.mark.parametrize("seq,pid", [(["T", "T"], 4), (["T", "R", "R", "T"], ghost_id(2, 2, 1))])
def test_bruteforce_singlet_agreement(seq, pid):
    lens = oracle.load_lens(LENSES["singlet"])
    z_out = lens.opts["sensor_z_mm"]
    rng = np.random.default_rng(11)
    n = 300
    rays = R.gen_rays(C.CONFIGS["C1"]["law"], 99, 0, n)
    rays["lambda_nm"] = rng.uniform(400, 700, n).astype(np.float32)
    t = oracle.trace(lens, pid, 0, rays)
    nval = 0
    for i in range(n):
        ray = [float(rays["ox"][i]), float(rays["oy"][i]), -5.0,
               float(rays["dx"][i]), float(rays["dy"][i]), float(rays["dz"][i])]
        bf = bruteforce_singlet(ray, float(rays["lambda_nm"][i]), seq, z_out)
        marg = t["margins"][i, 0]
        if marg < 1e-9:
            continue
        assert (bf is not None) == bool(t["valid"][i]), i
        if bf is None:
            continue
        nval += 1
        got = np.array([t[k][i] for k in ("px", "py", "dx", "dy", "dz", "I")])
        assert np.max(np.abs(got[:2] - bf[:2])) < 1e-9
        assert np.max(np.abs(got[2:5] - bf[2:5])) < 1e-11
        assert abs(got[5] - bf[5]) < 1e-12
    assert nval > 20


def test_snell_identity_at_single_surface():
    # output plane inside the glass: the exit direction is the refracted direction at the hit
    lens = oracle.load_lens("name one\n40 0 n:1.6 30\n", {"sensor_z_mm": 3.0})
    rays = R.gen_rays({"kind": "disc_cap", "plane_z": -5.0, "disc_r": 10.0, "cap_deg": 20.0,
                       "lam": 550.0}, 5, 0, 500)
    t = oracle.trace(lens, 1 << 1, 0, rays)
    assert t["valid"].all()
    for i in range(0, 500, 7):
        o = np.array([rays["ox"][i], rays["oy"][i], -5.0], float)
        w = np.array([rays["dx"][i], rays["dy"][i], rays["dz"][i]], float)
        w /= np.linalg.norm(w)
        p = _bf_intersect(o, w, 0.0, 40.0, 15.0)
        nv = _bf_normal(p, 0.0, 40.0)
        wt = np.array([t["dx"][i], t["dy"][i], t["dz"][i]])
        # n1 (w x n) = n2 (wt x n): tangential components match
        assert np.max(np.abs(1.0 * np.cross(w, nv) - 1.6 * np.cross(wt, nv))) < 1e-12
        assert abs(np.linalg.norm(wt) - 1.0) < 1e-14


def _rot(x, y, c, s):
    return c * x - s * y, s * x + c * y


@pytest.mark.parametrize("lensname,pid_fn", [("dgauss50", lambda m: 1 << m),
                                            ("dgauss50", lambda m: ghost_id(m, 7, 3)),
                                            ("wide22", lambda m: 1 << m)])
def test_rotation_and_reflection_symmetry(lensname, pid_fn):
    """Eq. 10: T(R p, R w) = R T(p, w) for rotations about the axis and
    reflections in planes containing it."""
    lens = oracle.load_lens(LENSES[lensname])
    pid = pid_fn(lens.n_optical)
    r = R.gen_rays(C.CONFIGS["C2"]["law"], 21, 0, 4000)
    r = {k: (np.asarray(v, np.float64) if k != "plane_z" else v) for k, v in r.items()}
    base = oracle.trace(lens, pid, 0, r)
    rng = np.random.default_rng(3)
    for _ in range(3):
        ang = rng.uniform(0, 2 * math.pi)
        c, s = math.cos(ang), math.sin(ang)
        rr = dict(r)
        rr["ox"], rr["oy"] = _rot(r["ox"], r["oy"], c, s)
        rr["dx"], rr["dy"] = _rot(r["dx"], r["dy"], c, s)
        t = oracle.trace(lens, pid, 0, rr)
        safe = base["margins"][:, 0] > 1e-9
        assert np.array_equal(t["valid"][safe], base["valid"][safe])
        v = base["valid"] & t["valid"]
        px, py = _rot(base["px"], base["py"], c, s)
        dx, dy = _rot(base["dx"], base["dy"], c, s)
        assert np.max(np.abs(t["px"][v] - px[v])) < 1e-10
        assert np.max(np.abs(t["dy"][v] - dy[v])) < 1e-12
        assert np.max(np.abs(t["I"][v] - base["I"][v])) < 1e-13
    rr = dict(r)
    rr["oy"], rr["dy"] = -r["oy"], -r["dy"]
    t = oracle.trace(lens, pid, 0, rr)
    assert np.array_equal(t["valid"], base["valid"])
    assert np.array_equal(t["py"], -base["py"]) and np.array_equal(t["I"], base["I"])


def test_backward_forward_reciprocity():
    """All-T map of the mirrored lens is the reverse of the forward map."""
    cfg = C.CONFIGS["C3"]
    lens = oracle.load_lens(LENSES["wide24"], cfg["opts"])
    r = R.gen_rays(cfg["law"], 3, 0, 20000)
    b = oracle.trace(lens, 1 << 12, 1, r)
    v = b["valid"]
    assert 0.03 < v.mean() < 0.15
    back = {"ox": b["px"][v], "oy": b["py"][v], "dx": -b["dx"][v], "dy": -b["dy"][v],
            "dz": -b["dz"][v], "lambda_nm": np.asarray(r["lambda_nm"][v], np.float64),
            "plane_z": cfg["opts"]["backward_exit_z_mm"]}
    f = oracle.trace(lens, 1 << 12, 0, back)
    assert f["valid"].all()
    assert np.max(np.abs(f["px"] - r["ox"][v])) < 1e-9
    assert np.max(np.abs(f["py"] - r["oy"][v])) < 1e-9
    d = np.stack([np.asarray(r[k][v], np.float64) for k in ("dx", "dy", "dz")])
    d /= np.linalg.norm(d, axis=0)  # the trace normalises its input direction
    assert np.max(np.abs(f["dz"] + d[2])) < 1e-12 and np.max(np.abs(f["dx"] + d[0])) < 1e-12
    assert np.max(np.abs(f["I"] - b["I"][v])) < 1e-13


def test_abcd_third_order_convergence():
    """Exact trace -> ABCD as h -> 0 with transverse residual ~ h^3 (SURVEY §8(c) O13 pin)."""
    for lam in (LF, LD, LC):
        lens = oracle.load_lens(LENSES["singlet"], {"sensor_z_mm": float("nan"), "lambda_ref_nm": lam})
        zf = lens.opts["sensor_z_mm"]
        hs = np.geomspace(0.02, 0.4, 12)
        rays = rays_of(0.0, hs, 0.0, 0.0, 1.0, lam, -5.0)
        t = oracle.trace(lens, 1 << 2, 0, rays)
        assert t["valid"].all()
        M = oracle.abcd_input_to_plane(lens, lam, -5.0, zf)
        y_abcd = M[0, 0] * hs  # u = 0
        res = np.abs(t["py"] - y_abcd)
        slope = np.polyfit(np.log(hs), np.log(res), 1)[0]
        assert abs(slope - 3.0) < 0.01, slope
        assert res[np.argmin(np.abs(hs - 0.4))] < 5e-5
    # off-axis slopes too: residual vs the ABCD prediction A h + B u is third order in (h, u):
    # halving (h, u) divides it by ~8
    lens = oracle.load_lens(LENSES["singlet"])
    ab = C.c1_abcd_rays()
    M = oracle.abcd_input_to_plane(lens, LD, -5.0, lens.opts["sensor_z_mm"])
    h = np.asarray(ab["oy"], np.float64)
    u = np.asarray(ab["dy"], np.float64) / np.asarray(ab["dz"], np.float64)
    res = []
    for s in (1.0, 0.5):
        rr = rays_of(0.0, s * h, 0.0, s * u, 1.0, LD, -5.0)
        t = oracle.trace(lens, 1 << 2, 0, rr)
        res.append(np.abs(t["py"] - (M[0, 0] * s * h + M[0, 1] * s * u)))
    assert res[0].max() < 6e-5
    big = res[0] > 1e-6
    ratio = res[0][big] / res[1][big]
    assert np.all(np.abs(ratio - 8.0) < 0.5), ratio.min()
