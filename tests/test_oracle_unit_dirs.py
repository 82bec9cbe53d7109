"""Oracle pins for rays given without dz (include/plt.h: omega in S^2_+ of P:180 given by
its (x, y) components; the query completes w_z = +-sqrt(1 - w_x^2 - w_y^2))."""
import numpy as np

import oracle
from plt_inputs import configs as C
from plt_inputs import rays as R


def test_hemisphere_dz_closed_form():
    """(sin t cos p, sin t sin p) completes to cos t, and the sign follows the request."""
    rng = np.random.default_rng(5)
    th = rng.uniform(0, 0.5 * np.pi, 1000)
    ph = rng.uniform(-np.pi, np.pi, 1000)
    dz = oracle.hemisphere_dz(np.sin(th) * np.cos(ph), np.sin(th) * np.sin(ph))
    np.testing.assert_allclose(dz, np.cos(th), atol=2e-8)   # sqrt of a cancellation near grazing
    np.testing.assert_allclose(oracle.hemisphere_dz(0.6, 0.0, -1.0), -0.8, rtol=0, atol=1e-15)
    assert oracle.hemisphere_dz(0.8, 0.7) == 0.0           # outside the unit disc: clamped


def _without_dz(rays):
    r = {k: v for k, v in rays.items() if k != "dz"}
    return r


def test_trace_without_dz_matches_unit_directions():
    """Forward (C2) and backward (C3) traces of rays given without dz equal the traces of the
    same rays with the float32 unit dz up to that dz's rounding (outputs) and agree on the
    mask away from edges."""
    for name, pid_of, direction in (("C2", None, 0), ("C3", None, 1)):
        cfg = C.CONFIGS[name]
        ol = oracle.load_lens(C.lens_text(name), cfg["opts"])
        pid = oracle.all_t_id(ol.n_optical)
        rays = R.gen_rays(cfg["law"], 3, 0, 1 << 13)
        a = oracle.trace(ol, pid, direction, rays)
        b = oracle.trace(ol, pid, direction, _without_dz(rays))
        # the completion has the request's sign and unit length
        want = np.abs(rays["dz"].astype(np.float64))
        got = oracle.hemisphere_dz(rays["dx"], rays["dy"])
        np.testing.assert_allclose(got, want, rtol=0, atol=3e-7)
        both = a["valid"] & b["valid"]
        near = (a["margins"][:, 0] < 1e-4) | (b["margins"][:, 0] < 1e-4)
        assert ((a["valid"] != b["valid"]) & ~near).sum() == 0
        assert both.mean() > 0.05
        for k in ("px", "py"):
            assert np.abs(a[k][both] - b[k][both]).max() < 2e-4, (name, k)
        for k in ("dx", "dy", "dz", "I"):
            assert np.abs(a[k][both] - b[k][both]).max() < 2e-5, (name, k)
        assert np.sign(b["dz"][both]).min() == np.sign(a["dz"][both]).min()


def test_propagate_without_dz_follows_the_query_direction():
    """Absent dz, w_z takes the sign of the query direction (A32, as the trace): a forward ray
    moved to a plane behind it travels backwards along its own line (t < 0), a backward
    (sensor) ray moved upstream or downstream stays on its line with w_z < 0."""
    rng = np.random.default_rng(2)
    th = rng.uniform(0, 0.3, 100)
    dx, dy = np.sin(th), np.zeros(100)
    rays = {"ox": np.zeros(100), "oy": np.zeros(100), "dx": dx, "dy": dy, "lambda_nm": np.full(100, 550.0),
            "plane_z": 10.0}
    fw = oracle.propagate(rays, 20.0)
    fw_back = oracle.propagate(rays, 0.0)                       # forward ray, plane behind it
    np.testing.assert_allclose(fw["ox"], 10.0 * np.tan(th), rtol=1e-12)
    np.testing.assert_allclose(fw_back["ox"], -10.0 * np.tan(th), rtol=1e-12)
    assert (fw["dz"] > 0).all() and (fw_back["dz"] > 0).all()
    for zt, sign in ((0.0, 1.0), (20.0, -1.0)):                 # backward rays (w_z < 0)
        bw = oracle.propagate(rays, zt, direction=oracle.BACKWARD)
        assert (bw["dz"] < 0).all()
        np.testing.assert_allclose(bw["ox"], sign * 10.0 * np.tan(th), rtol=1e-12)
        # the moved origin lies on the original line: (o' - o) parallel to w
        t = (zt - 10.0) / bw["dz"]
        np.testing.assert_allclose(bw["ox"], t * dx, rtol=1e-12, atol=1e-15)
