"""Pins for oracle O9-O10 (MLP + factorised map wrapper) and O11 (splat).  CPU only."""
import json
import math
import os

import numpy as np
import torch

import oracle
from plt_inputs import configs as C
from plt_inputs import rays as R

G = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_values.json")))


def test_mlp_zero_weights_give_bias():
    head = {"dims": [4, 32, 32, 6],
            "W": [np.zeros((32, 4)), np.zeros((32, 32)), np.zeros((6, 32))],
            "b": [np.full(32, 0.3), np.full(32, -0.2), np.arange(6, dtype=float)]}
    y = oracle.mlp_forward(head, np.random.default_rng(0).normal(size=(5, 4)))
    assert np.array_equal(y, np.tile(np.arange(6, dtype=float), (5, 1)))


def test_mlp_hand_set_single_unit():
    head = {"dims": [1, 1, 1], "W": [np.array([[0.5]]), np.array([[2.0]])],
            "b": [np.array([0.1]), np.array([-0.3])]}
    x = np.array([[-3.0], [0.0], [0.7]])
    y = oracle.mlp_forward(head, x)[:, 0]
    assert np.max(np.abs(y - (2.0 * np.tanh(0.5 * x[:, 0] + 0.1) - 0.3))) < 1e-15


def test_mlp_matches_torch_float64():
    m = oracle.parse_map_blob(C.map_blob("C2", 1 << 10))
    x = np.random.default_rng(1).uniform(-1, 1, size=(2000, 4))
    for key in ("classifier", "regressor"):
        h = m[key]
        t = torch.from_numpy(x)
        for li, (W, b) in enumerate(zip(h["W"], h["b"])):
            t = torch.nn.functional.linear(t, torch.from_numpy(W), torch.from_numpy(b))
            if li + 1 < len(h["W"]):
                t = torch.tanh(t)
        assert np.max(np.abs(oracle.mlp_forward(h, x) - t.numpy())) < 1e-13


def _rays(n=5000, seed=3):
    r = R.gen_rays(C.CONFIGS["C2"]["law"], seed, 0, n)
    return r


def test_map_gate_contract_and_zero_invalid():
    blob = C.map_blob("C2", 1 << 10)
    m = oracle.parse_map_blob(blob)
    r = _rays()
    out = oracle.map_eval(m, r)
    v = out["valid"]
    assert np.array_equal(v, out["raw"][:, 0] >= 0.0)           # valid <=> logit >= 0 (A13)
    assert 0.05 < v.mean() < 0.95
    for k in ("px", "py", "dx", "dy", "dz", "I"):
        assert np.all(out[k][~v] == 0.0)                          # {} -> zeros
    assert np.all(out["raw"][~v, 1:] == 0.0)
    d = np.stack([out["dx"][v], out["dy"][v], out["dz"][v]])
    assert np.max(np.abs(np.linalg.norm(d, axis=0) - 1.0)) < 1e-14
    assert out["I"][v].min() >= 0.0 and out["I"][v].max() <= 1.0


def _normalize(x, m):
    lo, hi = m["norm"][:4], m["norm"][4:8]
    return np.clip(2.0 * (x - lo) / (hi - lo) - 1.0, -1.0, 1.0)


def test_map_identity_on_canonical_inputs_and_regressor_value():
    """Canonical inputs (p on +x, w_y >= 0) are not transformed; raw outputs are
    exactly the classifier / regressor of the normalised input (factorisation)."""
    m = oracle.parse_map_blob(C.map_blob("C2", 1 << 10))
    rng = np.random.default_rng(5)
    n = 3000
    r_ = rng.uniform(0.1, 13.0, n)
    th = np.radians(rng.uniform(0, 25, n))
    ph = rng.uniform(0, math.pi, n)
    f = np.float32
    rays = {"ox": r_.astype(f), "oy": np.zeros(n, f), "dx": (np.sin(th) * np.cos(ph)).astype(f),
            "dy": (np.sin(th) * np.sin(ph)).astype(f), "dz": np.cos(th).astype(f),
            "lambda_nm": rng.uniform(400, 700, n).astype(f), "plane_z": -5.0}
    out = oracle.map_eval(m, rays)
    x = np.stack([np.asarray(rays[k], np.float64) for k in ("ox", "dx", "dy", "lambda_nm")], 1)
    xh = _normalize(x, m)
    logit = oracle.mlp_forward(m["classifier"], xh)[:, 0]
    assert np.max(np.abs(out["raw"][:, 0] - logit)) < 1e-14
    v = out["valid"]
    y = oracle.mlp_forward(m["regressor"], xh[v])
    assert np.max(np.abs(out["raw"][v, 1:] - y)) < 1e-14
    q = m["norm"][8:14] + m["norm"][14:20] * y
    assert np.max(np.abs(out["px"][v] - q[:, 0])) < 1e-12
    assert np.max(np.abs(out["py"][v] - q[:, 1])) < 1e-12


def test_map_symmetry_and_canonicalize_3_4():
    """Rotations (exact 90 deg in float32) and reflections commute with the map (Eq. 10)."""
    m = oracle.parse_map_blob(C.map_blob("C2", 1 << 10))
    r = _rays(4000, 9)
    base = oracle.map_eval(m, r)
    rot = dict(r)
    rot["ox"], rot["oy"] = -r["oy"], r["ox"]
    rot["dx"], rot["dy"] = -r["dy"], r["dx"]
    o = oracle.map_eval(m, rot)
    safe = np.abs(base["raw"][:, 0]) > 1e-9
    assert np.array_equal(o["valid"][safe], base["valid"][safe])
    v = o["valid"] & base["valid"]
    assert np.max(np.abs(o["px"][v] + base["py"][v])) < 1e-11
    assert np.max(np.abs(o["py"][v] - base["px"][v])) < 1e-11
    assert np.max(np.abs(o["I"][v] - base["I"][v])) < 1e-12
    ref = dict(r)
    ref["oy"], ref["dy"] = -r["oy"], -r["dy"]
    o = oracle.map_eval(m, ref)
    assert np.array_equal(o["valid"], base["valid"])
    assert np.max(np.abs(o["py"] + base["py"])) < 1e-12
    # (3,4) -> r = 5: p = (3,4) with w rotated like p is the same query as p = (5,0)
    g = G["canonicalize_3_4"]
    c, s = 3 / 5, 4 / 5
    w0 = np.array([0.1, 0.2, math.sqrt(1 - 0.05)])
    q1 = {"ox": np.array([g["r"]], np.float64), "oy": np.array([0.0]), "dx": np.array([w0[0]]),
          "dy": np.array([w0[1]]), "dz": np.array([w0[2]]), "lambda_nm": np.array([550.0]),
          "plane_z": -5.0}
    q2 = dict(q1)
    q2["ox"], q2["oy"] = np.array([3.0]), np.array([4.0])
    q2["dx"], q2["dy"] = np.array([c * w0[0] - s * w0[1]]), np.array([s * w0[0] + c * w0[1]])
    a, b = oracle.map_eval(m, q1), oracle.map_eval(m, q2)
    assert np.max(np.abs(a["raw"] - b["raw"])) < 1e-12


FILM = {"width_px": 64, "height_px": 32, "channels": 3, "sensor_w_mm": 24.0, "sensor_h_mm": 16.0,
        "center_x_mm": 0.0, "center_y_mm": 0.0}


def test_splat_centre_single_pixel_and_orientation():
    ix, iy = 10, 3
    x = -12.0 + (ix + 0.5) * 24.0 / 64
    y = 8.0 - (iy + 0.5) * 16.0 / 32
    film, dropped = oracle.splat(FILM, [1], [x], [y], [-0.8], [0.5], channel=[2], scale=1.0)
    nz = np.argwhere(film)
    assert dropped == 0 and nz.tolist() == [[2, iy, ix]]
    assert film[2, iy, ix] == round(0.5 * 0.800000011920929 * 2 ** 32)


def test_splat_conservation_order_independence_and_drops():
    rng = np.random.default_rng(2)
    n = 20000
    px = rng.uniform(-14, 14, n).astype(np.float32)
    py = rng.uniform(-9, 9, n).astype(np.float32)
    dz = rng.uniform(0.5, 1, n).astype(np.float32)
    I = rng.uniform(0, 1, n).astype(np.float32)
    v = rng.random(n) < 0.7
    ch = rng.integers(0, 3, n).astype(np.uint8)
    film, dropped = oracle.splat(FILM, v, px, py, dz, I, ch, scale=1e-3)
    inside = v & (np.abs(px) < 12) & (np.abs(py) < 8)
    assert dropped == int((v & ~inside).sum())
    w = I.astype(np.float64) * dz * np.float64(np.float32(1e-3)) * 2 ** 32
    assert abs(film.sum() - w[inside].sum()) <= 0.5 * inside.sum() + 1
    perm = rng.permutation(n)
    film2, _ = oracle.splat(FILM, v[perm], px[perm], py[perm], dz[perm], I[perm], ch[perm], 1e-3)
    assert np.array_equal(film, film2)
