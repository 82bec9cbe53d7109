"""float64 CPU ORACLE of the per-ray lens transport query.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference``) may import,
call, link or execute anything under ``oracle/``.  The product package
(``paper_2605_04017_b200``) never imports it and shares no code with it.

What it computes (citations: P = /root/reference/PAPER.md, S = SPEC.md,
O/A = SURVEY.md §8(c) steps/readings, restated in DESIGN.md):

* ``trace``      -- exact sequential trace T^P (Eq. 5-7) with the
                    validity rule of P:218, in IEEE double (oracle.c O2-O8).
* ``map_eval``   -- factorised network {y} = f(x) if g(x) = 1 else {}
                    with exact tanh on the blob's bf16 weights widened to double
                    (O9-O10), symmetry canonicalisation of §4.1.
* ``splat``      -- film accumulation of Eq. 8 / Listing 1
                    in int64 fixed point 2^-32 (O11).
* ``shade_plane``-- backward camera integrand on a checkerboard scene plane (O14,
                    Eq. 9); ``propagate``: free-space
                    ray propagation (closed form).
* ``lens``       -- glass (O1), ABCD (O13), path ids (O2), ghosts (O12).

Pins (tests/test_oracle_*.py) tie every function to something other than
itself: SPEC worked values, closed forms (lensmaker, normal-incidence Fresnel),
an independent brute-force singlet tracer, symmetry, reciprocity, ABCD
third-order convergence, torch float64 for the MLP, and the map-vs-trace relation
through fitted maps (maps/, trained on this oracle's labels by tests/fit_map.py):
map_eval reproduces trace to the fitting error (tests/test_oracle_map_vs_trace.py).
"""
from __future__ import annotations

import math
import os
import struct
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from . import _lib
from .lens import (OracleLens, all_t_id, decode_path, efl_bfl, encode_path,  # noqa: F401
                   enumerate_ghosts, ghost_id, mirrored, parse_lens, paraxial_focus_z, pupils,
                   surface_array, abcd_vertex_to_vertex, abcd_input_to_plane, glass_index)

FORWARD, BACKWARD = 0, 1


def build():
    return _lib.build()


def load_lens(text: str, opts: dict | None = None) -> OracleLens:
    """Parse + resolve lens options (sensor z NaN -> paraxial focus at lambda_ref)."""
    o = {"input_plane_z_mm": -5.0, "sensor_z_mm": float("nan"), "sensor_w_mm": 0.0,
         "sensor_h_mm": 0.0, "backward_exit_z_mm": -5.0, "housing_radius_mm": 0.0,
         "lambda_ref_nm": 587.5618}
    o.update(opts or {})
    lens = parse_lens(text, o)
    if math.isnan(o["sensor_z_mm"]):
        o["sensor_z_mm"] = paraxial_focus_z(lens, o["lambda_ref_nm"])
    lens.opts = o
    return lens


def _frame(lens: OracleLens, direction: int):
    """Surface array + lens params in the traversal frame (ray travels +z at entry)."""
    o = lens.opts
    if direction == FORWARD:
        S = surface_array(lens.surfaces)
        L = np.array([o["housing_radius_mm"], o["sensor_z_mm"], o["sensor_w_mm"],
                      o["sensor_h_mm"], 0.0, 0.0], dtype=np.float64)
        return S, L, 0.0, +1.0
    zS = lens.surfaces[-1].z
    S = surface_array(mirrored(lens))
    L = np.array([o["housing_radius_mm"], zS - o["backward_exit_z_mm"], 0.0, 0.0, 0.0, 0.0],
                 dtype=np.float64)
    return S, L, zS, -1.0


def _f64(rays, k):
    """Inputs as float64: float32 arrays are widened exactly; float64 arrays pass through."""
    return np.ascontiguousarray(rays[k], dtype=np.float64)


def hemisphere_dz(dx, dy, sign: float = 1.0):
    """z-component of the unit direction omega in S^2_+  given its (x, y)
    components: sign * sqrt(max(0, 1 - dx^2 - dy^2)), in float64 (include/plt.h: rays
    passed without dz)."""
    dx = np.asarray(dx, np.float64)
    dy = np.asarray(dy, np.float64)
    return sign * np.sqrt(np.maximum(0.0, 1.0 - dx * dx - dy * dy))


def _dz(rays, direction_sign: float):
    """The rays' dz, or -- absent / None -- the hemisphere completion towards the lens."""
    if rays.get("dz") is None:
        return np.ascontiguousarray(hemisphere_dz(rays["dx"], rays["dy"], direction_sign))
    return _f64(rays, "dz")


def trace(lens: OracleLens, path_id: int, direction: int, rays: dict, threads: int = 1) -> dict:
    """Exact float64 trace of ``rays`` (float32 arrays widened) along ``path_id``.

    Returns valid (bool), px, py, dx, dy, dz, I (float64) in the ORIGINAL lens
    frame, ``margins`` (n, 4) = (geometric edge mm, |kappa|, |disc| mm^2, |w_z|) and
    ``steps`` (n,) = surface steps begun (stop crossings included, +1 for the output
    plane) before the ray terminated -- bookkeeping for the algorithmic work count.
    """
    S, L, zS, sgn = _frame(lens, direction)
    ox, oy, dx, dy, lam = (_f64(rays, k) for k in ("ox", "oy", "dx", "dy", "lambda_nm"))
    dz = _dz(rays, 1.0 if direction == FORWARD else -1.0)
    n = ox.size
    if sgn < 0:
        plane_z = zS - float(rays["plane_z"])
        dz = np.ascontiguousarray(-dz)
    else:
        plane_z = float(rays["plane_z"])
    valid = np.zeros(n, np.uint8)
    out = np.zeros((n, 6), np.float64)
    marg = np.zeros((n, 4), np.float64)
    steps = np.zeros(n, np.int32)
    lib = _lib.lib()
    p = _lib.ptr

    def run(lo, hi):
        if hi <= lo:
            return
        lib.orc_trace(p(S), S.shape[0], p(L), int(path_id), hi - lo,
                      p(ox[lo:]), p(oy[lo:]), plane_z, p(dx[lo:]), p(dy[lo:]), p(dz[lo:]),
                      p(lam[lo:]), p(valid[lo:]), p(out[lo:]), p(marg[lo:]), p(steps[lo:]))

    _parallel(run, n, threads)
    res = {"valid": valid.astype(bool), "px": out[:, 0].copy(), "py": out[:, 1].copy(),
           "dx": out[:, 2].copy(), "dy": out[:, 3].copy(), "dz": out[:, 4].copy(),
           "I": out[:, 5].copy(), "margins": marg, "steps": steps}
    if sgn < 0:
        res["dz"] = -res["dz"]
        res["dz"][~res["valid"]] = 0.0
    return res


def _parallel(fn, n, threads):
    threads = max(1, int(threads))
    if threads == 1 or n < 4096:
        fn(0, n)
        return
    step = (n + threads - 1) // threads
    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(lambda t: fn(t * step, min(n, (t + 1) * step)), range(threads)))


# ---------------------------------------------------------------------------
# Map blobs (format: plt_inputs/rays.py make_map_blob) -- parsed independently
# ---------------------------------------------------------------------------
def parse_map_blob(blob: bytes) -> dict:
    if blob[:8] != b"PLTMAP01":
        raise ValueError("bad map magic")
    ver, direction, path_id, ncl, nrl = struct.unpack_from("<IIQII", blob, 8)
    off = 8 + struct.calcsize("<IIQII")
    if ver not in (1, 2):
        raise ValueError(f"unsupported map version {ver}")
    plane_z = None
    if ver == 2:                       # the input plane the map was trained on
        (plane_z,) = struct.unpack_from("<d", blob, off)
        off += 8
    norm = np.frombuffer(blob, np.float32, 20, off).astype(np.float64)
    off += 80
    heads = []
    for nl in (ncl, nrl):
        dims, Ws, Bs = [], [], []
        for _ in range(nl):
            fo, fi = struct.unpack_from("<II", blob, off)
            off += 8
            wbits = np.frombuffer(blob, np.uint16, fo * fi, off).astype(np.uint32) << 16
            off += 2 * fo * fi
            Ws.append(wbits.view(np.float32).astype(np.float64).reshape(fo, fi))
            Bs.append(np.frombuffer(blob, np.float32, fo, off).astype(np.float64))
            off += 4 * fo
            if not dims:
                dims.append(fi)
            dims.append(fo)
        heads.append({"dims": dims, "W": Ws, "b": Bs})
    return {"version": ver, "direction": direction, "path_id": path_id, "norm": norm, "plane_z": plane_z,
            "classifier": heads[0], "regressor": heads[1]}


def _head_arrays(h):
    dims = np.array(h["dims"], dtype=np.int32)
    W = np.ascontiguousarray(np.concatenate([w.ravel() for w in h["W"]]))
    B = np.ascontiguousarray(np.concatenate(h["b"]))
    return len(h["dims"]) - 1, dims, W, B


def mlp_forward(head: dict, x: np.ndarray) -> np.ndarray:
    """O9 on a batch x (n, dims[0]) -> (n, dims[-1])."""
    nl, dims, W, B = _head_arrays(head)
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.zeros((x.shape[0], dims[-1]), np.float64)
    p = _lib.ptr
    _lib.lib().orc_mlp_forward(nl, p(dims), p(W), p(B), x.shape[0], p(x), p(y))
    return y


def map_eval(model, rays: dict, threads: int = 1) -> dict:
    """O10 factorised query on float32 rays; returns valid, px..I and raw (n, 7)."""
    m = parse_map_blob(model) if isinstance(model, (bytes, bytearray)) else model
    if m.get("plane_z") is not None and abs(float(rays["plane_z"]) - m["plane_z"]) > 1e-6 * (1 + abs(m["plane_z"])):
        raise ValueError(f"rays on plane z = {rays['plane_z']} but the map was trained on z = {m['plane_z']}")
    ncl, cd, cW, cB = _head_arrays(m["classifier"])
    nrl, rd, rW, rB = _head_arrays(m["regressor"])
    norm = np.ascontiguousarray(m["norm"])
    ox, oy, dx, dy, lam = (_f64(rays, k) for k in ("ox", "oy", "dx", "dy", "lambda_nm"))
    dz = _dz(rays, 1.0)            # not used by O10 (the canonical input is (r, w'_x, w'_y, lambda))
    n = ox.size
    valid = np.zeros(n, np.uint8)
    out = np.zeros((n, 6), np.float64)
    raw = np.zeros((n, 7), np.float64)
    p = _lib.ptr
    lib = _lib.lib()

    def run(lo, hi):
        if hi <= lo:
            return
        lib.orc_map_eval(ncl, p(cd), p(cW), p(cB), nrl, p(rd), p(rW), p(rB), p(norm), hi - lo,
                         p(ox[lo:]), p(oy[lo:]), p(dx[lo:]), p(dy[lo:]), p(dz[lo:]), p(lam[lo:]),
                         p(valid[lo:]), p(out[lo:]), p(raw[lo:]))

    _parallel(run, n, threads)
    return {"valid": valid.astype(bool), "px": out[:, 0].copy(), "py": out[:, 1].copy(),
            "dx": out[:, 2].copy(), "dy": out[:, 3].copy(), "dz": out[:, 4].copy(),
            "I": out[:, 5].copy(), "raw": raw}


def splat(film: dict, valid, px, py, dz, I, channel=None, scale: float = 1.0):
    """O11 int64 fixed-point film (C, H, W); returns (film, dropped)."""
    Wd, Ht, Ch = film["width_px"], film["height_px"], film["channels"]
    f = np.zeros((Ch, Ht, Wd), np.int64)
    v = np.ascontiguousarray(valid, dtype=np.uint8)
    arrs = [np.ascontiguousarray(a, dtype=np.float32) for a in (px, py, dz, I)]
    ch = None if channel is None else np.ascontiguousarray(channel, dtype=np.uint8)
    p = _lib.ptr
    dropped = _lib.lib().orc_splat(Wd, Ht, Ch, film["sensor_w_mm"], film["sensor_h_mm"],
                                   film["center_x_mm"], film["center_y_mm"], p(f), v.size, p(v),
                                   p(arrs[0]), p(arrs[1]), p(arrs[2]), p(arrs[3]), p(ch),
                                   np.float32(scale))
    return f, int(dropped)


def shade_plane(scene: dict, z_hits: float, valid, px, py, dx, dy, dz, I, spp: int, pixels: int,
                scale: float = 1.0, in_dz=None):
    """O14 (Eq. 9): backward camera integrand on a
    checkerboard scene plane -> int64 film of `pixels` (film[i // spp]).  in_dz (optional,
    the sensor rays' w_z): weight each ray by cos^4(theta), the pupil-sampling estimator
    weight (include/plt.h plt_shade_plane_weighted)."""
    f = np.zeros(int(pixels), np.int64)
    v = np.ascontiguousarray(valid, dtype=np.uint8)
    a = [np.ascontiguousarray(x, dtype=np.float32) for x in (px, py, dx, dy, dz, I)]
    w = None if in_dz is None else np.ascontiguousarray(in_dz, dtype=np.float32)
    p = _lib.ptr
    _lib.lib().orc_shade_plane(float(scene["z_mm"]), float(scene["period_mm"]), float(scene["contrast"]),
                               float(z_hits), int(spp), int(pixels), np.float32(scale), p(f), v.size, p(v),
                               *[p(x) for x in a], p(w) if w is not None else None)
    return f


def shade_cards(cards: list, background: float, z_hits: float, valid, px, py, dx, dy, dz, I, spp: int, pixels: int,
                scale: float = 1.0, in_dz=None):
    """O14b: several checkerboard cards (dicts z_mm, period_mm, contrast, x0_mm, x1_mm,
    y0_mm, y1_mm); each valid ray takes the first card it meets inside its rectangle,
    else `background` (include/plt.h plt_shade_cards)."""
    f = np.zeros(int(pixels), np.int64)
    v = np.ascontiguousarray(valid, dtype=np.uint8)
    a = [np.ascontiguousarray(x, dtype=np.float32) for x in (px, py, dx, dy, dz, I)]
    w = None if in_dz is None else np.ascontiguousarray(in_dz, dtype=np.float32)
    cd = np.ascontiguousarray([[c["z_mm"], c["period_mm"], c["contrast"], c["x0_mm"], c["x1_mm"], c["y0_mm"],
                                c["y1_mm"]] for c in cards], dtype=np.float64)
    p = _lib.ptr
    _lib.lib().orc_shade_cards(p(cd), len(cards), float(background), float(z_hits), int(spp), int(pixels),
                               np.float32(scale), p(f), v.size, p(v), *[p(x) for x in a],
                               p(w) if w is not None else None)
    return f


def propagate(rays: dict, z_target: float, direction: int = FORWARD) -> dict:
    """Free-space propagation to z = z_target in float64 (closed form o + ((z_t - z_0)/w_z) w),
    along the ray's line in either sense.  Absent dz: omega in S^2_+  with the sign of
    the query direction (+ forward, - backward), the rule of the trace (A32)."""
    dz = _dz(rays, 1.0 if direction == FORWARD else -1.0)
    t = (float(z_target) - float(rays["plane_z"])) / dz
    out = {k: np.asarray(rays[k], np.float64).copy() for k in ("dx", "dy", "lambda_nm")}
    out["dz"] = dz.copy()
    out["ox"] = np.asarray(rays["ox"], np.float64) + t * out["dx"]
    out["oy"] = np.asarray(rays["oy"], np.float64) + t * out["dy"]
    out["plane_z"] = float(z_target)
    return out


def host_threads() -> int:
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
