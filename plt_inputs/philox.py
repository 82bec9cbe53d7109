"""Counter-based synthetic rays: Philox4x32-10 keyed by (seed, global ray index).

INPUT GENERATION ONLY (no method arithmetic).  This is the numpy implementation of the
generator the library also implements on the device (``plt_gen_rays``,
paper_2605_04017_b200/csrc/gen_rays.cu): the two share no code, they implement the same
specification, below, and produce bit-identical float32 rays -- so a test can draw a
sample of a full-size device batch (C3: 805 M rays, C5: 2^30) anywhere in the index range
and hand the oracle exactly the rays the GPU traced, without any oracle input coming from
the CUDA path.

Specification (every step is IEEE double with one rounding per operation, no fused
multiply-add; float32 outputs rounded to nearest):

* Philox4x32-10 (Salmon et al., SC'11): round constants M0 = 0xD2511F53, M1 = 0xCD9E8D57,
  Weyl increments W0 = 0x9E3779B9, W1 = 0xBB67AE85; a round maps (c0, c1, c2, c3) with key
  (k0, k1) to (hi(M1 c2) ^ c1 ^ k0, lo(M1 c2), hi(M0 c0) ^ c3 ^ k1, lo(M0 c0)), then the key
  is bumped by (W0, W1); ten rounds, the key bump after each of the first nine.
* Ray i (global index), block b in {0, 1}: counter (i mod 2^32, i div 2^32, b, 0x504C5452),
  key (seed mod 2^32, seed div 2^32) -> 8 words x0..x7; u_k = (x_k + 0.5) * 2^-32.
* angle(u) -> (cos 2 pi u, sin 2 pi u): t = 8u, k = floor(t), theta = (t - k - 0.5) * PI_4;
  sin/cos of theta by the Taylor polynomials below (Horner, fixed order), rotated by the
  octant centre (k + 1/2) pi/4 from the table CS.
* Laws (same fields as plt_inputs.rays; derived constants computed by the caller):
  disc_cap   : r = R sqrt(u0), (c, s) = angle(u1), o = (x0 + r c, r s);
               w_z = 1 - u2 (1 - cmin), s_z = sqrt(max(0, 1 - w_z^2)), (c', s') = angle(u3),
               w = (s_z c', s_z s', w_z); lambda = lo + (hi - lo) u4
  collimated : o as disc_cap; w = (dir_x, 0, dir_z); lambda = lo + (hi - lo) u4
  sensor_pupil: o = ((u0 - 0.5) W, (u1 - 0.5) H); pupil point q = Rp sqrt(u2) angle(u3);
               v = (q_x - o_x, q_y - o_y, z_p - z_0), w = v / sqrt(|v|^2); lambda from u4
  sensor_grid: pixel p = i div spp, (ix, iy) = (p mod Wpx, p div Wpx);
               o = (-W/2 + (ix + u0)(W / Wpx), H/2 - (iy + u1)(H / Hpx)); w, lambda as sensor_pupil
"""
from __future__ import annotations

import math

import numpy as np

M0, M1 = 0xD2511F53, 0xCD9E8D57
W0, W1 = 0x9E3779B9, 0xBB67AE85
TAG = 0x504C5452
MASK = 0xFFFFFFFF
INV32 = 2.0 ** -32
PI_4 = 0.78539816339744830962
# Taylor coefficients of sin and cos (|theta| <= pi/8: truncation < 1e-19)
S3, S5, S7, S9, S11, S13 = (-0.16666666666666666667, 0.0083333333333333333333, -0.00019841269841269841270,
                            2.7557319223985890653e-06, -2.5052108385441718775e-08, 1.6059043836821614599e-10)
C2, C4, C6, C8, C10, C12, C14 = (-0.5, 0.041666666666666666667, -0.0013888888888888888889,
                                 2.4801587301587301587e-05, -2.7557319223985890653e-07,
                                 2.0876756987868098979e-09, -1.1470745597729724714e-11)
_A, _B = 0.92387953251128673848, 0.38268343236508978178   # cos / sin of pi/8
# (cos, sin) of the octant centres (k + 1/2) pi / 4, k = 0..7
CS = ((_A, _B), (_B, _A), (-_B, _A), (-_A, _B), (-_A, -_B), (-_B, -_A), (_B, -_A), (_A, -_B))
_CK = np.array([c for c, _ in CS])
_SK = np.array([s for _, s in CS])


def philox4x32_10(c0, c1, c2, c3, k0, k1):
    """Vectorised Philox4x32-10 on uint64 arrays holding 32-bit values."""
    c0, c1, c2, c3 = (np.asarray(v, np.uint64) for v in (c0, c1, c2, c3))
    k0 = np.uint64(k0 & MASK)
    k1 = np.uint64(k1 & MASK)
    m0, m1, msk = np.uint64(M0), np.uint64(M1), np.uint64(MASK)
    for r in range(10):
        p0 = m0 * c0
        p1 = m1 * c2
        hi0, lo0 = p0 >> np.uint64(32), p0 & msk
        hi1, lo1 = p1 >> np.uint64(32), p1 & msk
        c0, c1, c2, c3 = hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0
        if r < 9:
            k0 = np.uint64((int(k0) + W0) & MASK)
            k1 = np.uint64((int(k1) + W1) & MASK)
    return c0, c1, c2, c3


def uniforms(seed: int, idx: np.ndarray) -> np.ndarray:
    """(8, n) doubles u_k = (x_k + 0.5) 2^-32 for global ray indices idx."""
    idx = np.asarray(idx, np.uint64)
    lo, hi = idx & np.uint64(MASK), idx >> np.uint64(32)
    out = np.empty((8, idx.size), np.float64)
    for b in (0, 1):
        x = philox4x32_10(lo, hi, np.full(idx.size, b, np.uint64), np.full(idx.size, TAG, np.uint64),
                          int(seed) & MASK, (int(seed) >> 32) & MASK)
        for j in range(4):
            out[4 * b + j] = (x[j].astype(np.float64) + 0.5) * INV32
    return out


def angle(u: np.ndarray):
    """(cos 2 pi u, sin 2 pi u) by the specification's octant reduction + polynomials."""
    t = u * 8.0
    k = np.floor(t)
    th = ((t - k) - 0.5) * PI_4
    t2 = th * th
    ps = S13
    for c in (S11, S9, S7, S5, S3):
        ps = ps * t2 + c
    s = th + (th * t2) * ps
    pc = C14
    for c in (C12, C10, C8, C6, C4, C2):
        pc = pc * t2 + c
    c = 1.0 + t2 * pc
    ki = k.astype(np.int64)
    ck, sk = _CK[ki], _SK[ki]
    return c * ck - s * sk, s * ck + c * sk


def law_constants(law: dict) -> dict:
    """Derived doubles of a ray law, computed once by the caller and handed to both
    generators (the device generator receives these same values through plt_ray_law)."""
    kind = law["kind"]
    lam = law["lam"]
    lo, hi = (float(lam[0]), float(lam[1])) if isinstance(lam, (tuple, list)) else (float(lam), float(lam))
    k = {"kind": kind, "plane_z": float(law["plane_z"]), "lam_lo": lo, "lam_hi": hi}
    if kind in ("disc_cap", "collimated"):
        k.update(disc_r=float(law["disc_r"]), disc_x0=float(law.get("disc_x0", 0.0)))
        if kind == "disc_cap":
            k["cap_cos_min"] = math.cos(math.radians(law["cap_deg"]))
        else:
            a = math.radians(law["angle_deg"])
            k.update(dir_x=math.sin(a), dir_z=math.cos(a))
    elif kind in ("sensor_pupil", "sensor_grid"):
        k.update(sensor_w=float(law["sensor_w"]), sensor_h=float(law["sensor_h"]), pupil_z=float(law["pupil_z"]),
                 pupil_r=float(law["pupil_r"]))
        if kind == "sensor_grid":
            k.update(width_px=int(law["width_px"]), height_px=int(law["height_px"]), spp=int(law["spp"]))
    else:
        raise ValueError(f"unknown ray law {kind!r}")
    return k


def rays_at(law: dict, seed: int, idx) -> dict:
    """float32 rays at global indices idx (any order, any subset of the index range)."""
    K = law_constants(law)
    idx = np.asarray(idx, np.int64)
    u = uniforms(seed, idx)
    kind = K["kind"]
    if kind in ("disc_cap", "collimated"):
        r = K["disc_r"] * np.sqrt(u[0])
        c, s = angle(u[1])
        ox, oy = K["disc_x0"] + r * c, r * s
        if kind == "disc_cap":
            wz = 1.0 - u[2] * (1.0 - K["cap_cos_min"])
            sz = np.sqrt(np.maximum(0.0, 1.0 - wz * wz))
            c2, s2 = angle(u[3])
            dx, dy, dz = sz * c2, sz * s2, wz
        else:
            dx = np.full(idx.size, K["dir_x"])
            dy = np.zeros(idx.size)
            dz = np.full(idx.size, K["dir_z"])
    else:
        W, H = K["sensor_w"], K["sensor_h"]
        if kind == "sensor_pupil":
            ox = (u[0] - 0.5) * W
            oy = (u[1] - 0.5) * H
        else:
            pix = idx // K["spp"]
            ix = (pix % K["width_px"]).astype(np.float64)
            iy = (pix // K["width_px"]).astype(np.float64)
            ox = (-0.5 * W) + (ix + u[0]) * (W / K["width_px"])
            oy = (0.5 * H) - (iy + u[1]) * (H / K["height_px"])
        r = K["pupil_r"] * np.sqrt(u[2])
        c, s = angle(u[3])
        vx, vy, vz = r * c - ox, r * s - oy, K["pupil_z"] - K["plane_z"]
        inv = 1.0 / np.sqrt((vx * vx + vy * vy) + vz * vz)
        dx, dy, dz = vx * inv, vy * inv, vz * inv
    lam = K["lam_lo"] + (K["lam_hi"] - K["lam_lo"]) * u[4]
    f = lambda a: np.ascontiguousarray(np.broadcast_to(a, idx.shape), dtype=np.float32)
    return {"ox": f(ox), "oy": f(oy), "dx": f(dx), "dy": f(dy), "dz": f(dz), "lambda_nm": f(lam),
            "plane_z": K["plane_z"]}


def gen_rays(law: dict, seed: int, start: int, count: int) -> dict:
    """Rays [start, start + count) of the global index range."""
    return rays_at(law, seed, np.arange(int(start), int(start) + int(count), dtype=np.int64))
