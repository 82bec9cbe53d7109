"""Seeded synthetic ray batches and map blobs (SURVEY.md §8(d) input recipe).

INPUT GENERATION ONLY.  Nothing here evaluates the method (no intersection,
refraction, Fresnel, network or canonicalisation arithmetic).  Both the
float64 oracle and the CUDA path consume exactly the float32 arrays produced
here; the oracle widens them to double.

Rays are produced in fixed chunks of ``CHUNK`` rays; chunk ``c`` of a config
draws from ``numpy.random.default_rng([seed, c])``, so any contiguous,
chunk-aligned shard of the global index range is reproduced bit-identically
no matter how many ranks split the job.
"""
from __future__ import annotations

import math
import struct

import numpy as np

CHUNK = 1 << 20

# Fraunhofer lines (nm) used by C1 and the RGB flare channels (§8(c) A21)
LAMBDA_F, LAMBDA_D, LAMBDA_C = 486.1327, 587.5618, 656.2725
FLARE_CHANNELS_NM = (610.0, 550.0, 465.0)


def _uniform_disc(rng, n, radius):
    r = radius * np.sqrt(rng.random(n))
    phi = 2.0 * math.pi * rng.random(n)
    return r * np.cos(phi), r * np.sin(phi)


def _uniform_cap(rng, n, half_angle_deg):
    cmin = math.cos(math.radians(half_angle_deg))
    cz = 1.0 - rng.random(n) * (1.0 - cmin)
    sz = np.sqrt(np.maximum(0.0, 1.0 - cz * cz))
    phi = 2.0 * math.pi * rng.random(n)
    return sz * np.cos(phi), sz * np.sin(phi), cz


def _f32(*arrs):
    return [np.ascontiguousarray(a, dtype=np.float32) for a in arrs]


def _chunk_rng(seed: int, c: int):
    return np.random.default_rng([int(seed), int(c)])


def gen_chunk(law: dict, seed: int, c: int, count: int = CHUNK) -> dict:
    """Generate chunk ``c`` (``count`` rays, normally CHUNK) of a ray law.

    Laws (keys of ``law``):
      kind="disc_cap": origin uniform on a disc of radius ``disc_r`` centred at
        (``disc_x0``, 0) on plane ``plane_z``; direction uniform on a cap of
        ``cap_deg`` about +z; lambda uniform in ``lam`` (nm) or constant.
      kind="collimated": origin as disc_cap, direction fixed at ``angle_deg``
        in the x-z plane.
      kind="sensor_pupil" (backward camera): origin uniform on the sensor
        rectangle ``sensor_w`` x ``sensor_h`` at ``plane_z``; direction towards
        a point uniform on the disc of radius ``pupil_r`` at ``pupil_z``
        (normalised), pointing to -z.
      kind="sensor_grid": as sensor_pupil, but stratified by pixel: global ray i
        starts in pixel i // ``spp`` of a ``width_px`` x ``height_px`` sensor grid
        (row-major, row 0 at +y).
    """
    rng = _chunk_rng(seed, c)
    kind = law["kind"]
    if kind in ("disc_cap", "collimated"):
        ox, oy = _uniform_disc(rng, count, law["disc_r"])
        ox = ox + law.get("disc_x0", 0.0)
        if kind == "disc_cap":
            dx, dy, dz = _uniform_cap(rng, count, law["cap_deg"])
        else:
            a = math.radians(law["angle_deg"])
            dx = np.full(count, math.sin(a))
            dy = np.zeros(count)
            dz = np.full(count, math.cos(a))
    elif kind == "sensor_pupil":
        ox = (rng.random(count) - 0.5) * law["sensor_w"]
        oy = (rng.random(count) - 0.5) * law["sensor_h"]
        px, py = _uniform_disc(rng, count, law["pupil_r"])
        vz = law["pupil_z"] - law["plane_z"]
        vx, vy = px - ox, py - oy
        inv = 1.0 / np.sqrt(vx * vx + vy * vy + vz * vz)
        dx, dy, dz = vx * inv, vy * inv, np.full(count, vz) * inv
    elif kind == "sensor_grid":
        # pixel-stratified backward camera rays: global ray i belongs to pixel i // spp
        # (row-major, row 0 at +y), origin uniform within that pixel, direction towards a
        # point uniform on the rear pupil disc (as sensor_pupil)
        W, H, spp = law["width_px"], law["height_px"], law["spp"]
        gi = c * CHUNK + np.arange(count, dtype=np.int64)
        pix = gi // spp
        ix, iy = pix % W, pix // W
        ox = -0.5 * law["sensor_w"] + (ix + rng.random(count)) * (law["sensor_w"] / W)
        oy = 0.5 * law["sensor_h"] - (iy + rng.random(count)) * (law["sensor_h"] / H)
        px, py = _uniform_disc(rng, count, law["pupil_r"])
        vz = law["pupil_z"] - law["plane_z"]
        vx, vy = px - ox, py - oy
        inv = 1.0 / np.sqrt(vx * vx + vy * vy + vz * vz)
        dx, dy, dz = vx * inv, vy * inv, np.full(count, vz) * inv
    else:
        raise ValueError(f"unknown ray law {kind!r}")
    lam = law["lam"]
    if isinstance(lam, (tuple, list)):
        lam_arr = lam[0] + (lam[1] - lam[0]) * rng.random(count)
    else:
        lam_arr = np.full(count, float(lam))
    ox, oy, dx, dy, dz, lam_arr = _f32(ox, oy, dx, dy, dz, lam_arr)
    return {"ox": ox, "oy": oy, "dx": dx, "dy": dy, "dz": dz, "lambda_nm": lam_arr,
            "plane_z": float(law["plane_z"])}


def gen_rays(law: dict, seed: int, start: int, count: int) -> dict:
    """Rays [start, start+count) of the global index range (chunk-aligned generation).
    Laws with rng="philox" use the counter-based generator of plt_inputs/philox.py (the
    one plt_gen_rays implements on the device) instead of numpy chunks."""
    if law.get("rng") == "philox":
        from . import philox
        return philox.gen_rays(law, seed, start, max(0, count))
    if count <= 0:
        e = np.zeros(0, np.float32)
        return {k: e.copy() for k in ("ox", "oy", "dx", "dy", "dz", "lambda_nm")} | {"plane_z": float(law["plane_z"])}
    c0, c1 = start // CHUNK, (start + count - 1) // CHUNK
    parts = []
    for c in range(c0, c1 + 1):
        ch = gen_chunk(law, seed, c)
        lo = max(start, c * CHUNK) - c * CHUNK
        hi = min(start + count, (c + 1) * CHUNK) - c * CHUNK
        parts.append({k: v[lo:hi] for k, v in ch.items() if k != "plane_z"})
    out = {k: np.ascontiguousarray(np.concatenate([p[k] for p in parts])) for k in parts[0]}
    out["plane_z"] = float(law["plane_z"])
    return out


def sample_indices(n_total: int, n_sample: int, seed: int) -> np.ndarray:
    """Sorted, distinct, seeded sample of ray indices across [0, n_total)."""
    rng = np.random.default_rng([int(seed), 0x5A3])
    if n_sample >= n_total:
        return np.arange(n_total, dtype=np.int64)
    return np.sort(rng.choice(n_total, size=n_sample, replace=False)).astype(np.int64)


def gen_rays_at(law: dict, seed: int, idx: np.ndarray) -> dict:
    """Rays at arbitrary global indices (regenerates the chunks that contain them)."""
    if law.get("rng") == "philox":
        from . import philox
        return philox.rays_at(law, seed, idx)
    idx = np.asarray(idx, dtype=np.int64)
    out = {k: np.empty(idx.size, np.float32) for k in ("ox", "oy", "dx", "dy", "dz", "lambda_nm")}
    chunks = idx // CHUNK
    for c in np.unique(chunks):
        sel = np.nonzero(chunks == c)[0]
        ch = gen_chunk(law, seed, int(c))
        loc = idx[sel] - int(c) * CHUNK
        for k in out:
            out[k][sel] = ch[k][loc]
    out["plane_z"] = float(law["plane_z"])
    return out


# ----------------------------------------------------------------------------
# Map blobs: seeded Xavier-uniform weights stored as bf16 (SURVEY.md §8(d) "Weights")
# ----------------------------------------------------------------------------
MAP_MAGIC = b"PLTMAP01"
CLASSIFIER_DIMS = (4, 32, 32, 1)               # PAPER.md:391-392 (2 hidden layers of 32)
REGRESSOR_DIMS = (4, 32, 32, 32, 32, 32, 6)    # PAPER.md:391-392 (5 hidden layers of 32)


def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """Round float32 to bfloat16 (round-to-nearest-even); returns the uint16 bit patterns."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) >> 16
    return u.astype(np.uint16)


def _header(path_id: int, direction: int, ncl: int, nrl: int, plane_z) -> list:
    """Magic + header; version 2 (with the f64 input plane z) when plane_z is given."""
    if plane_z is None:
        return [MAP_MAGIC, struct.pack("<IIQII", 1, int(direction), int(path_id), ncl, nrl)]
    return [MAP_MAGIC, struct.pack("<IIQII", 2, int(direction), int(path_id), ncl, nrl),
            struct.pack("<d", float(plane_z))]


def write_map_blob(path_id: int, direction: int, in_lo, in_hi, out_mid, out_half, cls_layers, reg_layers,
                   plane_z=None) -> bytes:
    """Serialise a factorised map from given layers [(W float32 (out, in), b float32 (out,)), ...];
    W is rounded to bf16 (round-to-nearest-even).  Same layout as make_map_blob; plane_z (the
    input plane of the training rays) makes a version-2 blob."""
    parts = _header(path_id, direction, len(cls_layers), len(reg_layers), plane_z)
    for arr, n in ((in_lo, 4), (in_hi, 4), (out_mid, 6), (out_half, 6)):
        a = np.asarray(arr, dtype=np.float32)
        assert a.shape == (n,)
        parts.append(a.tobytes())
    for layers in (cls_layers, reg_layers):
        for W, b in layers:
            W = np.asarray(W, dtype=np.float32)
            b = np.asarray(b, dtype=np.float32)
            parts.append(struct.pack("<II", W.shape[0], W.shape[1]))
            parts.append(f32_to_bf16_bits(W).tobytes())
            parts.append(b.tobytes())
    return b"".join(parts)


def make_map_blob(path_id: int, direction: int, seed: int, in_lo, in_hi, out_mid, out_half,
                  bias_range: float = 0.1, plane_z=None) -> bytes:
    """Serialise one path's factorised map (classifier + regressor) as a blob.

    Layout (little-endian): magic 'PLTMAP01'; u32 version (1, or 2 with plane_z); u32
    direction; u64 path_id; u32 n_cls_layers; u32 n_reg_layers; [v2: f64 plane_z_mm, the
    input plane the map was trained on]; f32 in_lo[4], in_hi[4],
    out_mid[6], out_half[6]; then for every layer (classifier first, then
    regressor): u32 out, u32 in, u16 W_bf16[out*in] (row-major, W[o][i]),
    f32 b[out].  Weights: Xavier-uniform gain 1, biases U(-bias_range, bias_range).
    """
    rng = np.random.default_rng([int(seed), int(path_id) & 0xFFFFFFFF, int(path_id) >> 32, 0xB10B])
    parts = _header(path_id, direction, len(CLASSIFIER_DIMS) - 1, len(REGRESSOR_DIMS) - 1, plane_z)
    for arr, n in ((in_lo, 4), (in_hi, 4), (out_mid, 6), (out_half, 6)):
        a = np.asarray(arr, dtype=np.float32)
        assert a.shape == (n,)
        parts.append(a.tobytes())
    for dims in (CLASSIFIER_DIMS, REGRESSOR_DIMS):
        for fi, fo in zip(dims[:-1], dims[1:]):
            lim = math.sqrt(6.0 / (fi + fo))
            w = rng.uniform(-lim, lim, size=(fo, fi)).astype(np.float32)
            b = rng.uniform(-bias_range, bias_range, size=fo).astype(np.float32)
            parts.append(struct.pack("<II", fo, fi))
            parts.append(f32_to_bf16_bits(w).tobytes())
            parts.append(b.tobytes())
    return b"".join(parts)
