"""Python binding of libplt.so -- the B200 (sm_100a) lens-transport query library.

Argument marshalling only: every step of the query runs in the library's CUDA
kernels (``include/plt.h``).  PyTorch supplies device memory, streams and (in
``bench.py``) process groups.  There is no CPU fallback: importing works on a
CPU-only box, but every compute call requires the built ``libplt.so`` and an
sm_100a device and raises otherwise.

Names follow the ABI: ``Lens`` (plt_lens_load / info / enumerate_ghosts),
``Map`` (plt_map_load), ``trace_rays``, ``eval_map``, ``splat_sensor``,
``film_resolve``.
"""
from __future__ import annotations

import ctypes as C
import math
import os

__all__ = ["load", "PltError", "Lens", "Map", "trace_rays", "trace_paths", "eval_map", "splat_sensor", "film_resolve",
           "alloc_hits", "rays_to_device", "FORWARD", "BACKWARD", "FP32", "FP64", "LIB_PATH"]

LIB_PATH = os.environ.get("PLT_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libplt.so")
FORWARD, BACKWARD = 0, 1
FP32, FP64 = 0, 1

_STATUS = {0: "PLT_OK", 1: "PLT_E_INVALID_ARG", 2: "PLT_E_PARSE", 3: "PLT_E_VALIDATION",
           4: "PLT_E_CAPACITY", 5: "PLT_E_UNSUPPORTED", 6: "PLT_E_CUDA", 7: "PLT_E_OOM"}

EXPORTED = ("plt_last_error", "plt_version", "plt_lens_load", "plt_lens_free", "plt_lens_info",
            "plt_enumerate_ghosts", "plt_trace_rays", "plt_map_load", "plt_map_free", "plt_eval_map",
            "plt_splat_sensor", "plt_film_resolve", "plt_trace_rays_splat", "plt_eval_map_splat",
            "plt_trace_jit_cubin", "plt_shade_plane", "plt_shade_plane_weighted", "plt_shade_cards",
            "plt_propagate_rays", "plt_lens_pupils", "plt_trace_kernel", "plt_gen_rays", "plt_query_host",
            "plt_pupil_weight", "plt_trace_paths")


class PltError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{_STATUS.get(status, status)}: {msg}")
        self.status = status


class LensOpts(C.Structure):
    _fields_ = [("input_plane_z_mm", C.c_double), ("sensor_z_mm", C.c_double), ("sensor_w_mm", C.c_double),
                ("sensor_h_mm", C.c_double), ("backward_exit_z_mm", C.c_double),
                ("housing_radius_mm", C.c_double), ("lambda_ref_nm", C.c_double)]


class Rays(C.Structure):
    _fields_ = [("ox", C.c_void_p), ("oy", C.c_void_p), ("dx", C.c_void_p), ("dy", C.c_void_p),
                ("dz", C.c_void_p), ("lambda_nm", C.c_void_p), ("plane_z_mm", C.c_double)]


class Hits(C.Structure):
    _fields_ = [("mask_bits", C.c_void_p), ("px", C.c_void_p), ("py", C.c_void_p), ("dx", C.c_void_p),
                ("dy", C.c_void_p), ("dz", C.c_void_p), ("throughput", C.c_void_p), ("flags", C.c_void_p)]


class FilmDesc(C.Structure):
    _fields_ = [("width_px", C.c_int), ("height_px", C.c_int), ("channels", C.c_int),
                ("sensor_w_mm", C.c_double), ("sensor_h_mm", C.c_double),
                ("center_x_mm", C.c_double), ("center_y_mm", C.c_double)]


class ScenePlane(C.Structure):
    _fields_ = [("z_mm", C.c_double), ("period_mm", C.c_double), ("contrast", C.c_double)]


class RayLaw(C.Structure):
    _fields_ = [("kind", C.c_int), ("width_px", C.c_int), ("height_px", C.c_int), ("spp", C.c_int),
                ("plane_z_mm", C.c_double), ("disc_r_mm", C.c_double), ("disc_x0_mm", C.c_double),
                ("cap_cos_min", C.c_double), ("dir_x", C.c_double), ("dir_z", C.c_double),
                ("sensor_w_mm", C.c_double), ("sensor_h_mm", C.c_double), ("pupil_z_mm", C.c_double),
                ("pupil_r_mm", C.c_double), ("lambda_lo_nm", C.c_double), ("lambda_hi_nm", C.c_double)]


LAW_KINDS = {"disc_cap": 0, "collimated": 1, "sensor_pupil": 2, "sensor_grid": 3}


class SplatTarget(C.Structure):
    _fields_ = [("film_desc", C.c_void_p), ("film", C.c_void_p), ("channel", C.c_void_p),
                ("weight_scale", C.c_float), ("dropped", C.c_void_p)]


_lib = None


def load():
    """Load libplt.so (raises if it has not been built -- there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: run `python -m paper_2605_04017_b200.build` "
                           "(the CUDA extension is required; there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    p, i, i64, u64, d, st = C.c_void_p, C.c_int, C.c_int64, C.c_uint64, C.c_double, C.c_int
    L.plt_last_error.restype = C.c_char_p
    L.plt_version.restype = C.c_char_p
    L.plt_lens_load.argtypes = [C.c_char_p, C.c_size_t, p, C.POINTER(p)]
    L.plt_lens_free.argtypes = [p]
    L.plt_lens_free.restype = None
    L.plt_lens_info.argtypes = [p, d, p, p, p, p, p, p]
    L.plt_enumerate_ghosts.argtypes = [p, i, d, p, p, i, p]
    L.plt_trace_rays.argtypes = [p, u64, i, i, p, p, i64, p]
    L.plt_map_load.argtypes = [p, C.c_char_p, C.c_size_t, C.POINTER(p)]
    L.plt_map_free.argtypes = [p]
    L.plt_map_free.restype = None
    L.plt_eval_map.argtypes = [p, p, p, p, i64, p]
    L.plt_splat_sensor.argtypes = [p, p, p, p, C.c_float, i64, p, p]
    L.plt_film_resolve.argtypes = [p, p, p, d, p]
    L.plt_trace_rays_splat.argtypes = [p, u64, i, i, p, p, p, i64, p]
    L.plt_eval_map_splat.argtypes = [p, p, p, p, p, i64, p]
    L.plt_trace_jit_cubin.argtypes = [p, u64, i, p, C.c_size_t, C.POINTER(C.c_size_t)]
    L.plt_shade_plane.argtypes = [p, d, p, i, i64, C.c_float, p, i64, p]
    L.plt_shade_plane_weighted.argtypes = [p, d, p, i, i64, C.c_float, p, p, i64, p]
    L.plt_shade_cards.argtypes = [p, i, d, d, p, i, i64, C.c_float, p, p, i64, p]
    L.plt_propagate_rays.argtypes = [p, p, d, i, i64, p]
    L.plt_trace_kernel.argtypes = [p, u64, i, i, p]
    L.plt_gen_rays.argtypes = [p, u64, i64, p, i64, p]
    L.plt_query_host.argtypes = [p, u64, i, i, p, p, p, p, p, p, i64, i64, p]
    L.plt_pupil_weight.argtypes = [d, d, d, p]
    L.plt_lens_pupils.argtypes = [p, d, p, p, p, p]
    L.plt_trace_paths.argtypes = [p, p, i, i, i, p, p, p, i64, p]
    for f in ("plt_lens_load", "plt_lens_info", "plt_enumerate_ghosts", "plt_trace_rays", "plt_map_load",
              "plt_eval_map", "plt_splat_sensor", "plt_film_resolve", "plt_trace_rays_splat",
              "plt_eval_map_splat", "plt_trace_jit_cubin", "plt_shade_plane", "plt_shade_plane_weighted",
              "plt_shade_cards", "plt_propagate_rays", "plt_lens_pupils", "plt_trace_kernel", "plt_gen_rays",
              "plt_query_host", "plt_pupil_weight", "plt_trace_paths"):
        getattr(L, f).restype = st
    _lib = L
    return L


def _check(status: int):
    if status != 0:
        raise PltError(status, load().plt_last_error().decode(errors="replace"))


def version() -> str:
    return load().plt_version().decode()


class Lens:
    """plt_lens_load: parse + validate a prescription (.lens table or JSON)."""

    def __init__(self, text: str, **opts):
        o = LensOpts(input_plane_z_mm=opts.get("input_plane_z_mm", -5.0),
                     sensor_z_mm=opts.get("sensor_z_mm", float("nan")),
                     sensor_w_mm=opts.get("sensor_w_mm", 0.0), sensor_h_mm=opts.get("sensor_h_mm", 0.0),
                     backward_exit_z_mm=opts.get("backward_exit_z_mm", -5.0),
                     housing_radius_mm=opts.get("housing_radius_mm", 0.0),
                     lambda_ref_nm=opts.get("lambda_ref_nm", 587.5618))
        raw = text.encode()
        h = C.c_void_p()
        self._h = None
        _check(load().plt_lens_load(raw, len(raw), C.byref(o), C.byref(h)))
        self._h = h

    @property
    def handle(self):
        return self._h

    def info(self, lambda_nm: float = 587.5618) -> dict:
        n_opt, stop = C.c_int(), C.c_int()
        abcd = (C.c_double * 4)()
        efl, bfl, sz = C.c_double(), C.c_double(), C.c_double()
        _check(load().plt_lens_info(self._h, lambda_nm, C.byref(n_opt), C.byref(stop), abcd, C.byref(efl),
                                    C.byref(bfl), C.byref(sz)))
        return {"n_optical": n_opt.value, "stop_index": stop.value, "abcd": list(abcd), "efl_mm": efl.value,
                "bfl_mm": bfl.value, "sensor_z_mm": sz.value}

    def enumerate_ghosts(self, max_bounces: int = 2, min_throughput: float = 0.0):
        L = load()
        cnt = C.c_int()
        st = L.plt_enumerate_ghosts(self._h, max_bounces, min_throughput, None, None, 0, C.byref(cnt))
        if st not in (0, 4):
            _check(st)
        ids = (C.c_uint64 * cnt.value)()
        ij = (C.c_int32 * (2 * cnt.value))()
        _check(L.plt_enumerate_ghosts(self._h, max_bounces, min_throughput, ids, ij, cnt.value, C.byref(cnt)))
        return list(ids), [(ij[2 * k], ij[2 * k + 1]) for k in range(cnt.value)]

    def trace_jit_cubin(self, path_id: int, direction: int = 0) -> bytes:
        """plt_trace_jit_cubin: the sm_100a cubin of the trace kernel specialised for this path."""
        L = load()
        size = C.c_size_t()
        _check(L.plt_trace_jit_cubin(self._h, int(path_id), direction, None, 0, C.byref(size)))
        buf = C.create_string_buffer(size.value)
        _check(L.plt_trace_jit_cubin(self._h, int(path_id), direction, buf, size.value, C.byref(size)))
        return buf.raw[:size.value]

    def pupils(self, lambda_nm: float = 587.5618) -> dict:
        """plt_lens_pupils: paraxial entrance / exit pupil positions and radii (mm)."""
        v = [C.c_double() for _ in range(4)]
        _check(load().plt_lens_pupils(self._h, lambda_nm, *[C.byref(x) for x in v]))
        return {"entrance_z_mm": v[0].value, "entrance_r_mm": v[1].value, "exit_z_mm": v[2].value,
                "exit_r_mm": v[3].value}

    def all_t_id(self) -> int:
        return 1 << self.info()["n_optical"]

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.plt_lens_free(self._h)
            self._h = None


class Map:
    """plt_map_load: one path's factorised network from a PLTMAP01 blob."""

    def __init__(self, blob: bytes, lens: Lens | None = None):
        h = C.c_void_p()
        self._h = None
        _check(load().plt_map_load(lens.handle if lens else None, blob, len(blob), C.byref(h)))
        self._h = h

    @property
    def handle(self):
        return self._h

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.plt_map_free(self._h)
            self._h = None


# ---------------------------------------------------------------- marshalling helpers
RAY_KEYS = ("ox", "oy", "dx", "dy", "dz", "lambda_nm")
HIT_KEYS = ("px", "py", "dx", "dy", "dz", "throughput")


def _ptr(t, n=None, dtype=None):
    import torch
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("plt buffers must be CUDA tensors (no CPU fallback)")
    if not t.is_contiguous():
        raise ValueError("plt buffers must be contiguous")
    if dtype is not None and t.dtype != dtype:
        raise ValueError(f"expected {dtype}, got {t.dtype}")
    if n is not None and t.numel() < n:
        raise ValueError(f"buffer has {t.numel()} elements, need {n}")
    return t.data_ptr()


def _stream(stream):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _rays_struct(rays: dict, n: int) -> Rays:
    """rays["dz"] may be absent or None: directions in S^2_+ given by (dx, dy)."""
    import torch
    f = torch.float32
    return Rays(*(_ptr(rays.get(k) if k == "dz" else rays[k], n, f) for k in RAY_KEYS), float(rays["plane_z"]))


def _hits_struct(hits: dict, n: int) -> Hits:
    import torch
    f = torch.float32
    mask = _ptr(hits["mask_bits"], (n + 31) // 32, torch.int32)
    flags = _ptr(hits.get("flags"), n, torch.uint8) if hits.get("flags") is not None else None
    return Hits(mask, *(_ptr(hits[k], n, f) for k in HIT_KEYS), flags)


def alloc_hits(n: int, device="cuda", flags: bool = False) -> dict:
    import torch
    h = {k: torch.empty(n, dtype=torch.float32, device=device) for k in HIT_KEYS}
    h["mask_bits"] = torch.empty((n + 31) // 32, dtype=torch.int32, device=device)
    h["flags"] = torch.empty(n, dtype=torch.uint8, device=device) if flags else None
    return h


def rays_to_device(rays: dict, device="cuda", pin: bool = False, with_dz: bool = True) -> dict:
    """Copy a dict of float32 numpy arrays (plt_inputs format) to device tensors.
    with_dz=False leaves dz out (None): the kernels complete omega in S^2_+ from (dx, dy)."""
    import numpy as np
    import torch
    out = {}
    for k in RAY_KEYS:
        if k == "dz" and (not with_dz or rays.get("dz") is None):
            out[k] = None
            continue
        t = torch.from_numpy(np.ascontiguousarray(rays[k], dtype=np.float32))
        if pin:
            t = t.pin_memory()
        out[k] = t.to(device, non_blocking=pin)
    out["plane_z"] = float(rays["plane_z"])
    return out


def _n_of(rays, n):
    return int(rays["ox"].numel()) if n is None else int(n)


def _splat_struct(splat: dict, n: int):
    """splat = {"film_desc": dict, "film": int64 tensor, "channel": uint8 tensor | None,
    "weight_scale": float, "dropped": int64 tensor | None} -> (SplatTarget, keep-alive)."""
    import torch
    fd = film_desc(splat["film_desc"])
    npx = fd.channels * fd.height_px * fd.width_px
    ch, dr = splat.get("channel"), splat.get("dropped")
    t = SplatTarget(C.addressof(fd), _ptr(splat["film"], npx, torch.int64),
                    _ptr(ch, n, torch.uint8) if ch is not None else None, float(splat.get("weight_scale", 1.0)),
                    _ptr(dr, 1, torch.int64) if dr is not None else None)
    return t, fd


def trace_rays(lens: Lens, path_id: int, rays: dict, hits: dict, direction: int = FORWARD,
               precision: int = FP32, n: int | None = None, stream=None, splat: dict | None = None):
    """plt_trace_rays (exact sequential trace of one path, Eq. 5-7); with `splat`,
    plt_trace_rays_splat (the valid hits are also splatted into splat["film"] in-kernel)."""
    n = _n_of(rays, n)
    r, h = _rays_struct(rays, n), _hits_struct(hits, n)
    if splat is None:
        _check(load().plt_trace_rays(lens.handle, int(path_id), direction, precision, C.byref(r), C.byref(h), n,
                                     _stream(stream)))
    else:
        t, _keep = _splat_struct(splat, n)
        _check(load().plt_trace_rays_splat(lens.handle, int(path_id), direction, precision, C.byref(r), C.byref(h),
                                           C.byref(t), n, _stream(stream)))


def trace_paths(lens: Lens, path_ids, rays: dict, hits_list, direction: int = FORWARD, precision: int = FP32,
                n: int | None = None, stream=None, splat: dict | None = None):
    """plt_trace_paths: the batch traced along every path of `path_ids` (hits_list[p] gets path
    p's hits) -- the same results as one trace_rays call per path; in float64 the paths'
    common all-T prefix is traced once (include/plt.h)."""
    n = _n_of(rays, n)
    ids = [int(g) for g in path_ids]
    if len(hits_list) != len(ids):
        raise ValueError("need one hits dict per path")
    r = _rays_struct(rays, n)
    outs = (Hits * max(1, len(ids)))(*[_hits_struct(h, n) for h in hits_list])
    arr = (C.c_uint64 * max(1, len(ids)))(*ids)
    t, _keep = _splat_struct(splat, n) if splat is not None else (None, None)
    _check(load().plt_trace_paths(lens.handle, arr, len(ids), direction, precision, C.byref(r), outs,
                                  C.byref(t) if t is not None else None, n, _stream(stream)))


def eval_map(m: Map, rays: dict, hits: dict, raw=None, n: int | None = None, stream=None, splat: dict | None = None):
    """plt_eval_map (fused classifier-gated regressor on tcgen05); with `splat`,
    plt_eval_map_splat (valid outputs also splatted in the regressor epilogue)."""
    import torch
    n = _n_of(rays, n)
    r, h = _rays_struct(rays, n), _hits_struct(hits, n)
    rp = _ptr(raw, 7 * n, torch.float32) if raw is not None else None
    if splat is None:
        _check(load().plt_eval_map(m.handle, C.byref(r), C.byref(h), rp, n, _stream(stream)))
    else:
        t, _keep = _splat_struct(splat, n)
        _check(load().plt_eval_map_splat(m.handle, C.byref(r), C.byref(h), rp, C.byref(t), n, _stream(stream)))


def film_desc(d: dict) -> FilmDesc:
    return FilmDesc(d["width_px"], d["height_px"], d["channels"], d["sensor_w_mm"], d["sensor_h_mm"],
                    d.get("center_x_mm", 0.0), d.get("center_y_mm", 0.0))


def splat_sensor(film_d: dict, film, hits: dict, channel=None, weight_scale: float = 1.0, n: int | None = None,
                 dropped=None, stream=None):
    """plt_splat_sensor (int64 fixed-point film, warp-aggregated atomics)."""
    import torch
    n = int(hits["px"].numel()) if n is None else int(n)
    fd = film_desc(film_d)
    npx = film_d["channels"] * film_d["height_px"] * film_d["width_px"]
    h = _hits_struct(hits, n)
    _check(load().plt_splat_sensor(C.byref(fd), _ptr(film, npx, torch.int64), C.byref(h),
                                   _ptr(channel, n, torch.uint8) if channel is not None else None,
                                   float(weight_scale), n,
                                   _ptr(dropped, 1, torch.int64) if dropped is not None else None,
                                   _stream(stream)))


def shade_plane(scene: dict, z_hits_mm: float, hits: dict, film, spp: int, pixels: int | None = None,
                weight_scale: float = 1.0, n: int | None = None, stream=None, in_dz=None):
    """plt_shade_plane: backward camera integrand on a checkerboard scene plane (Eq. 9);
    with in_dz (the sensor rays' w_z, device float32), plt_shade_plane_weighted (the
    cos^4 pupil-sampling weight)."""
    import torch
    n = int(hits["px"].numel()) if n is None else int(n)
    pixels = int(film.numel()) if pixels is None else int(pixels)
    sc = ScenePlane(float(scene["z_mm"]), float(scene["period_mm"]), float(scene["contrast"]))
    h = _hits_struct(hits, n)
    if in_dz is None:
        _check(load().plt_shade_plane(C.byref(sc), float(z_hits_mm), C.byref(h), int(spp), pixels,
                                      float(weight_scale), _ptr(film, pixels, torch.int64), n, _stream(stream)))
    else:
        _check(load().plt_shade_plane_weighted(C.byref(sc), float(z_hits_mm), C.byref(h), int(spp), pixels,
                                               float(weight_scale), _ptr(in_dz, n, torch.float32),
                                               _ptr(film, pixels, torch.int64), n, _stream(stream)))


class SceneCard(C.Structure):
    _fields_ = [("z_mm", C.c_double), ("period_mm", C.c_double), ("contrast", C.c_double), ("x0_mm", C.c_double),
                ("x1_mm", C.c_double), ("y0_mm", C.c_double), ("y1_mm", C.c_double)]


def shade_cards(cards: list, background: float, z_hits_mm: float, hits: dict, film, spp: int,
                pixels: int | None = None, weight_scale: float = 1.0, n: int | None = None, stream=None, in_dz=None):
    """plt_shade_cards: backward camera integrand on a scene of several checkerboard cards
    (dicts z_mm, period_mm, contrast, x0_mm, x1_mm, y0_mm, y1_mm); in_dz as shade_plane."""
    import torch
    n = int(hits["px"].numel()) if n is None else int(n)
    pixels = int(film.numel()) if pixels is None else int(pixels)
    arr = (SceneCard * len(cards))(*[SceneCard(c["z_mm"], c["period_mm"], c["contrast"], c["x0_mm"], c["x1_mm"],
                                               c["y0_mm"], c["y1_mm"]) for c in cards])
    h = _hits_struct(hits, n)
    _check(load().plt_shade_cards(arr, len(cards), float(background), float(z_hits_mm), C.byref(h), int(spp), pixels,
                                  float(weight_scale), _ptr(in_dz, n, torch.float32) if in_dz is not None else None,
                                  _ptr(film, pixels, torch.int64), n, _stream(stream)))


def propagate_rays(rays: dict, out: dict, z_target_mm: float, direction: int = FORWARD, n: int | None = None,
                   stream=None):
    """plt_propagate_rays: free-space propagation to z = z_target_mm along each ray's line
    (out may alias rays); `direction` gives the sign of w_z for rays without dz."""
    n = _n_of(rays, n)
    r = _rays_struct(rays, n)
    o = _rays_struct(dict(out, plane_z=z_target_mm), n)
    _check(load().plt_propagate_rays(C.byref(r), C.byref(o), float(z_target_mm), int(direction), n,
                                     _stream(stream)))
    out["plane_z"] = float(z_target_mm)


def ray_law(k: dict) -> RayLaw:
    """plt_ray_law from a dict of the law's DERIVED constants (kind, plane_z, lam_lo, lam_hi,
    disc_r, disc_x0, cap_cos_min, dir_x, dir_z, sensor_w, sensor_h, pupil_z, pupil_r,
    width_px, height_px, spp), e.g. plt_inputs.philox.law_constants(law)."""
    g = lambda key: float(k.get(key, 0.0))
    return RayLaw(LAW_KINDS[k["kind"]], int(k.get("width_px", 0)), int(k.get("height_px", 0)), int(k.get("spp", 0)),
                  g("plane_z"), g("disc_r"), g("disc_x0"), g("cap_cos_min"), g("dir_x"), g("dir_z"), g("sensor_w"),
                  g("sensor_h"), g("pupil_z"), g("pupil_r"), g("lam_lo"), g("lam_hi"))


def gen_rays(law_constants: dict, seed: int, start: int, n: int, out: dict | None = None, with_dz: bool = True,
             stream=None, device="cuda") -> dict:
    """plt_gen_rays: rays [start, start + n) of a law, generated on the device (Philox4x32-10
    keyed by seed, counted by the global index).  `out` (optional) holds preallocated arrays."""
    import torch
    n = int(n)
    if out is None:
        out = {k: torch.empty(n, dtype=torch.float32, device=device) for k in RAY_KEYS if with_dz or k != "dz"}
        if not with_dz:
            out["dz"] = None
    out["plane_z"] = float(law_constants["plane_z"])
    law = ray_law(law_constants)
    r = _rays_struct(out, n)
    _check(load().plt_gen_rays(C.byref(law), int(seed) & 0xFFFFFFFFFFFFFFFF, int(start), C.byref(r), n,
                               _stream(stream)))
    return out


def _host_ptr(t, n=None, dtype=None):
    """Pointer to a contiguous CPU tensor (pinned for overlap) -- host side of plt_query_host."""
    if t is None:
        return None
    if t.is_cuda:
        raise ValueError("plt_query_host takes HOST tensors for rays / returned hits")
    if not t.is_contiguous():
        raise ValueError("host buffers must be contiguous")
    if dtype is not None and t.dtype != dtype:
        raise ValueError(f"expected {dtype}, got {t.dtype}")
    if n is not None and t.numel() < n:
        raise ValueError(f"host buffer holds {t.numel()} < {n} elements")
    return C.c_void_p(t.data_ptr())


def alloc_host_hits(n: int, pin: bool = True) -> dict:
    import torch
    h = {k: torch.empty(n, dtype=torch.float32, pin_memory=pin) for k in HIT_KEYS}
    h["mask_bits"] = torch.empty((n + 31) // 32, dtype=torch.int32, pin_memory=pin)
    return h


def query_host(lens, path_id: int, m, host_rays: dict, film_desc: dict | None = None, film=None, film_host=None,
               host_trace: dict | None = None, host_map: dict | None = None, weight_scale: float = 1.0,
               chunk: int = 1 << 21, direction: int = FORWARD, precision: int = FP32, channel=None,
               n: int | None = None, stream=None):
    """plt_query_host: trace (lens != None) and/or map (m != None) a batch whose rays are HOST
    tensors (pinned), chunked host -> device copies on the library's copy stream overlapping
    the kernels; hits optionally returned to host dicts (alloc_host_hits), valid hits
    splatted into the device `film`, copied to `film_host` at the end."""
    import torch
    n = int(host_rays["ox"].numel()) if n is None else int(n)
    f = torch.float32
    r = Rays(*(_host_ptr(host_rays.get(k) if k == "dz" else host_rays[k], n, f) for k in RAY_KEYS),
             float(host_rays["plane_z"]))

    def hh(h):
        if h is None:
            return None
        return Hits(_host_ptr(h["mask_bits"], (n + 31) // 32, torch.int32), *(_host_ptr(h[k], n, f) for k in HIT_KEYS),
                    None)

    ht, hm = hh(host_trace), hh(host_map)
    spl, keep = (None, None)
    if film is not None:
        spl, keep = _splat_struct({"film_desc": film_desc, "film": film, "channel": channel,
                                   "weight_scale": weight_scale}, n)
    npx = film_desc["channels"] * film_desc["height_px"] * film_desc["width_px"] if film_desc else 0
    _check(load().plt_query_host(lens.handle if lens is not None else None, int(path_id), int(direction),
                                 int(precision), m.handle if m is not None else None, C.byref(r),
                                 C.byref(ht) if ht is not None else None, C.byref(hm) if hm is not None else None,
                                 C.byref(spl) if spl is not None else None,
                                 _host_ptr(film_host, npx, torch.int64) if film_host is not None else None,
                                 n, int(chunk), _stream(stream)))
    return film_host


def pupil_weight(sensor_z_mm: float, disc_z_mm: float, disc_r_mm: float) -> float:
    """plt_pupil_weight: pi r^2 / (sensor_z - disc_z)^2, the pupil-sampling factor of
    plt_shade_plane_weighted."""
    w = C.c_double()
    _check(load().plt_pupil_weight(float(sensor_z_mm), float(disc_z_mm), float(disc_r_mm), C.byref(w)))
    return w.value


KERNEL_KINDS = {0: "jit", 1: "packed", 2: "scalar", 3: "fp64"}


def trace_kernel(lens: "Lens", path_id: int, direction: int = FORWARD, precision: int = FP32) -> str:
    """plt_trace_kernel: which kernel plt_trace_rays runs for this path in this process
    ("jit", "packed", "scalar" or "fp64")."""
    k = C.c_int(-1)
    _check(load().plt_trace_kernel(lens.handle, int(path_id), int(direction), int(precision), C.byref(k)))
    return KERNEL_KINDS[k.value]


def film_resolve(film_d: dict, film, out, scale: float = 1.0, stream=None):
    import torch
    fd = film_desc(film_d)
    npx = film_d["channels"] * film_d["height_px"] * film_d["width_px"]
    _check(load().plt_film_resolve(C.byref(fd), _ptr(film, npx, torch.int64), _ptr(out, npx, torch.float32),
                                   float(scale), _stream(stream)))
