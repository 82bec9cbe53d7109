"""The five workload configurations of BASELINE.json ``configs``.

Pure data: lens name, direction, lens options, ray law, sizes and seeds.
Sensor planes of forward configs are NaN, i.e. "paraxial focus at
lambda_ref", which the oracle and the CUDA library each resolve on their
own.  The backward config (C3) starts rays ON the sensor, so its sensor
plane is an explicit number: rear vertex of the 24 mm stand-in
(36.3658661036 mm = sum of its thickness column) + 15.603 mm (SURVEY.md A.3
BFL), recorded here as a plain constant.
"""
from __future__ import annotations

import math
import os

import numpy as np

from . import rays as R
from .lenses import LENSES

NAN = float("nan")

FORWARD, BACKWARD = 0, 1


def lens_opts(**kw) -> dict:
    o = {"input_plane_z_mm": -5.0, "sensor_z_mm": NAN, "sensor_w_mm": 0.0, "sensor_h_mm": 0.0,
         "backward_exit_z_mm": -5.0, "housing_radius_mm": 0.0, "lambda_ref_nm": R.LAMBDA_D}
    o.update(kw)
    return o


WIDE24_REAR_VERTEX_Z = 36.3658661036
WIDE24_SENSOR_Z = WIDE24_REAR_VERTEX_Z + 15.603

CONFIGS = {
    # C1 singlet + stop: 4096 (p, w) x 3 Fraunhofer lambdas, exact trace vs oracle + ABCD
    "C1": {"lens": "singlet", "direction": FORWARD, "opts": lens_opts(), "seed": 1,
           "n_base": 4096, "lambdas": (R.LAMBDA_F, R.LAMBDA_D, R.LAMBDA_C),
           "law": {"kind": "disc_cap", "plane_z": -5.0, "disc_r": 10.0, "cap_deg": 10.0,
                   "lam": R.LAMBDA_D}},
    # C2 double-Gauss 50 mm, 16 M rays, 400-700 nm (the bench workload at N=1)
    "C2": {"lens": "dgauss50", "direction": FORWARD, "opts": lens_opts(), "seed": 2,
           "n": 1 << 24,
           "law": {"kind": "disc_cap", "plane_z": -5.0, "disc_r": 1.05 * 12.6, "cap_deg": 25.0,
                   "lam": (400.0, 700.0)},
           "map_norm": {"in_lo": (0.0, -0.43, 0.0, 400.0), "in_hi": (13.23, 0.43, 0.43, 700.0),
                        "out_mid": (0.0, 0.0, 0.0, 0.0, 0.9, 0.5),
                        "out_half": (25.0, 25.0, 0.5, 0.5, 0.1, 0.5)}},
    # C3 24 mm backward camera batch at 32768 spp scale (192x128 px x 32768 spp); C3 and C5
    # draw their rays from the counter-based generator (plt_inputs/philox.py = plt_gen_rays
    # on the device), so full-size batches are generated in HBM and sampled anywhere
    "C3": {"lens": "wide24", "direction": BACKWARD,
           "opts": lens_opts(sensor_z_mm=WIDE24_SENSOR_Z, sensor_w_mm=24.0, sensor_h_mm=16.0,
                             backward_exit_z_mm=-5.0),
           "seed": 3, "n": 192 * 128 * 32768,
           "law": {"kind": "sensor_pupil", "plane_z": WIDE24_SENSOR_Z, "sensor_w": 24.0,
                   "sensor_h": 16.0, "pupil_z": WIDE24_REAR_VERTEX_Z, "pupil_r": 9.8055,
                   "lam": (400.0, 700.0), "rng": "philox"},
           "map_norm": {"in_lo": (0.0, -0.8, 0.0, 400.0), "in_hi": (14.5, 0.8, 0.8, 700.0),
                        "out_mid": (0.0, 0.0, 0.0, 0.0, -0.8, 0.5),
                        "out_half": (30.0, 30.0, 0.8, 0.8, 0.2, 0.5)}},
    # C3 as a depth-of-field camera: pixel-stratified rays of a
    # 192 x 128 image over the 24 x 16 mm sensor, a checkerboard scene plane 1 m in front of
    # the lens (object side, lens frame), sensor shifts for the focus sweep
    "C3_DOF": {"lens": "wide24", "direction": BACKWARD,
               "opts": lens_opts(sensor_z_mm=WIDE24_SENSOR_Z, sensor_w_mm=24.0, sensor_h_mm=16.0,
                                 backward_exit_z_mm=-5.0),
               "seed": 33, "width_px": 192, "height_px": 128, "spp": 64,
               "scene": {"z_mm": -1000.0, "period_mm": 50.0, "contrast": 0.1},
               "sensor_shifts_mm": (-1.0, 0.0, 0.6, 1.5),
               "law": {"kind": "sensor_grid", "plane_z": WIDE24_SENSOR_Z, "sensor_w": 24.0, "sensor_h": 16.0,
                       "width_px": 192, "height_px": 128, "spp": 64, "pupil_z": WIDE24_REAR_VERTEX_Z,
                       "pupil_r": 9.8055, "lam": (400.0, 700.0)}},
    # C4 flare: 22 mm @ 15 deg and 59 mm @ 10 deg, 2^20 rays per ghost per RGB channel
    "C4_22": {"lens": "wide22", "direction": FORWARD,
              "opts": lens_opts(sensor_w_mm=24.0, sensor_h_mm=16.0), "seed": 4,
              "n_per_channel": 1 << 20, "channels": R.FLARE_CHANNELS_NM,
              "film": {"width_px": 768, "height_px": 512, "channels": 3, "sensor_w_mm": 24.0,
                       "sensor_h_mm": 16.0, "center_x_mm": 0.0, "center_y_mm": 0.0},
              "law": {"kind": "collimated", "plane_z": -5.0, "disc_r": 11.858,
                      "disc_x0": -5.0 * math.tan(math.radians(15.0)), "angle_deg": 15.0,
                      "lam": 550.0}},
    "C4_59": {"lens": "dgauss59", "direction": FORWARD,
              "opts": lens_opts(sensor_w_mm=24.0, sensor_h_mm=16.0), "seed": 4,
              "n_per_channel": 1 << 20, "channels": R.FLARE_CHANNELS_NM,
              "film": {"width_px": 768, "height_px": 512, "channels": 3, "sensor_w_mm": 24.0,
                       "sensor_h_mm": 16.0, "center_x_mm": 0.0, "center_y_mm": 0.0},
              "law": {"kind": "collimated", "plane_z": -5.0, "disc_r": 14.762286,
                      "disc_x0": -5.0 * math.tan(math.radians(10.0)), "angle_deg": 10.0,
                      "lam": 550.0}},
    # C5 sweep 2^20 .. 2^30 with the C2 lens and law
    "C5": {"lens": "dgauss50", "direction": FORWARD, "opts": lens_opts(), "seed": 5,
           "sizes": tuple(1 << k for k in range(20, 31, 2)),
           "law": {"kind": "disc_cap", "plane_z": -5.0, "disc_r": 1.05 * 12.6, "cap_deg": 25.0,
                   "lam": (400.0, 700.0), "rng": "philox"}},
}


def dof_law(shift_mm: float = 0.0, spp: int | None = None, pupil: tuple | None = None) -> dict:
    """C3_DOF rays with the sensor moved by shift_mm along z (away from the lens for > 0).
    pupil = (z_mm, radius_mm) re-aims the rays at another disc, e.g. the lens's exit pupil
    from plt_lens_pupils (default: the rear clear aperture)."""
    cfg = CONFIGS["C3_DOF"]
    law = dict(cfg["law"])
    law["plane_z"] = law["plane_z"] + shift_mm
    if spp is not None:
        law["spp"] = spp
    if pupil is not None:
        law["pupil_z"], law["pupil_r"] = float(pupil[0]), float(pupil[1])
    return law


def lens_text(cfg_name: str) -> str:
    return LENSES[CONFIGS[cfg_name]["lens"]]


def c1_rays() -> dict:
    """C1: the same 4096 (p, w) repeated for the three Fraunhofer wavelengths (12,288 rays)."""
    cfg = CONFIGS["C1"]
    base = R.gen_rays(cfg["law"], cfg["seed"], 0, cfg["n_base"])
    out = {k: np.concatenate([base[k]] * 3) for k in ("ox", "oy", "dx", "dy", "dz")}
    out["lambda_nm"] = np.concatenate(
        [np.full(cfg["n_base"], lam, np.float32) for lam in cfg["lambdas"]])
    out["plane_z"] = base["plane_z"]
    return out


def c1_abcd_rays(n: int = 256) -> dict:
    """C1 ABCD subset: meridional rays, h in [-0.4, 0.4] mm, slope u in [-2e-3, 2e-3]."""
    rng = np.random.default_rng([1, 0xABCD])
    h = rng.uniform(-0.4, 0.4, n)
    u = rng.uniform(-2e-3, 2e-3, n)
    inv = 1.0 / np.sqrt(1.0 + u * u)
    f = np.float32
    return {"ox": np.zeros(n, f), "oy": h.astype(f), "dx": np.zeros(n, f),
            "dy": (u * inv).astype(f), "dz": inv.astype(f),
            "lambda_nm": np.full(n, R.LAMBDA_D, f), "plane_z": -5.0}


def flare_rays(cfg_name: str, channel: int, start: int, count: int) -> dict:
    """C4 rays of one RGB channel (same (p, w) law, channel wavelength, channel-specific stream)."""
    cfg = CONFIGS[cfg_name]
    law = dict(cfg["law"])
    law["lam"] = cfg["channels"][channel]
    return R.gen_rays(law, cfg["seed"] * 16 + channel, start, count)


MAPS_DIR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "maps")


def fitted_map_blob(cfg_name: str, path_tag: int = 0) -> bytes:
    """A committed fitted map, maps/<cfg>_<tag>.pltmap (tag 0 = all-T), written by
    tests/fit_map.py from float64 oracle labels (maps/README.md)."""
    with open(os.path.join(MAPS_DIR, f"{cfg_name}_{int(path_tag)}.pltmap"), "rb") as f:
        return f.read()


def map_blob(cfg_name: str, path_id: int, seed: int = 1234) -> bytes:
    cfg = CONFIGS[cfg_name]
    nm = cfg.get("map_norm") or CONFIGS["C2"]["map_norm"]
    return R.make_map_blob(path_id, cfg["direction"], seed, nm["in_lo"], nm["in_hi"],
                           nm["out_mid"], nm["out_half"], plane_z=cfg["law"]["plane_z"])
