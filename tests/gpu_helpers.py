"""Helpers for the -m gpu parity tests: run the CUDA path through the C-ABI binding
and compare against the float64 oracle under the SURVEY.md §8(c) rules."""
from __future__ import annotations

import numpy as np

# North-star tolerances (BASELINE.json north_star)
TOL_P = 1e-4      # mm, exit origin
TOL_W = 1e-5      # exit direction components
TOL_I = 1e-5      # Fresnel throughput
TOL_NET = 2e-3    # network outputs (normalised units, bf16 weights)
BAND_GEO = 1e-6   # mm, aperture-edge band excluded from mask exactness
BAND_KAPPA = 1e-9
BAND_DISC = 1e-9
BAND_DIR = 1e-9


def unpack_mask(words: np.ndarray, n: int) -> np.ndarray:
    w = np.ascontiguousarray(words).view(np.uint32)
    bits = (w[:, None] >> np.arange(32, dtype=np.uint32)[None, :]) & 1
    return bits.reshape(-1)[:n].astype(bool)


def gpu_trace(plt, lens, path_id, rays_np, direction=0, precision=0, flags=True):
    import torch
    n = rays_np["ox"].size
    d = plt.rays_to_device(rays_np)
    h = plt.alloc_hits(n, flags=flags)
    plt.trace_rays(lens, path_id, d, h, direction=direction, precision=precision)
    torch.cuda.synchronize()
    out = {k: h[k].cpu().numpy().astype(np.float64) for k in ("px", "py", "dx", "dy", "dz", "throughput")}
    out["I"] = out.pop("throughput")
    out["valid"] = unpack_mask(h["mask_bits"].cpu().numpy(), n)
    out["flags"] = h["flags"].cpu().numpy() if flags else None
    return out


def near_edge(margins: np.ndarray) -> np.ndarray:
    return ((margins[:, 0] < BAND_GEO) | (margins[:, 1] < BAND_KAPPA) |
            (margins[:, 2] < BAND_DISC) | (margins[:, 3] < BAND_DIR))


def compare_trace(gpu: dict, ora: dict, tol_p=TOL_P, tol_w=TOL_W, tol_i=TOL_I, assert_ok=True) -> dict:
    excl = near_edge(ora["margins"])
    mism = (gpu["valid"] != ora["valid"]) & ~excl
    both = gpu["valid"] & ora["valid"]
    stats = {"n": int(gpu["valid"].size), "valid_frac": float(ora["valid"].mean()),
             "mask_mismatch": int(mism.sum()), "excluded": int(excl.sum()), "n_both": int(both.sum())}
    if both.any():
        stats["max_dp"] = float(max(np.abs(gpu["px"][both] - ora["px"][both]).max(),
                                    np.abs(gpu["py"][both] - ora["py"][both]).max()))
        stats["max_dw"] = float(max(np.abs(gpu[k][both] - ora[k][both]).max() for k in ("dx", "dy", "dz")))
        stats["max_dI"] = float(np.abs(gpu["I"][both] - ora["I"][both]).max())
    else:
        stats.update(max_dp=0.0, max_dw=0.0, max_dI=0.0)
    inval = ~gpu["valid"]
    stats["invalid_nonzero"] = int(sum(np.count_nonzero(gpu[k][inval]) for k in ("px", "py", "dx", "dy", "dz", "I")))
    print("compare_trace", stats)
    if assert_ok:
        assert stats["mask_mismatch"] == 0, stats
        assert stats["max_dp"] <= tol_p, stats
        assert stats["max_dw"] <= tol_w, stats
        assert stats["max_dI"] <= tol_i, stats
        assert stats["invalid_nonzero"] == 0, stats
    return stats
