"""Pin of the oracle's map query (O9-O10: canonicalisation, normalisation, gated MLP,
de-normalisation and rotation back) against the oracle's exact trace through
the committed fitted maps (maps/*.pltmap, written by tests/fit_map.py from oracle labels).

A correctly evaluated fitted map reproduces the exact transport to the fitting error
(tens of microns); a dropped rotation, a wrong reflection sign, a swapped normalisation
bound or a transposed weight matrix moves exit points by millimetres and fails here.
This is what makes the map-vs-trace relation pinned."""
import glob
import os

import numpy as np
import pytest

import oracle
from plt_inputs import configs as C
from plt_inputs import rays as R

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
MAPS = sorted(glob.glob(os.path.join(ROOT, "maps", "*.pltmap")))
SEED = 7_000_005            # disjoint from the fitting seeds (7_000_001 .. 7_000_004)


@pytest.mark.parametrize("path", MAPS, ids=[os.path.basename(p) for p in MAPS])
def test_fitted_map_reproduces_exact_trace(path):
    cfg_name, pid = os.path.basename(path)[:-7].rsplit("_", 1)
    cfg = C.CONFIGS[cfg_name]
    lens = oracle.load_lens(C.lens_text(cfg_name), cfg["opts"])
    pid = int(pid) or oracle.all_t_id(lens.n_optical)
    law = dict(cfg["law"])
    if "channels" in cfg:
        law["lam"] = (400.0, 700.0)
    rays = R.gen_rays(law, SEED, 0, 1 << 15)
    thr = oracle.host_threads()
    t = oracle.trace(lens, pid, cfg["direction"], rays, threads=thr)
    m = oracle.map_eval(open(path, "rb").read(), rays, threads=thr)
    both = t["valid"] & m["valid"]
    agree = float((t["valid"] == m["valid"]).mean())
    dp = np.hypot(m["px"] - t["px"], m["py"] - t["py"])[both]
    dw = np.sqrt(sum((m[k] - t[k]) ** 2 for k in ("dx", "dy", "dz")))[both]
    dI = np.abs(m["I"] - t["I"])[both]
    stats = {"valid": float(t["valid"].mean()), "agree": agree, "n_both": int(both.sum()),
             "dp99": float(np.quantile(dp, 0.99)), "dw99": float(np.quantile(dw, 0.99)),
             "dI99": float(np.quantile(dI, 0.99))}
    print(os.path.basename(path), stats)
    assert stats["n_both"] >= 300, stats
    assert agree >= 0.99, stats
    assert stats["dp99"] <= 0.1 and stats["dw99"] <= 5e-3 and stats["dI99"] <= 1e-3, stats
    # the symmetry the map relies on: rotating every input by 90 degrees rotates
    # the map's outputs exactly the same way (the canonical inputs are unchanged)
    rot = dict(rays, ox=-rays["oy"], oy=rays["ox"], dx=-rays["dy"], dy=rays["dx"])
    m2 = oracle.map_eval(open(path, "rb").read(), rot, threads=thr)
    v = m["valid"] & m2["valid"]
    assert float((m["valid"] == m2["valid"]).mean()) >= 0.999
    np.testing.assert_allclose(m2["px"][v], -m["py"][v], atol=2e-4)
    np.testing.assert_allclose(m2["py"][v], m["px"][v], atol=2e-4)
