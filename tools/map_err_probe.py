"""Per-output error of eval_map vs the oracle on a map blob (diagnostic; prints a table).
    python tools/map_err_probe.py [C2_0 ...]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2605_04017_b200 as plt  # noqa: E402
from plt_inputs import configs as C  # noqa: E402
from plt_inputs import rays as R  # noqa: E402
from gpu_helpers import unpack_mask  # noqa: E402

tags = sys.argv[1:] or ["C2_0", "C3_0", "C4_22_65616", "C4_59_16404", "random"]
for tag in tags:
    if tag == "random":
        name, blob = "C2", C.map_blob("C2", 1 << 10)
    else:
        name, ptag = tag.rsplit("_", 1)
        blob = C.fitted_map_blob(name, int(ptag))
    cfg = C.CONFIGS[name]
    law = dict(cfg["law"])
    if "channels" in cfg:
        law["lam"] = (400.0, 700.0)
    rays = R.gen_rays(law, 41, 0, 1 << 17)
    n = rays["ox"].size
    m = plt.Map(blob)
    d = plt.rays_to_device(rays)
    h = plt.alloc_hits(n)
    raw = torch.zeros(7 * n, dtype=torch.float32, device="cuda")
    plt.eval_map(m, d, h, raw=raw)
    torch.cuda.synchronize()
    g = raw.cpu().numpy().reshape(7, n).T.astype(np.float64)
    gv = unpack_mask(h["mask_bits"].cpu().numpy(), n)
    o = oracle.map_eval(blob, rays, threads=oracle.host_threads())
    lo = o["raw"][:, 0]
    dl = np.abs(g[:, 0] - lo)
    both = gv & o["valid"]
    print(f"{tag:14s} valid {o['valid'].mean():.3f} |logit| p50 {np.median(np.abs(lo)):6.2f} max {np.abs(lo).max():6.1f}"
          f"  dlogit max {dl.max():.2e} rel max {(dl / np.maximum(1, np.abs(lo))).max():.2e}"
          f"  mask mismatches {int((gv != o['valid']).sum())} (|logit|<2e-3: {int(((gv != o['valid']) & (np.abs(lo) <= 2e-3)).sum())})")
    for j, k in enumerate(("px'", "py'", "wx'", "wy'", "wz'", "I")):
        e = np.abs(g[both, 1 + j] - o["raw"][both, 1 + j])
        print(f"    {k:4s} max {e.max():.2e}  p99 {np.quantile(e, 0.99):.2e}  |y| max {np.abs(o['raw'][both, 1 + j]).max():.2f}")
