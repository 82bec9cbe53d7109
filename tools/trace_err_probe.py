"""Probe: fp32 trace (the kernel the process selects: JIT for all-T paths) against the float64
oracle on C1 / C2 / C3 rays (2^18 each) -- max |dp|, |dw|, |dI| over rays valid in both and
mask mismatches outside the band.  For A/B of arithmetic choices via PLT_JIT_DEFINES."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle  # noqa: E402
import paper_2605_04017_b200 as plt  # noqa: E402
from gpu_helpers import compare_trace, gpu_trace  # noqa: E402
from plt_inputs import configs as C  # noqa: E402
from plt_inputs import rays as R  # noqa: E402

res = {}
for name in ("C1", "C2", "C3"):
    cfg = C.CONFIGS[name]
    gl = plt.Lens(C.lens_text(name), **cfg["opts"])
    ol = oracle.load_lens(C.lens_text(name), cfg["opts"])
    rays = R.gen_rays(cfg["law"], 101, 0, 1 << 18)
    pid = gl.all_t_id()
    g = gpu_trace(plt, gl, pid, rays, direction=cfg["direction"])
    o = oracle.trace(ol, pid, cfg["direction"], rays, threads=oracle.host_threads())
    st = compare_trace(g, o, assert_ok=False)
    res[name] = {k: st[k] for k in ("mask_mismatch", "max_dp", "max_dw", "max_dI", "n_both")}
print(json.dumps({"defines": os.environ.get("PLT_JIT_DEFINES", ""), **res}))
