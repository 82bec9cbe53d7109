"""Dev probe: hits of the JIT-specialised trace vs the generic packed kernel on the same rays
(run twice with PLT_TRACE_JIT=0/1; compares the saved outputs)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2605_04017_b200 as plt  # noqa: E402
from plt_inputs import configs as C  # noqa: E402
from plt_inputs import rays as R  # noqa: E402

out = sys.argv[1]
cfg = C.CONFIGS["C2"]
lens = plt.Lens(C.lens_text("C2"), **cfg["opts"])
n = 1 << 20
d = plt.rays_to_device(R.gen_rays(cfg["law"], 5, 0, n))
h = plt.alloc_hits(n, flags=True)
plt.trace_rays(lens, lens.all_t_id(), d, h)
torch.cuda.synchronize()
np.savez(out, **{k: h[k].cpu().numpy() for k in plt.HIT_KEYS + ("mask_bits", "flags")})
if len(sys.argv) > 2:
    a, b = np.load(sys.argv[1]), np.load(sys.argv[2])
    for k in a.files:
        diff = np.nonzero(a[k].view(np.uint32 if a[k].dtype == np.float32 else a[k].dtype) !=
                          b[k].view(np.uint32 if b[k].dtype == np.float32 else b[k].dtype))[0]
        print(k, "differs at", diff.size, "positions", diff[:5],
              (a[k][diff[:3]], b[k][diff[:3]]) if diff.size else "")
