"""Dev probe: time eval_map / trace_rays on the C2 workload and report the network
error against the oracle (max |raw gpu - raw oracle| on a sample).  Used for tuning
(e.g. PLT_MAP_GROUPS); not part of the library."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import oracle
import paper_2605_04017_b200 as plt
from plt_inputs import configs as C
from plt_inputs import rays as R


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 24
    cfg = C.CONFIGS["C2"]
    rays = R.gen_rays(cfg["law"], cfg["seed"], 0, n)
    lens = plt.Lens(C.lens_text("C2"), **cfg["opts"])
    pid = lens.all_t_id()
    blob = C.map_blob("C2", pid) if os.environ.get("MAP") == "random" else C.fitted_map_blob("C2")
    m = plt.Map(blob, lens=lens)
    d = plt.rays_to_device(rays)
    h = plt.alloc_hits(n)
    raw = torch.empty(7 * n, dtype=torch.float32, device="cuda")
    for _ in range(3):
        plt.eval_map(m, d, h, raw=raw)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    reps = 20
    e0.record()
    for _ in range(reps):
        plt.eval_map(m, d, h)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    th = plt.alloc_hits(n)
    for _ in range(3):
        plt.trace_rays(lens, pid, d, th)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        plt.trace_rays(lens, pid, d, th)
    e1.record()
    torch.cuda.synchronize()
    tms = e0.elapsed_time(e1) / reps
    idx = R.sample_indices(n, 1 << 17, 5)
    sub = {k: rays[k][idx] for k in plt.RAY_KEYS}
    sub["plane_z"] = rays["plane_z"]
    o = oracle.map_eval(blob, sub, threads=oracle.host_threads())
    g = raw.cpu().numpy().reshape(7, n).T[idx]
    dec = np.abs(o["raw"][:, 0]) > 2e-3
    both = dec & o["valid"] & (g[:, 0] >= 0)
    err_logit = np.abs(g[:, 0] - o["raw"][:, 0]).max()
    err_reg = np.abs(g[both, 1:] - o["raw"][both, 1:]).max(axis=0)
    print(f"lib={os.path.basename(plt.LIB_PATH)} groups={os.environ.get('PLT_MAP_GROUPS', 'default')} n={n} eval_map {ms:.3f} ms "
          f"({n / ms / 1e6:.2f} G rays/s)  trace {tms:.3f} ms ({n / tms / 1e6:.2f} G rays/s)  "
          f"valid={o['valid'].mean():.3f} err_logit={err_logit:.2e} err_reg={np.array2string(err_reg, precision=2)}")


if __name__ == "__main__":
    main()
