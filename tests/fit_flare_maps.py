"""Fit the factorised map of EVERY two-bounce ghost path of a flare config in one batched
training run (SURVEY.md §8(f) NEXT-2 prerequisite; the paper's per-path training,
PAPER.md:382-394, "each type of path").

    python tests/fit_flare_maps.py --config C4_22 [--rays 2^22] [--steps 20000] [--qat-steps 5000]
                                   [--out maps/flare] [--report profiles/r01_fit_flare_C4_22.json]

TEST INFRASTRUCTURE (under tests/ because it calls the oracle): labels for every path
come from the float64 oracle (oracle.trace), never from the CUDA path, so the blobs may
be oracle inputs.  All P paths train at once: the networks are stacked ([P, out, in]
weights, batched matmuls), each path sampling its own data, one Adam over the stack --
the same losses, canonicalisation, normalisation and bf16-aware fine-tuning as
tests/fit_map.py (whose helpers this reuses).  Paths with fewer than --min-valid valid
training rays get no map (their flare contribution is below the Monte-Carlo noise; the
renderer traces them).
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
from fit_map import canonical, oracle_labels  # noqa: E402
from plt_inputs import configs as C  # noqa: E402
from plt_inputs import rays as R  # noqa: E402

CLS = (4, 32, 32, 1)
REG = (4, 32, 32, 32, 32, 32, 6)


class StackedMLP(torch.nn.Module):
    """P independent tanh MLPs evaluated with batched matmuls: x [P, B, in] -> [P, B, out]."""

    def __init__(self, P, dims, device):
        super().__init__()
        self.W = torch.nn.ParameterList()
        self.b = torch.nn.ParameterList()
        for fi, fo in zip(dims[:-1], dims[1:]):
            lim = (6.0 / (fi + fo)) ** 0.5
            self.W.append(torch.nn.Parameter((torch.rand(P, fo, fi, device=device) * 2 - 1) * lim))
            self.b.append(torch.nn.Parameter(torch.zeros(P, fo, device=device)))
        self.quant = False

    def forward(self, x):
        n = len(self.W)
        for i, (W, b) in enumerate(zip(self.W, self.b)):
            if self.quant:
                W = W + (W.to(torch.bfloat16).float() - W).detach()
            x = torch.baddbmm(b[:, None, :], x, W.transpose(1, 2))
            if i + 1 < n:
                x = torch.tanh(x)
        return x

    def layers(self, p):
        return [(W[p].detach().cpu().numpy(), b[p].detach().cpu().numpy()) for W, b in zip(self.W, self.b)]


def train_stacked(model, loss_fn, sample, steps, lr0, lr1, name, log_every=5000):
    opt = torch.optim.Adam(model.parameters(), lr=lr0)
    sched = torch.optim.lr_scheduler.ExponentialLR(opt, (lr1 / lr0) ** (1.0 / max(1, steps)))
    for it in range(steps):
        x, y = sample()
        loss = loss_fn(model(x), y)
        opt.zero_grad(set_to_none=True)
        loss.backward()
        opt.step()
        sched.step()
        if log_every and (it % log_every == 0 or it == steps - 1):
            print(f"  {name} step {it:6d} loss {loss.item():.3e}", flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C4_22")
    ap.add_argument("--rays", type=int, default=1 << 22)
    ap.add_argument("--steps", type=int, default=20000)
    ap.add_argument("--qat-steps", type=int, default=5000)
    ap.add_argument("--batch", type=int, default=1 << 13)
    ap.add_argument("--min-valid", type=int, default=2000)
    ap.add_argument("--out", default=os.path.join(ROOT, "maps", "flare"))
    ap.add_argument("--report", default=None)
    ap.add_argument("--max-paths", type=int, default=0, help="debug: only the first k ghosts")
    ap.add_argument("--only", default="", help="comma-separated path ids to fit (others untouched)")
    ap.add_argument("--mcmc", type=int, default=0,
                    help="paths with fewer than --min-valid uniform valid rays get this many extra valid "
                         "training rays from the valid-region MCMC sampler (P:385; tests/mcmc_valid.py)")
    a = ap.parse_args()
    torch.manual_seed(0)
    dev = "cuda" if torch.cuda.is_available() else "cpu"
    cfg = C.CONFIGS[a.config]
    law = dict(cfg["law"], lam=(400.0, 700.0))          # continuous lambda, rendered at RGB
    olens = oracle.load_lens(C.lens_text(a.config), cfg["opts"])
    all_ids, _ = oracle.enumerate_ghosts(olens, 2)                     # (ids, (i, j) pairs)
    ids = [int(i) for i in all_ids if int(i) != oracle.all_t_id(olens.n_optical)]
    if a.max_paths:
        ids = ids[:a.max_paths]
    if a.only:
        want = {int(x) for x in a.only.split(",")}
        ids = [i for i in ids if i in want]
    if a.mcmc and not a.only:
        ap.error("--mcmc is meant for the low-valid paths: list them with --only (equal sample counts)")
    t0 = time.time()
    xs, ys, vs, keep = [], [], [], []
    for k, pid in enumerate(ids):
        inp, out, valid = oracle_labels(olens, pid, cfg["direction"], law, 8_000_000 + k, a.rays, "cpu")
        nv = int(valid.sum())
        if nv < a.min_valid and a.mcmc:
            from fit_map import RAY_KEYS
            from mcmc_valid import sample_valid, to_rays
            try:
                st = sample_valid(olens, pid, cfg["direction"], law, law["lam"], a.mcmc, seed=9_000_000 + k,
                                  threads=oracle.host_threads())
            except RuntimeError as e:
                print(e, flush=True)
                st = None
            if st is not None:
                mr = to_rays(st, law)
                o = oracle.trace(olens, pid, cfg["direction"], mr, threads=oracle.host_threads())
                inp = torch.cat([inp, torch.from_numpy(np.stack([mr[kk] for kk in RAY_KEYS], 1))])
                out = torch.cat([out, torch.from_numpy(np.stack([o[kk] for kk in ("px", "py", "dx", "dy", "dz", "I")], 1))])
                valid = torch.cat([valid, torch.from_numpy(o["valid"])])
                print(f"path {pid}: {nv} uniform valid rays + {int(o['valid'].sum())} from MCMC", flush=True)
                nv = int(valid.sum())
        if nv < a.min_valid:
            print(f"path {pid}: {nv} valid training rays -> no map", flush=True)
            continue
        x, y = canonical(inp, out)
        xs.append(x); ys.append(y); vs.append(valid); keep.append(pid)
    P = len(keep)
    print(f"labels for {len(ids)} paths ({P} fitted) in {time.time() - t0:.1f} s", flush=True)
    if P == 0:
        print("no path has enough valid rays to fit", flush=True)
        return

    # per-path normalisation (as fit_map): inputs to [-1, 1] with a 1 % margin, outputs (mid, half)
    lo = torch.stack([x.min(0).values for x in xs]); hi = torch.stack([x.max(0).values for x in xs])
    span = (hi - lo).clamp_min(1e-6)
    lo, hi = lo - 0.01 * span, hi + 0.01 * span
    ymid = torch.stack([0.5 * (y[v].max(0).values + y[v].min(0).values) for y, v in zip(ys, vs)])
    yhalf = torch.stack([(0.5 * (y[v].max(0).values - y[v].min(0).values)).clamp_min(1e-6) * 1.02
                         for y, v in zip(ys, vs)])
    N = xs[0].shape[0]
    XH = torch.stack([((2.0 * (x - l) / (h - l)) - 1.0).clamp(-1, 1).float() for x, l, h in zip(xs, lo, hi)]).to(dev)
    LBL = torch.stack([v.float() for v in vs]).to(dev)                      # [P, N]
    nval = torch.tensor([int(v.sum()) for v in vs], device=dev)
    YV = [((y[v] - m) / h).float() for y, v, m, h in zip(ys, vs, ymid, yhalf)]
    XV = [XH[p][vs[p].to(dev)] for p in range(P)]
    maxv = int(nval.max())
    YVp = torch.zeros(P, maxv, 6, device=dev); XVp = torch.zeros(P, maxv, 4, device=dev)
    for p in range(P):
        YVp[p, :YV[p].shape[0]] = YV[p].to(dev); XVp[p, :XV[p].shape[0]] = XV[p]
    del xs, ys, YV, XV
    frac = LBL.mean(1)                                                       # balanced BCE
    pos_w = ((1 - frac) / frac.clamp_min(1e-9))[:, None, None]
    ar = torch.arange(P, device=dev)[:, None]
    g = torch.Generator(device=dev).manual_seed(99)

    def sample_cls():
        idx = torch.randint(0, N, (P, a.batch), device=dev, generator=g)
        return XH[ar, idx], LBL[ar, idx][..., None]

    def sample_reg():
        idx = (torch.rand(P, a.batch, device=dev, generator=g) * nval[:, None]).long()
        return XVp[ar, idx], YVp[ar, idx]

    ymid_d, yhalf_d = ymid.float().to(dev), yhalf.float().to(dev)

    def bce(z, t):
        l = torch.nn.functional.binary_cross_entropy_with_logits(z, t, pos_weight=pos_w, reduction="none")
        return l.mean(dim=(1, 2)).sum()

    def reg_loss(p, t):
        mse = ((p[..., [0, 1, 5]] - t[..., [0, 1, 5]]) ** 2).mean(dim=(1, 2))
        wp = p[..., 2:5] * yhalf_d[:, None, 2:5] + ymid_d[:, None, 2:5]
        wt = t[..., 2:5] * yhalf_d[:, None, 2:5] + ymid_d[:, None, 2:5]
        cos = torch.nn.functional.cosine_similarity(wp, wt, dim=2).mean(1)
        return (mse + (1.0 - cos)).sum()                                      # P:392, summed over paths

    cls, reg = StackedMLP(P, CLS, dev), StackedMLP(P, REG, dev)
    for phase, steps, lr0, lr1 in (("fp32", a.steps, 3e-3, 1e-5), ("bf16-qat", a.qat_steps, 1e-5, 1e-6)):
        cls.quant = reg.quant = phase != "fp32"
        train_stacked(cls, bce, sample_cls, steps, lr0, lr1, f"classifier/{phase}")
        train_stacked(reg, reg_loss, sample_reg, steps, lr0, lr1, f"regressor/{phase}")

    os.makedirs(os.path.join(a.out, a.config), exist_ok=True)
    rep = {"config": a.config, "paths": len(ids), "fitted": P, "rays_per_path": a.rays, "labels": "oracle (float64)",
           "steps": a.steps, "qat_steps": a.qat_steps, "batch_per_path": a.batch, "seconds": None,
           "valid_train": {str(pid): float(f) for pid, f in zip(keep, frac.tolist())},
           "skipped": [pid for pid in ids if pid not in keep]}
    for p, pid in enumerate(keep):
        blob = R.write_map_blob(pid, cfg["direction"], lo[p].float().numpy(), hi[p].float().numpy(),
                                ymid[p].float().numpy(), yhalf[p].float().numpy(), cls.layers(p), reg.layers(p),
                                plane_z=cfg["law"]["plane_z"])
        with open(os.path.join(a.out, a.config, f"{pid}.pltmap"), "wb") as f:
            f.write(blob)
    rep["seconds"] = time.time() - t0
    print(json.dumps({k: v for k, v in rep.items() if k != "valid_train"}, indent=1))
    if a.report:
        with open(a.report, "w") as f:
            json.dump(rep, f, indent=1)


if __name__ == "__main__":
    main()
