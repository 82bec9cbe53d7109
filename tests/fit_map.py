"""Offline weight fitting of one light path's factorised map on exact-trace data
(the paper's data collection and training).

    python tests/fit_map.py --config C2 [--path <id>] [--train-rays 2^24] [--steps 20000]
                            [--out maps/C2_0.pltmap] [--report profiles/r01_fit_C2_0.json]

TEST INFRASTRUCTURE (it lives under tests/ because it calls the oracle): the committed
blobs in maps/ are inputs of parity tests and of bench.py, so — like every stored
oracle input — they are written by a script whose labels come from the float64 ORACLE
only (oracle.trace), never from the CUDA path.  PyTorch fits the weights
(any device); the optional --report then measures the LIBRARY's eval_map against the
library's exact trace on held-out rays.

Data: seeded rays of the config's law (a training seed disjoint from the evaluation
seeds), labelled by oracle.trace in float64.  Inputs and targets are reduced by the rotation/reflection symmetry of §4.1
(P:310-325): x = (r, w'_x, w'_y, lambda), targets (p'_x, p'_y, w'_x, w'_y, w'_z, I) in
the canonical frame.  Classifier 4-32-32-1 (tanh) with BCE on all rays,
regressor 4-32^5-6 (tanh) on valid rays only with MSE on position/throughput
and (1 - cos) on direction.  Adam with an exponentially decaying learning rate
(the paper's 1e-4 x 0.95 per 10k batches over 40-200 epochs of 81 M samples, P:393-394,
is compressed to a few thousand large batches here).  The trained weights are rounded
to bf16 and written as a PLTMAP01 blob; accuracy of the LIBRARY's eval_map against the
exact trace is reported on held-out rays.

The product path (eval_map) is the tcgen05 kernel; nothing here is on it.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time

RAY_KEYS = ("ox", "oy", "dx", "dy", "dz", "lambda_nm")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
from plt_inputs import configs as C  # noqa: E402
from plt_inputs import rays as R  # noqa: E402


def unpack_mask(words: torch.Tensor, n: int) -> torch.Tensor:
    w = words.view(torch.int32).to(torch.int64) & 0xFFFFFFFF
    bits = (w[:, None] >> torch.arange(32, device=w.device)) & 1
    return bits.reshape(-1)[:n].bool()


def oracle_labels(olens, pid, direction, law, seed, n, device):
    """Exact float64 labels from the oracle for rays [0, n) of the law (seeded chunks)."""
    rays = R.gen_rays(law, seed, 0, n)
    o = oracle.trace(olens, pid, direction, rays, threads=oracle.host_threads())
    inp = torch.from_numpy(np.stack([rays[k] for k in RAY_KEYS], 1)).to(device)
    out = torch.from_numpy(np.stack([o[k] for k in ("px", "py", "dx", "dy", "dz", "I")], 1)).to(device)
    return inp, out, torch.from_numpy(o["valid"]).to(device)


def library_labels(plt, lens, pid, direction, law, seed, n, precision):
    """Exact-trace labels from the library (report only; chunked)."""
    chunk = 1 << 22
    xs, ys, vs = [], [], []
    for s0 in range(0, n, chunk):
        cnt = min(chunk, n - s0)
        d = plt.rays_to_device(R.gen_rays(law, seed, s0, cnt))
        h = plt.alloc_hits(cnt)
        plt.trace_rays(lens, pid, d, h, direction=direction, precision=precision)
        vs.append(unpack_mask(h["mask_bits"], cnt))
        xs.append(torch.stack([d[k] for k in RAY_KEYS], 1))
        ys.append(torch.stack([h[k] for k in ("px", "py", "dx", "dy", "dz", "throughput")], 1))
    return torch.cat(xs), torch.cat(ys), torch.cat(vs)


def canonical(inp, out=None):
    """§4.1 reduction: rotate p onto +x, reflect so w'_y >= 0 (and map outputs alike)."""
    px, py, wx, wy = inp[:, 0].double(), inp[:, 1].double(), inp[:, 2].double(), inp[:, 3].double()
    r = torch.sqrt(px * px + py * py)
    tt = torch.sqrt(wx * wx + wy * wy)
    c = torch.where(r > 0, px / r.clamp_min(1e-30), torch.where(tt > 0, wx / tt.clamp_min(1e-30), torch.ones_like(r)))
    s = torch.where(r > 0, py / r.clamp_min(1e-30), torch.where(tt > 0, wy / tt.clamp_min(1e-30), torch.zeros_like(r)))
    wpx = c * wx + s * wy
    wpy = -s * wx + c * wy
    flip = wpy < 0
    wpy = torch.where(flip, -wpy, wpy)
    x = torch.stack([r, wpx, wpy, inp[:, 5].double()], 1)
    if out is None:
        return x
    qx, qy = c * out[:, 0] + s * out[:, 1], -s * out[:, 0] + c * out[:, 1]
    vx, vy = c * out[:, 2] + s * out[:, 3], -s * out[:, 2] + c * out[:, 3]
    qy = torch.where(flip, -qy, qy)
    vy = torch.where(flip, -vy, vy)
    y = torch.stack([qx, qy, vx, vy, out[:, 4].double(), out[:, 5].double()], 1)
    return x, y


class QLinear(torch.nn.Linear):
    """Linear layer whose forward can see its weights rounded to bf16 (straight-through
    gradient), so the last phase of training fits the weights eval_map actually uses."""
    quant = False

    def forward(self, x):
        w = self.weight
        if QLinear.quant:
            w = w + (w.to(torch.bfloat16).float() - w).detach()
        return torch.nn.functional.linear(x, w, self.bias)


def mlp(dims):
    layers = []
    for i, (a, b) in enumerate(zip(dims[:-1], dims[1:])):
        layers.append(QLinear(a, b))
        if i + 2 < len(dims):
            layers.append(torch.nn.Tanh())
    return torch.nn.Sequential(*layers)


def train(model, loss_fn, X, Y, steps, batch, lr0, lr_end, log_every=1000, name=""):
    opt = torch.optim.Adam(model.parameters(), lr=lr0)
    gamma = (lr_end / lr0) ** (1.0 / max(1, steps))
    sched = torch.optim.lr_scheduler.ExponentialLR(opt, gamma)
    n = X.shape[0]
    g = torch.Generator(device=X.device).manual_seed(1234)
    for it in range(steps):
        idx = torch.randint(0, n, (batch,), device=X.device, generator=g)
        loss = loss_fn(model(X[idx]), Y[idx])
        opt.zero_grad(set_to_none=True)
        loss.backward()
        opt.step()
        sched.step()
        if log_every and (it % log_every == 0 or it == steps - 1):
            print(f"  {name} step {it:6d} loss {loss.item():.3e} lr {sched.get_last_lr()[0]:.2e}", flush=True)
    return model


def flare_films(plt, cfg_name, lens, m, pid, seed_shift=0):
    """RGB flare films of one ghost path on the config's rays (2^20 rays per
    channel), splatted from the exact trace (float64 mode) and from the map, same rays."""
    cfg = C.CONFIGS[cfg_name]
    fd, n = cfg["film"], cfg["n_per_channel"]
    npx = fd["channels"] * fd["height_px"] * fd["width_px"]
    films = {k: torch.zeros(npx, dtype=torch.int64, device="cuda") for k in ("trace", "map")}
    for c, lam in enumerate(cfg["channels"]):
        law = dict(cfg["law"])
        law["lam"] = lam
        rays = R.gen_rays(law, cfg["seed"] * 16 + c + seed_shift, 0, n)
        d = plt.rays_to_device(rays)
        ch = torch.full((n,), c, dtype=torch.uint8, device="cuda")
        h = plt.alloc_hits(n)
        plt.trace_rays(lens, pid, d, h, direction=cfg["direction"], precision=plt.FP64)
        plt.splat_sensor(fd, films["trace"], h, channel=ch, weight_scale=1.0 / n)
        h = plt.alloc_hits(n)
        plt.eval_map(m, d, h)
        plt.splat_sensor(fd, films["map"], h, channel=ch, weight_scale=1.0 / n)
    torch.cuda.synchronize()
    return {k: v.double() * 2.0 ** -32 for k, v in films.items()}


def film_diff(img, ref, fd, bins=(1, 4, 16)):
    """Reading A30: film error of a path as the energy-normalised L1 distance
    sum|img - ref| / sum ref, on the film and on films binned b x b (the paper's per-image
    MAPE, does not state its normalisation or resolution); plus MAPE over
    the pixels the reference lights, mean |img - ref| / ref, on the 16 x 16 binned film."""
    out = {}
    C_, H, W = fd["channels"], fd["height_px"], fd["width_px"]
    for b in bins:
        i = img.view(C_, H // b, b, W // b, b).sum((2, 4))
        r = ref.view(C_, H // b, b, W // b, b).sum((2, 4))
        out[f"rel_l1_bin{b}"] = float((i - r).abs().sum() / r.sum().clamp_min(1e-300))
        if b == bins[-1]:
            lit = r > 0
            out[f"mape_lit_bin{b}"] = float(((i - r).abs()[lit] / r[lit]).mean())
    out["energy_ratio"] = float(img.sum() / ref.sum().clamp_min(1e-300))
    return out


def flare_report(plt, cfg_name, lens, m, pid):
    fd = C.CONFIGS[cfg_name]["film"]
    f = flare_films(plt, cfg_name, lens, m, pid)
    g = flare_films(plt, cfg_name, lens, m, pid, seed_shift=8)   # independent rays: Monte-Carlo floor
    return {"map_vs_trace_same_rays": film_diff(f["map"], f["trace"], fd),
            "trace_vs_trace_other_rays": film_diff(g["trace"], f["trace"], fd),
            "map_vs_trace_other_rays": film_diff(g["map"], f["trace"], fd)}


def quantiles(t):
    t = t.float()[: 1 << 20]
    if t.numel() == 0:
        return {"p50": float("nan"), "p90": float("nan"), "p99": float("nan")}
    return {f"p{int(p * 100)}": float(torch.quantile(t, p)) for p in (0.5, 0.9, 0.99)}


def model_errors(reg, cls, xh, y, valid, ymid, yhalf):
    """Errors of the PyTorch model itself, in the canonical frame (|dp|, |dw| are invariant
    under the rotation/reflection): separates fitting error from bf16/kernel error."""
    with torch.no_grad():
        pv = (cls(xh)[:, 0] > 0)
        p = reg(xh[valid]).double() * yhalf + ymid
        t = y[valid]
        w = p[:, 2:5] / p[:, 2:5].norm(dim=1, keepdim=True)     # eval_map renormalises w (A15)
        dp = torch.sqrt(((p[:, :2] - t[:, :2]) ** 2).sum(1))
        dw = torch.sqrt(((w - t[:, 2:5]) ** 2).sum(1))
    return {"mask_agreement": float((pv == valid).float().mean()), "dp_mm": quantiles(dp), "dw": quantiles(dw)}


def library_report(a, cfg, law, pid, blob, rep):
    """Held-out accuracy of the LIBRARY's eval_map against the library's exact trace."""
    import paper_2605_04017_b200 as plt
    lens = plt.Lens(C.lens_text(a.config), **cfg["opts"])
    prec = plt.FP32 if pid == lens.all_t_id() else plt.FP64
    inp, out, valid = library_labels(plt, lens, pid, cfg["direction"], law, 7_000_002, a.eval_rays, prec)
    m = plt.Map(blob, lens=lens)
    n = inp.shape[0]
    d = {k: inp[:, j].contiguous() for j, k in enumerate(RAY_KEYS)}
    d["plane_z"] = law["plane_z"]
    hm = plt.alloc_hits(n)
    plt.eval_map(m, d, hm)
    torch.cuda.synchronize()
    mv = unpack_mask(hm["mask_bits"], n)
    both = mv & valid
    dp = torch.sqrt((hm["px"] - out[:, 0]) ** 2 + (hm["py"] - out[:, 1]) ** 2)[both]
    dw = torch.sqrt((hm["dx"] - out[:, 2]) ** 2 + (hm["dy"] - out[:, 3]) ** 2 + (hm["dz"] - out[:, 4]) ** 2)[both]
    dI = (hm["throughput"] - out[:, 5]).abs()[both]
    rep["eval_map_vs_library_trace"] = {
        "rays": n, "valid_trace": float(valid.float().mean()), "valid_map": float(mv.float().mean()),
        "mask_agreement": float((mv == valid).float().mean()),
        "false_valid": float((mv & ~valid).float().mean()), "false_blocked": float((~mv & valid).float().mean()),
        "dp_mm": quantiles(dp), "dw": quantiles(dw), "dI": quantiles(dI)}
    if "channels" in cfg:
        rep["flare"] = flare_report(plt, a.config, lens, m, pid)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--path", type=int, default=0, help="path id (0 = all-T)")
    ap.add_argument("--train-rays", type=int, default=1 << 24)
    ap.add_argument("--holdout-rays", type=int, default=1 << 21)
    ap.add_argument("--eval-rays", type=int, default=1 << 22)
    ap.add_argument("--steps", type=int, default=20000)
    ap.add_argument("--qat-steps", type=int, default=5000)
    ap.add_argument("--batch", type=int, default=1 << 15)
    ap.add_argument("--balance", choices=("paper", "none"), default="paper",
                    help="paper: valid and invalid rays weigh equally in the BCE (P:387)")
    ap.add_argument("--out", default=None)
    ap.add_argument("--report", default=None, help="also measure the library (needs a GPU)")
    a = ap.parse_args()
    torch.manual_seed(0)
    dev = "cuda" if torch.cuda.is_available() else "cpu"
    cfg = C.CONFIGS[a.config]
    law = dict(cfg["law"])
    if "channels" in cfg:
        law["lam"] = (400.0, 700.0)       # flare configs: train over the visible band
    olens = oracle.load_lens(C.lens_text(a.config), cfg["opts"])
    pid = a.path or oracle.all_t_id(olens.n_optical)
    direction = cfg["direction"]
    t0 = time.time()
    inp, out, valid = oracle_labels(olens, pid, direction, law, 7_000_001, a.train_rays, dev)
    x, y = canonical(inp, out)
    del inp, out
    print(f"train data: {a.train_rays} rays (oracle), valid {valid.float().mean().item():.4f}, "
          f"{time.time() - t0:.1f} s", flush=True)
    lo, hi = x.min(0).values, x.max(0).values
    span = (hi - lo).clamp_min(1e-6)
    lo, hi = lo - 0.01 * span, hi + 0.01 * span
    yv = y[valid]
    ymid = 0.5 * (yv.max(0).values + yv.min(0).values)
    yhalf = (0.5 * (yv.max(0).values - yv.min(0).values)).clamp_min(1e-6) * 1.02
    norm_x = lambda x: ((2.0 * (x - lo) / (hi - lo)) - 1.0).clamp(-1, 1).float()
    xh = norm_x(x)
    yh = ((yv - ymid) / yhalf).float()
    del x, y, yv

    cls = mlp([4, 32, 32, 1]).to(dev)
    reg = mlp([4, 32, 32, 32, 32, 32, 6]).to(dev)
    lbl = valid.float()[:, None]
    frac = float(lbl.mean())
    pos_w = torch.tensor((1 - frac) / max(frac, 1e-9) if a.balance == "paper" else 1.0, device=dev)
    bce = torch.nn.BCEWithLogitsLoss(pos_weight=pos_w)
    yh_mid, yh_half = ymid.float(), yhalf.float()

    def reg_loss(p, t):
        mse = ((p[:, [0, 1, 5]] - t[:, [0, 1, 5]]) ** 2).mean()
        wp = p[:, 2:5] * yh_half[2:5] + yh_mid[2:5]
        wt = t[:, 2:5] * yh_half[2:5] + yh_mid[2:5]
        cos = torch.nn.functional.cosine_similarity(wp, wt, dim=1).mean()
        return mse + (1.0 - cos)
    xv = xh[valid]
    inp_e, out_e, valid_e = oracle_labels(olens, pid, direction, law, 7_000_004, a.holdout_rays, dev)
    xe, ye = canonical(inp_e, out_e)
    xeh = norm_x(xe)
    rep = {"config": a.config, "path_id": pid, "labels": "oracle (float64)", "train_rays": a.train_rays,
           "holdout_rays": a.holdout_rays, "steps": a.steps, "qat_steps": a.qat_steps, "batch": a.batch,
           "balance": a.balance, "train_device": dev, "valid_train": frac,
           "valid_holdout": float(valid_e.float().mean())}
    # phase 1: fp32 weights; phase 2: weights seen through bf16 rounding (eval_map's operand type)
    for phase, steps, lr0, lr1 in (("fp32", a.steps, 3e-3, 1e-5), ("bf16-qat", a.qat_steps, 1e-5, 1e-6)):
        QLinear.quant = phase != "fp32"
        train(cls, bce, xh, lbl, steps, a.batch, lr0, lr1, log_every=5000, name=f"classifier/{phase}")
        train(reg, reg_loss, xv, yh, steps, a.batch, lr0, lr1, log_every=5000, name=f"regressor/{phase}")
        if phase == "fp32":
            rep["torch_fp32_weights"] = model_errors(reg, cls, xeh, ye, valid_e, ymid, yhalf)
            QLinear.quant = True
            rep["torch_bf16_rounded_before_qat"] = model_errors(reg, cls, xeh, ye, valid_e, ymid, yhalf)
    rep["torch_bf16_after_qat"] = model_errors(reg, cls, xeh, ye, valid_e, ymid, yhalf)
    del xh, xv, yh, lbl, xe, ye, xeh, inp_e, out_e, valid_e

    def layers_of(m):
        return [(l.weight.detach().cpu().numpy(), l.bias.detach().cpu().numpy())
                for l in m if isinstance(l, torch.nn.Linear)]
    blob = R.write_map_blob(pid, direction, lo.float().cpu().numpy(), hi.float().cpu().numpy(),
                            ymid.float().cpu().numpy(), yhalf.float().cpu().numpy(), layers_of(cls), layers_of(reg),
                            plane_z=law["plane_z"])
    if a.out:
        os.makedirs(os.path.dirname(os.path.abspath(a.out)), exist_ok=True)
        with open(a.out, "wb") as f:
            f.write(blob)
    if a.report:
        library_report(a, cfg, law, pid, blob, rep)
    rep["seconds"] = time.time() - t0
    print(json.dumps(rep, indent=1))
    if a.report:
        with open(a.report, "w") as f:
            json.dump(rep, f, indent=1)


if __name__ == "__main__":
    main()
