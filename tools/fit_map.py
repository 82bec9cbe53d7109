"""Offline weight fitting of one light path's factorised map on exact-trace data
(the paper's data collection and training).

    python tools/fit_map.py --config C2 [--path <id>] [--train-rays 2^23] [--steps 6000]
                            [--out maps/c2_allT.pltmap] [--report maps/c2_allT.json]

Data: seeded rays of the config's law (a training seed disjoint from the evaluation
seed), labelled by the library's exact trace (plt_trace_rays; float64 mode for ghost
paths).  Inputs and targets are reduced by the rotation/reflection symmetry of §4.1
(P:310-325): x = (r, w'_x, w'_y, lambda), targets (p'_x, p'_y, w'_x, w'_y, w'_z, I) in
the canonical frame.  Classifier 4-32-32-1 (tanh) with BCE on all rays,
regressor 4-32^5-6 (tanh) on valid rays only with MSE on position/throughput
and (1 - cos) on direction.  Adam with an exponentially decaying learning rate
(the paper's 1e-4 x 0.95 per 10k batches over 40-200 epochs of 81 M samples, P:393-394,
is compressed to a few thousand large batches here).  The trained weights are rounded
to bf16 and written as a PLTMAP01 blob; accuracy of the LIBRARY's eval_map against the
exact trace is reported on held-out rays.

This is an offline tool: PyTorch trains the weights; the product path (eval_map) is the
tcgen05 kernel.  It does not import the oracle.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2605_04017_b200 as plt  # noqa: E402
from plt_inputs import configs as C  # noqa: E402
from plt_inputs import rays as R  # noqa: E402


def unpack_mask(words: torch.Tensor, n: int) -> torch.Tensor:
    w = words.view(torch.int32).to(torch.int64) & 0xFFFFFFFF
    bits = (w[:, None] >> torch.arange(32, device=w.device)) & 1
    return bits.reshape(-1)[:n].bool()


def trace_labels(lens, pid, direction, law, seed, n, precision):
    """Exact-trace labels for n rays (chunked through the library)."""
    chunk = 1 << 22
    xs, ys, vs = [], [], []
    for s0 in range(0, n, chunk):
        cnt = min(chunk, n - s0)
        rays = R.gen_rays(law, seed, s0, cnt)
        d = plt.rays_to_device(rays)
        h = plt.alloc_hits(cnt)
        plt.trace_rays(lens, pid, d, h, direction=direction, precision=precision)
        v = unpack_mask(h["mask_bits"], cnt)
        inp = torch.stack([d["ox"], d["oy"], d["dx"], d["dy"], d["dz"], d["lambda_nm"]], 1)
        out = torch.stack([h["px"], h["py"], h["dx"], h["dy"], h["dz"], h["throughput"]], 1)
        xs.append(inp)
        ys.append(out)
        vs.append(v)
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


def flare_films(cfg_name, lens, m, pid, seed_shift=0):
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


def flare_report(cfg_name, lens, m, pid):
    fd = C.CONFIGS[cfg_name]["film"]
    f = flare_films(cfg_name, lens, m, pid)
    g = flare_films(cfg_name, lens, m, pid, seed_shift=8)   # independent rays: Monte-Carlo floor
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--path", type=int, default=0, help="path id (0 = all-T)")
    ap.add_argument("--train-rays", type=int, default=1 << 24)
    ap.add_argument("--eval-rays", type=int, default=1 << 22)
    ap.add_argument("--steps", type=int, default=20000)
    ap.add_argument("--qat-steps", type=int, default=5000)
    ap.add_argument("--batch", type=int, default=1 << 15)
    ap.add_argument("--balance", choices=("paper", "none"), default="paper",
                    help="paper: valid and invalid rays weigh equally in the BCE (P:387)")
    ap.add_argument("--out", default=None)
    ap.add_argument("--report", default=None)
    a = ap.parse_args()
    torch.manual_seed(0)
    cfg = C.CONFIGS[a.config]
    law = dict(cfg["law"])
    if "channels" in cfg:
        law["lam"] = (400.0, 700.0)       # flare configs: train over the visible band
    lens = plt.Lens(C.lens_text(a.config), **cfg["opts"])
    pid = a.path or lens.all_t_id()
    direction = cfg["direction"]
    prec = plt.FP32 if pid == lens.all_t_id() else plt.FP64
    t0 = time.time()
    inp, out, valid = trace_labels(lens, pid, direction, law, 7_000_001, a.train_rays, prec)
    x, y = canonical(inp, out)
    del inp, out
    print(f"train data: {a.train_rays} rays, valid {valid.float().mean().item():.4f}, {time.time() - t0:.1f} s")
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

    cls = mlp([4, 32, 32, 1]).cuda()
    reg = mlp([4, 32, 32, 32, 32, 32, 6]).cuda()
    lbl = valid.float()[:, None]
    frac = float(lbl.mean())
    pos_w = torch.tensor((1 - frac) / max(frac, 1e-9) if a.balance == "paper" else 1.0, device="cuda")
    bce = torch.nn.BCEWithLogitsLoss(pos_weight=pos_w)
    yh_mid, yh_half = ymid.float(), yhalf.float()

    def reg_loss(p, t):
        mse = ((p[:, [0, 1, 5]] - t[:, [0, 1, 5]]) ** 2).mean()
        wp = p[:, 2:5] * yh_half[2:5] + yh_mid[2:5]
        wt = t[:, 2:5] * yh_half[2:5] + yh_mid[2:5]
        cos = torch.nn.functional.cosine_similarity(wp, wt, dim=1).mean()
        return mse + (1.0 - cos)
    xv = xh[valid]
    inp_e, out_e, valid_e = trace_labels(lens, pid, direction, law, 7_000_002, a.eval_rays, prec)
    xe, ye = canonical(inp_e, out_e)
    xeh = norm_x(xe)
    rep = {"config": a.config, "path_id": pid, "train_rays": a.train_rays, "eval_rays": int(inp_e.shape[0]),
           "steps": a.steps, "qat_steps": a.qat_steps, "batch": a.batch, "balance": a.balance,
           "valid_trace": float(valid_e.float().mean())}
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
    del xh, xv, yh, lbl, xe, ye, xeh

    def layers_of(m):
        return [(l.weight.detach().cpu().numpy(), l.bias.detach().cpu().numpy())
                for l in m if isinstance(l, torch.nn.Linear)]
    blob = R.write_map_blob(pid, direction, lo.float().cpu().numpy(), hi.float().cpu().numpy(),
                            ymid.float().cpu().numpy(), yhalf.float().cpu().numpy(), layers_of(cls), layers_of(reg))
    if a.out:
        os.makedirs(os.path.dirname(os.path.abspath(a.out)), exist_ok=True)
        with open(a.out, "wb") as f:
            f.write(blob)

    # ---- held-out accuracy of the LIBRARY eval_map vs the exact trace
    inp, out, valid = inp_e, out_e, valid_e

    m = plt.Map(blob, lens=lens)
    n = inp.shape[0]
    d = {k: inp[:, j].contiguous() for j, k in enumerate(plt.RAY_KEYS)}
    d["plane_z"] = law["plane_z"]
    hm = plt.alloc_hits(n)
    plt.eval_map(m, d, hm)
    torch.cuda.synchronize()
    mv = unpack_mask(hm["mask_bits"], n)
    both = mv & valid
    dp = torch.sqrt((hm["px"] - out[:, 0]) ** 2 + (hm["py"] - out[:, 1]) ** 2)[both]
    dw = torch.sqrt((hm["dx"] - out[:, 2]) ** 2 + (hm["dy"] - out[:, 3]) ** 2 + (hm["dz"] - out[:, 4]) ** 2)[both]
    dI = (hm["throughput"] - out[:, 5]).abs()[both]
    rep["eval_map"] = {"valid_map": float(mv.float().mean()),
                       "mask_agreement": float((mv == valid).float().mean()),
                       "false_valid": float((mv & ~valid).float().mean()),
                       "false_blocked": float((~mv & valid).float().mean()),
                       "dp_mm": quantiles(dp), "dw": quantiles(dw), "dI": quantiles(dI)}
    if "channels" in cfg:
        rep["flare"] = flare_report(a.config, lens, m, pid)
    rep["seconds"] = time.time() - t0
    print(json.dumps(rep, indent=1))
    if a.report:
        with open(a.report, "w") as f:
            json.dump(rep, f, indent=1)


if __name__ == "__main__":
    main()
