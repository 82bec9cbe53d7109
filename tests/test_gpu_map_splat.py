"""GPU parity of plt_eval_map (tcgen05 fused gated MLP) and plt_splat_sensor against
the float64 oracle.  Network tolerance: 2e-3 absolute on raw outputs at bf16
(SURVEY A18); splat: bit-exact int64 film."""
import numpy as np
import pytest

import oracle
from plt_inputs import configs as C
from plt_inputs import rays as R

from gpu_helpers import TOL_NET, gpu_trace, unpack_mask

pytestmark = pytest.mark.gpu


def gpu_map(plt, m, rays_np, offset=0):
    """Run eval_map; `offset` shifts every device array by that many floats (breaks 16-B
    alignment so the kernel takes its non-TMA load path)."""
    import torch
    n = rays_np["ox"].size
    d = {}
    for k in plt.RAY_KEYS:
        t = torch.zeros(n + offset, dtype=torch.float32, device="cuda")
        t[offset:] = torch.from_numpy(np.ascontiguousarray(rays_np[k], np.float32)).cuda()
        d[k] = t[offset:]
    d["plane_z"] = rays_np["plane_z"]
    h = plt.alloc_hits(n)
    raw = torch.full((7 * n,), float("nan"), dtype=torch.float32, device="cuda")
    plt.eval_map(m, d, h, raw=raw)
    torch.cuda.synchronize()
    out = {k: h[k].cpu().numpy().astype(np.float64) for k in ("px", "py", "dx", "dy", "dz", "throughput")}
    out["I"] = out.pop("throughput")
    out["valid"] = unpack_mask(h["mask_bits"].cpu().numpy(), n)
    out["raw"] = raw.cpu().numpy().reshape(7, n).T.astype(np.float64)
    return out


def compare_map(g, o):
    logit_o = o["raw"][:, 0]
    decided = np.abs(logit_o) > TOL_NET
    assert np.array_equal(g["valid"][decided], o["valid"][decided])
    assert np.all(np.isfinite(g["raw"]))
    assert np.max(np.abs(g["raw"][:, 0] - logit_o)) <= TOL_NET
    both = g["valid"] & o["valid"] & decided
    if both.any():
        err = np.abs(g["raw"][both, 1:] - o["raw"][both, 1:]).max()
        assert err <= TOL_NET, err
        assert np.max(np.abs(g["I"][both] - o["I"][both])) <= TOL_NET * 0.5 + 1e-6
    inval = ~g["valid"]
    for k in ("px", "py", "dx", "dy", "dz", "I"):
        assert np.count_nonzero(g[k][inval]) == 0
    return float(g["valid"].mean())


@pytest.mark.parametrize("n", [1, 127, 128, 129, 1000, 4096 + 37])
def test_eval_map_ragged(gpu_lib, n):
    plt = gpu_lib
    blob = C.map_blob("C2", 1 << 10)
    m = plt.Map(blob)
    rays = R.gen_rays(C.CONFIGS["C2"]["law"], 31, 0, n)
    compare_map(gpu_map(plt, m, rays), oracle.map_eval(blob, rays))


def test_eval_map_c2_2e18_and_unaligned(gpu_lib):
    plt = gpu_lib
    blob = C.map_blob("C2", 1 << 10)
    gl = plt.Lens(C.lens_text("C2"))
    m = plt.Map(blob, lens=gl)
    rays = R.gen_rays(C.CONFIGS["C2"]["law"], 2, 0, 1 << 18)
    o = oracle.map_eval(blob, rays, threads=oracle.host_threads())
    v = compare_map(gpu_map(plt, m, rays), o)
    assert 0.05 < v < 0.95
    compare_map(gpu_map(plt, m, rays, offset=1), o)


def test_eval_map_full_size_sampled(gpu_lib):
    """Full C2 size in the bench's launch configuration; oracle on a 2^15 sample."""
    plt = gpu_lib
    blob = C.map_blob("C2", 1 << 10)
    m = plt.Map(blob)
    cfg = C.CONFIGS["C2"]
    rays = R.gen_rays(cfg["law"], cfg["seed"], 0, cfg["n"])
    g = gpu_map(plt, m, rays)
    idx = R.sample_indices(cfg["n"], 1 << 15, 7)
    sub = {k: rays[k][idx] for k in plt.RAY_KEYS}
    sub["plane_z"] = rays["plane_z"]
    o = oracle.map_eval(blob, sub, threads=oracle.host_threads())
    compare_map({k: v[idx] for k, v in g.items()}, o)


def test_eval_map_backward_map_c3(gpu_lib):
    plt = gpu_lib
    blob = C.map_blob("C3", 1 << 12)
    m = plt.Map(blob, lens=plt.Lens(C.lens_text("C3"), **C.CONFIGS["C3"]["opts"]))
    rays = R.gen_rays(C.CONFIGS["C3"]["law"], 3, 0, 1 << 16)
    compare_map(gpu_map(plt, m, rays), oracle.map_eval(blob, rays, threads=oracle.host_threads()))


@pytest.mark.parametrize("tag", [("C2", 0), ("C3", 0), ("C4_22", 65616), ("C4_59", 16404)],
                         ids=lambda t: f"{t[0]}_{t[1]}")
def test_eval_map_fitted_weights(gpu_lib, tag):
    """Parity on the committed fitted maps (realistic valid fractions and weight scales; the
    blobs come from oracle labels, tests/fit_map.py), 2^17 rays of the config's law."""
    plt = gpu_lib
    name, ptag = tag
    cfg = C.CONFIGS[name]
    blob = C.fitted_map_blob(name, ptag)
    m = plt.Map(blob, lens=plt.Lens(C.lens_text(name), **cfg["opts"]))
    law = dict(cfg["law"])
    if "channels" in cfg:
        law["lam"] = (400.0, 700.0)
    rays = R.gen_rays(law, 41, 0, (1 << 17) + 77)
    v = compare_map(gpu_map(plt, m, rays), oracle.map_eval(blob, rays, threads=oracle.host_threads()))
    assert v > 0.005


FILM = C.CONFIGS["C4_22"]["film"]


def test_splat_bit_exact_vs_oracle(gpu_lib):
    import torch
    plt = gpu_lib
    rng = np.random.default_rng(4)
    n = 300_000
    hits = {"px": rng.uniform(-13, 13, n), "py": rng.uniform(-9, 9, n), "dz": rng.uniform(0.3, 1, n),
            "I": rng.uniform(0, 1, n)}
    # bright compact spot: many hits in a few pixels (atomic hot spot / warp aggregation)
    hot = rng.random(n) < 0.3
    hits["px"][hot] = rng.normal(1.0, 0.01, hot.sum())
    hits["py"][hot] = rng.normal(-2.0, 0.01, hot.sum())
    valid = rng.random(n) < 0.8
    ch = rng.integers(0, 3, n).astype(np.uint8)
    f32 = {k: v.astype(np.float32) for k, v in hits.items()}
    ref, dropped = oracle.splat(FILM, valid, f32["px"], f32["py"], f32["dz"], f32["I"], ch, scale=1.0 / n)
    dev = {"px": torch.from_numpy(f32["px"]).cuda(), "py": torch.from_numpy(f32["py"]).cuda(),
           "dz": torch.from_numpy(f32["dz"]).cuda(), "throughput": torch.from_numpy(f32["I"]).cuda(),
           "dx": torch.zeros(n, device="cuda"), "dy": torch.zeros(n, device="cuda")}
    words = np.zeros((n + 31) // 32, np.uint32)
    for b in range(32):
        sel = np.arange(b, n, 32)
        words[sel // 32] |= valid[sel].astype(np.uint32) << np.uint32(b)
    dev["mask_bits"] = torch.from_numpy(words.view(np.int32)).cuda()
    film = torch.zeros(3 * FILM["height_px"] * FILM["width_px"], dtype=torch.int64, device="cuda")
    drop = torch.zeros(1, dtype=torch.int64, device="cuda")
    plt.splat_sensor(FILM, film, dev, channel=torch.from_numpy(ch).cuda(), weight_scale=1.0 / n, dropped=drop)
    torch.cuda.synchronize()
    assert np.array_equal(film.cpu().numpy().reshape(ref.shape), ref)
    assert int(drop.item()) == dropped
    out = torch.empty(film.numel(), dtype=torch.float32, device="cuda")
    plt.film_resolve(FILM, film, out, scale=2.0)
    torch.cuda.synchronize()
    assert np.allclose(out.cpu().numpy(), ref.reshape(-1) * 2.0 ** -32 * 2.0, rtol=1e-6, atol=0)


def _splat_both(plt, f32, valid, ch, scale):
    import torch
    n = f32["px"].size
    ref, dropped = oracle.splat(FILM, valid, f32["px"], f32["py"], f32["dz"], f32["I"], ch, scale=scale)
    dev = {"px": torch.from_numpy(f32["px"]).cuda(), "py": torch.from_numpy(f32["py"]).cuda(),
           "dz": torch.from_numpy(f32["dz"]).cuda(), "throughput": torch.from_numpy(f32["I"]).cuda(),
           "dx": torch.zeros(n, device="cuda"), "dy": torch.zeros(n, device="cuda")}
    words = np.zeros((n + 31) // 32, np.uint32)
    for b in range(32):
        sel = np.arange(b, n, 32)
        words[sel // 32] |= valid[sel].astype(np.uint32) << np.uint32(b)
    dev["mask_bits"] = torch.from_numpy(words.view(np.int32)).cuda()
    film = torch.zeros(3 * FILM["height_px"] * FILM["width_px"], dtype=torch.int64, device="cuda")
    drop = torch.zeros(1, dtype=torch.int64, device="cuda")
    plt.splat_sensor(FILM, film, dev, channel=torch.from_numpy(ch).cuda(), weight_scale=scale, dropped=drop)
    torch.cuda.synchronize()
    return film.cpu().numpy().reshape(ref.shape), ref, int(drop.item()), dropped


@pytest.mark.parametrize("scale", [1.0, 2.0 ** -20, 2.0 ** -7, 2.0 ** 30, 1.0 / 3.0, 0.75],
                         ids=["1", "2^-20", "2^-7", "2^30", "1/3", "0.75"])
def test_splat_edges_and_scales_bit_exact(gpu_lib, scale):
    """Integer-exact weight path (power-of-two scales) and the double path (others) against
    O11, with hits on pixel edges, film borders, outside the film, and zero / subnormal /
    tie-producing / negative weights."""
    plt = gpu_lib
    rng = np.random.default_rng(12)
    n = 200_003
    W, H, wp, hp = FILM["sensor_w_mm"], FILM["sensor_h_mm"], FILM["width_px"], FILM["height_px"]
    px = rng.uniform(-0.55 * W, 0.55 * W, n)
    py = rng.uniform(-0.55 * H, 0.55 * H, n)
    edge = rng.random(n) < 0.3                           # exactly on pixel boundaries / borders
    px[edge] = (rng.integers(0, wp + 1, edge.sum()) / wp - 0.5) * W
    py[edge] = (0.5 - rng.integers(0, hp + 1, edge.sum()) / hp) * H
    I = rng.uniform(0, 1, n)
    dz = rng.uniform(-1, 1, n)
    kind = rng.integers(0, 8, n)
    I[kind == 0] = 0.0
    I[kind == 1] = 1e-42                                 # subnormal
    I[kind == 2] = rng.integers(1, 2 ** 10, (kind == 2).sum()) / 2.0 ** 10   # short mantissas: ties
    dz[kind == 2] = rng.integers(1, 2 ** 10, (kind == 2).sum()) / 2.0 ** 10
    I[kind == 3] = 1.0
    dz[kind == 3] = 1.0
    I[kind == 4] = -I[kind == 4]                         # negative throughput (API allows it)
    f32 = {"px": px.astype(np.float32), "py": py.astype(np.float32), "dz": dz.astype(np.float32),
           "I": I.astype(np.float32)}
    valid = rng.random(n) < 0.9
    ch = rng.integers(0, 3, n).astype(np.uint8)
    got, ref, gd, rd = _splat_both(plt, f32, valid, ch, scale)
    assert gd == rd
    assert np.array_equal(got, ref), int((got != ref).sum())


def test_flare_ghost_end_to_end_fp64(gpu_lib):
    """GPU fp64 trace of one ghost -> GPU splat equals the oracle splat of the GPU hits
    (binding) and the oracle trace->splat film up to bin flips of edge rays."""
    import torch
    plt = gpu_lib
    cfg = C.CONFIGS["C4_22"]
    gl = plt.Lens(C.lens_text("C4_22"), **cfg["opts"])
    ol = oracle.load_lens(C.lens_text("C4_22"), cfg["opts"])
    pid = oracle.ghost_id(12, 5, 3)   # the paper's path 65616
    assert pid == 65616
    n = 1 << 18
    rays = C.flare_rays("C4_22", 0, 0, n)
    d = plt.rays_to_device(rays)
    h = plt.alloc_hits(n)
    plt.trace_rays(gl, pid, d, h, precision=1)
    film = torch.zeros(3 * 512 * 768, dtype=torch.int64, device="cuda")
    plt.splat_sensor(FILM, film, h, weight_scale=1.0 / n)
    torch.cuda.synchronize()
    gv = unpack_mask(h["mask_bits"].cpu().numpy(), n)
    ref_g, _ = oracle.splat(FILM, gv, h["px"].cpu().numpy(), h["py"].cpu().numpy(), h["dz"].cpu().numpy(),
                            h["throughput"].cpu().numpy(), None, scale=1.0 / n)
    assert np.array_equal(film.cpu().numpy().reshape(ref_g.shape), ref_g)
    o = oracle.trace(ol, pid, 0, rays, threads=oracle.host_threads())
    ref_o, _ = oracle.splat(FILM, o["valid"], o["px"].astype(np.float32), o["py"].astype(np.float32),
                            o["dz"].astype(np.float32), o["I"].astype(np.float32), None, scale=1.0 / n)
    diff = np.abs(ref_o.astype(np.float64) - ref_g.astype(np.float64)).sum()
    assert diff <= 1e-6 * max(1.0, float(ref_o.sum()))
