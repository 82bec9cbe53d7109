"""plt_trace_paths: one ray batch along many paths (the flare image's per-path forward loop,
Listing 1).  In float64 the paths' common all-T prefix is traced once and each
path resumes from the state before its first reflection; the hits, masks and film must be
bit-identical to one plt_trace_rays(_splat) call per path -- on both flare lenses (every
two-bounce ghost), backward, with four-bounce paths, an aspheric coated element, a housing,
ragged batch sizes and forced chunking -- and a sample of paths is checked against the
oracle directly."""
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle
from plt_inputs import configs as C
from plt_inputs import rays as R
from plt_inputs.lenses import LENSES

from gpu_helpers import compare_trace, unpack_mask

pytestmark = pytest.mark.gpu

KEYS = ("px", "py", "dx", "dy", "dz", "throughput")


def _host(h, n):
    import torch
    torch.cuda.synchronize()
    out = {k: h[k].cpu().numpy().copy() for k in KEYS}
    out["mask_bits"] = h["mask_bits"].cpu().numpy().copy()
    out["flags"] = h["flags"].cpu().numpy().copy() if h.get("flags") is not None else None
    return out


def _run_both(plt, lens, ids, rays_np, direction, precision, film_desc=None, channel=None):
    """trace_paths vs one trace_rays per path: (list of host hit dicts, film) for each."""
    import torch
    n = rays_np["ox"].size
    d = plt.rays_to_device(rays_np)
    res = []
    for mode in ("paths", "single"):
        film = None
        spl = None
        if film_desc is not None:
            film = torch.zeros(film_desc["channels"] * film_desc["height_px"] * film_desc["width_px"],
                               dtype=torch.int64, device="cuda")
            ch = None if channel is None else torch.from_numpy(channel).cuda()
            spl = {"film_desc": film_desc, "film": film, "channel": ch, "weight_scale": 1.0 / n}
        hs = [plt.alloc_hits(n, flags=True) for _ in ids]
        for h in hs:   # poison: every output must be written
            for k in KEYS:
                h[k].fill_(7.0)
            h["mask_bits"].fill_(-1)
            h["flags"].fill_(9)
        if mode == "paths":
            plt.trace_paths(lens, ids, d, hs, direction=direction, precision=precision, splat=spl)
        else:
            for g, h in zip(ids, hs):
                plt.trace_rays(lens, g, d, h, direction=direction, precision=precision, splat=spl)
        res.append(([_host(h, n) for h in hs], None if film is None else film.cpu().numpy()))
    return res


def _assert_identical(res, ids, n):
    (hp, fp), (hs, fs) = res
    nvalid = 0
    for g, a, b in zip(ids, hp, hs):
        for k in KEYS:
            assert np.array_equal(a[k].view(np.uint32), b[k].view(np.uint32)), (g, k)
        words = (n + 31) // 32
        assert np.array_equal(a["mask_bits"][:words], b["mask_bits"][:words]), g
        assert np.array_equal(a["flags"], b["flags"]), g
        nvalid += int(unpack_mask(a["mask_bits"], n).sum())
    if fp is not None:
        assert np.array_equal(fp, fs)
        assert fp.sum() > 0
    return nvalid


@pytest.mark.parametrize("name", ["C4_22", "C4_59"])
def test_all_ghosts_bit_identical_to_per_path_traces(gpu_lib, name):
    plt = gpu_lib
    cfg = C.CONFIGS[name]
    lens = plt.Lens(C.lens_text(name), **cfg["opts"])
    ids = [int(g) for g in lens.enumerate_ghosts(2)[0]]        # all-T + every two-bounce ghost
    n = (1 << 16) + 77                                          # ragged tail
    rays = C.flare_rays(name, 1, 0, n)
    chan = np.ones(n, np.uint8)
    res = _run_both(plt, lens, ids, rays, 0, plt.FP64, film_desc=cfg["film"], channel=chan)
    nvalid = _assert_identical(res, ids, n)
    assert nvalid > 1000


def test_oracle_parity_through_trace_paths(gpu_lib):
    """Two ghosts and the all-T path of the 22 mm lens from one plt_trace_paths call,
    against the oracle (fp64 tolerances)."""
    plt = gpu_lib
    name = "C4_22"
    cfg = C.CONFIGS[name]
    lens = plt.Lens(C.lens_text(name), **cfg["opts"])
    ol = oracle.load_lens(C.lens_text(name), cfg["opts"])
    all_ids = [int(g) for g in lens.enumerate_ghosts(2)[0]]
    ids = [all_ids[0], 65616, all_ids[-1]]
    n = (1 << 15) + 5
    rays = C.flare_rays(name, 2, 0, n)
    (hp, _), _ = _run_both(plt, lens, ids, rays, 0, plt.FP64)
    for g, h in zip(ids, hp):
        o = oracle.trace(ol, g, 0, rays, threads=oracle.host_threads())
        gpu = {k: h[k].astype(np.float64) for k in KEYS}
        gpu["I"] = gpu.pop("throughput")
        gpu["valid"] = unpack_mask(h["mask_bits"], n)
        compare_trace(gpu, o, tol_p=5e-5, tol_w=2e-7, tol_i=2e-7)


def test_backward_four_bounce_asphere_coating(gpu_lib):
    """Backward camera rays through the 24 mm lens with an aspheric, coated element; the
    all-T path, two-bounce and four-bounce ghosts in one call."""
    plt = gpu_lib
    cfg = C.CONFIGS["C3"]
    lines, k = [], 0
    for line in LENSES["wide24"].splitlines():
        body = line.split("#", 1)[0].split()
        if len(body) >= 4 and body[0] != "name" and body[2].lower() != "stop" and float(body[0]) != 0.0:
            k += 1
            if k == 3:
                line = line.split("#", 1)[0].rstrip() + " asph:-0.5,3e-5,-1e-7 coat:1.38,550"
        lines.append(line)
    lens = plt.Lens("\n".join(lines) + "\n", **cfg["opts"])
    ids2 = [int(g) for g in lens.enumerate_ghosts(2)[0]]
    ids4 = [int(g) for g in lens.enumerate_ghosts(4)[0] if int(g) not in set(ids2)]
    ids = ids2[:12] + ids4[:: max(1, len(ids4) // 10)]
    n = (1 << 15) + 129
    rays = R.gen_rays(cfg["law"], 31, 0, n)
    res = _run_both(plt, lens, ids, rays, 1, plt.FP64)
    assert _assert_identical(res, ids, n) > 100


def test_housing_and_fp32_and_edge_cases(gpu_lib):
    """A housing cylinder (C2 lens), the float32 mode (per-path traces), n = 0, no paths,
    one path, repeated ids."""
    import torch
    plt = gpu_lib
    cfg = C.CONFIGS["C2"]
    lens = plt.Lens(LENSES["dgauss50"], **dict(cfg["opts"], housing_radius_mm=10.0))
    g = [int(x) for x in lens.enumerate_ghosts(2)[0]]
    ids = [g[5], g[1], g[5], g[0], g[-1]]
    n = 40000 + 3
    rays = R.gen_rays(cfg["law"], 5, 0, n)
    for prec in (plt.FP64, plt.FP32):
        _assert_identical(_run_both(plt, lens, ids, rays, 0, prec), ids, n)
    _assert_identical(_run_both(plt, lens, ids[:1], rays, 0, plt.FP64), ids[:1], n)
    d = plt.rays_to_device(rays)
    plt.trace_paths(lens, [], d, [], precision=plt.FP64)
    h = plt.alloc_hits(n)
    h["px"].fill_(3.0)
    plt.trace_paths(lens, ids[:1], d, [h], precision=plt.FP64, n=0)
    torch.cuda.synchronize()
    assert float(h["px"][0]) == 3.0
    with pytest.raises(plt.PltError):
        plt.trace_paths(lens, [12345678901], d, [h], precision=plt.FP64)   # id inconsistent with the lens


def test_forced_chunking_is_bit_identical(gpu_lib):
    """The prefix scratch is processed in chunks of whole tiles when large; force 3 chunks
    (PLT_PREFIX_CHUNK, read per call) in a subprocess and compare with the unchunked run."""
    code = r'''
import sys, numpy as np, torch
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import paper_2605_04017_b200 as plt
from plt_inputs import configs as C
cfg = C.CONFIGS["C4_59"]
lens = plt.Lens(C.lens_text("C4_59"), **cfg["opts"])
ids = [int(g) for g in lens.enumerate_ghosts(2)[0]][::4]
n = 3 * 8192 + 100
d = plt.rays_to_device(C.flare_rays("C4_59", 0, 0, n))
fd = cfg["film"]
film = torch.zeros(fd["channels"] * fd["height_px"] * fd["width_px"], dtype=torch.int64, device="cuda")
hs = [plt.alloc_hits(n) for _ in ids]
plt.trace_paths(lens, ids, d, hs, precision=plt.FP64, splat={"film_desc": fd, "film": film, "weight_scale": 1.0 / n})
torch.cuda.synchronize()
np.savez(sys.argv[1], film=film.cpu().numpy(), **{f"{k}{j}": h[k].cpu().numpy() for j, h in enumerate(hs) for k in ("px", "dz", "throughput", "mask_bits")})
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for chunk in ("0", "8192"):
        path = f"/tmp/plt_chunk_{chunk}.npz"
        env = dict(os.environ, PLT_PREFIX_CHUNK=chunk)
        subprocess.run([sys.executable, "-c", code, path], cwd=root, env=env, check=True, timeout=300)
        outs.append(np.load(path))
    a, b = outs
    assert set(a.files) == set(b.files)
    for k in a.files:
        assert np.array_equal(a[k], b[k]), k
    assert a["film"].sum() > 0


def test_render_flare_per_path_films_through_trace_paths(gpu_lib):
    """render_flare(per_path=...) traces the ghosts with one plt_trace_paths call per channel and
    splats each path's hits into its own film (plt_splat_sensor); every film must equal the
    per-path fused trace + splat bit for bit, and so must the summed image."""
    import torch
    from paper_2605_04017_b200.render import render_flare
    plt = gpu_lib
    name = "C4_59"
    cfg = C.CONFIGS[name]
    lens = plt.Lens(C.lens_text(name), **cfg["opts"])
    ghosts = [int(g) for g in lens.enumerate_ghosts(2)[0][1:]][::3]
    n = (1 << 14) + 9
    rays = [plt.rays_to_device(C.flare_rays(name, c, 0, n)) for c in range(3)]
    fd = cfg["film"]
    npx = fd["channels"] * fd["height_px"] * fd["width_px"]
    per = {g: torch.zeros(npx, dtype=torch.int64, device="cuda") for g in ghosts}
    render_flare(lens, ghosts, rays, fd, None, per_path=per, weight_scale=1.0 / n)
    whole = torch.zeros(npx, dtype=torch.int64, device="cuda")
    render_flare(lens, ghosts, rays, fd, whole, weight_scale=1.0 / n)
    h = plt.alloc_hits(n)
    total = torch.zeros(npx, dtype=torch.int64, device="cuda")
    for g in ghosts:
        ref = torch.zeros(npx, dtype=torch.int64, device="cuda")
        for c in range(3):
            ch = torch.full((n,), c, dtype=torch.uint8, device="cuda")
            plt.trace_rays(lens, g, rays[c], h, precision=plt.FP64,
                           splat={"film_desc": fd, "film": ref, "channel": ch, "weight_scale": 1.0 / n})
        torch.cuda.synchronize()
        assert torch.equal(per[g], ref), g
        total += ref
    assert torch.equal(whole, total) and int(total.sum()) > 0
