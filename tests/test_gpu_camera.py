"""GPU parity of the backward camera integrand (plt_shade_plane, O14) and free-space
propagation (plt_propagate_rays) against the oracle, and the depth-of-field camera of
SURVEY §8(f) NEXT-3: map image vs exact-trace image on the same rays, and the
sensor-shift focus sweep with one precomputed map."""
import numpy as np
import pytest

import oracle
from plt_inputs import configs as C
from plt_inputs import rays as R

from gpu_helpers import unpack_mask

pytestmark = pytest.mark.gpu

SCENE = C.CONFIGS["C3_DOF"]["scene"]


@pytest.mark.parametrize("spp", [1, 7, 64])
def test_shade_plane_bit_exact_on_trace_hits(gpu_lib, spp):
    import torch
    plt = gpu_lib
    cfg = C.CONFIGS["C3_DOF"]
    lens = plt.Lens(C.lens_text("C3_DOF"), **cfg["opts"])
    law = C.dof_law(0.0, spp)
    n = cfg["width_px"] * cfg["height_px"] * spp // 4 + 13          # ragged: last pixel partial
    d = plt.rays_to_device(R.gen_rays(law, 5, 0, n))
    h = plt.alloc_hits(n)
    plt.trace_rays(lens, lens.all_t_id(), d, h, direction=plt.BACKWARD)
    pixels = (n + spp - 1) // spp - 2                                 # some rays beyond the film
    film = torch.zeros(pixels, dtype=torch.int64, device="cuda")
    plt.shade_plane(SCENE, cfg["opts"]["backward_exit_z_mm"], h, film, spp, pixels=pixels, weight_scale=0.5)
    torch.cuda.synchronize()
    hh = {k: h[k].cpu().numpy() for k in plt.HIT_KEYS}
    valid = unpack_mask(h["mask_bits"].cpu().numpy(), n)
    ref = oracle.shade_plane(SCENE, cfg["opts"]["backward_exit_z_mm"], valid, hh["px"], hh["py"], hh["dx"], hh["dy"],
                             hh["dz"], hh["throughput"], spp=spp, pixels=pixels, scale=0.5)
    assert valid.mean() > 0.02
    assert np.array_equal(film.cpu().numpy(), ref)
    # the pupil-sampling weighted form (cos^4 of the sensor rays), bit-exact as well
    fw = torch.zeros(pixels, dtype=torch.int64, device="cuda")
    plt.shade_plane(SCENE, cfg["opts"]["backward_exit_z_mm"], h, fw, spp, pixels=pixels, weight_scale=0.5,
                    in_dz=d["dz"])
    torch.cuda.synchronize()
    refw = oracle.shade_plane(SCENE, cfg["opts"]["backward_exit_z_mm"], valid, hh["px"], hh["py"], hh["dx"],
                              hh["dy"], hh["dz"], hh["throughput"], spp=spp, pixels=pixels, scale=0.5,
                              in_dz=d["dz"].cpu().numpy())
    assert np.array_equal(fw.cpu().numpy(), refw)
    assert 0 < refw.sum() < ref.sum()


def test_propagate_matches_closed_form(gpu_lib):
    import torch
    plt = gpu_lib
    law = C.dof_law(1.5, 16)
    rays = R.gen_rays(law, 9, 0, 100_003)
    d = plt.rays_to_device(rays)
    out = {k: torch.empty_like(d[k]) for k in plt.RAY_KEYS}
    z0 = C.CONFIGS["C3"]["law"]["plane_z"]
    plt.propagate_rays(d, out, z0, direction=plt.BACKWARD)
    torch.cuda.synchronize()
    ref = oracle.propagate(rays, z0, direction=oracle.BACKWARD)
    for k in ("ox", "oy"):
        assert np.max(np.abs(out[k].cpu().numpy() - ref[k])) <= 2e-5
    for k in ("dx", "dy", "dz", "lambda_nm"):
        assert np.array_equal(out[k].cpu().numpy(), rays[k])
    plt.propagate_rays(d, d, z0, direction=plt.BACKWARD)               # in place (aliasing allowed)
    torch.cuda.synchronize()
    assert torch.equal(d["ox"], out["ox"]) and torch.equal(d["oy"], out["oy"])


def test_dof_map_vs_trace_and_focus_sweep(gpu_lib):
    import torch
    from paper_2605_04017_b200.render import render_dof
    plt = gpu_lib
    cfg = C.CONFIGS["C3_DOF"]
    lens = plt.Lens(C.lens_text("C3_DOF"), **cfg["opts"])
    m = plt.Map(C.fitted_map_blob("C3"), lens=lens)
    spp = 256
    W, H = cfg["width_px"], cfg["height_px"]

    def sharp(img):
        return float(np.abs(np.diff(img, axis=1)).mean() + np.abs(np.diff(img, axis=0)).mean()) / img.mean()

    res = {}
    for shift in (-1.0, 0.6, 1.5):
        d = plt.rays_to_device(R.gen_rays(C.dof_law(shift, spp), cfg["seed"], 0, W * H * spp))
        imgs = {}
        for key, mm in (("trace", None), ("map", m)):
            film = torch.zeros(W * H, dtype=torch.int64, device="cuda")
            render_dof(lens, d, SCENE, film, spp, cfg["opts"]["backward_exit_z_mm"], m=mm,
                       map_plane_z=C.CONFIGS["C3"]["law"]["plane_z"], weight_scale=1.0 / spp)
            torch.cuda.synchronize()
            imgs[key] = film.double().cpu().numpy().reshape(H, W)
        t, mp = imgs["trace"], imgs["map"]
        lit = t > 0
        res[shift] = {"mape": float(np.mean(np.abs(mp[lit] - t[lit]) / t[lit])), "energy": float(mp.sum() / t.sum()),
                      "sharp_t": sharp(t), "sharp_m": sharp(mp)}
    print(res)
    for r in res.values():
        assert r["mape"] <= 0.08 and abs(r["energy"] - 1) <= 0.04
        assert abs(r["sharp_m"] / r["sharp_t"] - 1) <= 0.03
    for key in ("sharp_t", "sharp_m"):      # the object plane focuses ~0.6 mm behind the infinity focus
        assert res[0.6][key] > res[-1.0][key] and res[0.6][key] > res[1.5][key]


def test_exit_pupil_sampling_raises_the_valid_fraction(gpu_lib):
    """Aiming the sensor rays at the paraxial exit pupil (plt_lens_pupils) instead of the rear
    clear aperture: same lens, many more rays reach the scene."""
    import torch
    plt = gpu_lib
    cfg = C.CONFIGS["C3_DOF"]
    lens = plt.Lens(C.lens_text("C3_DOF"), **cfg["opts"])
    pp = lens.pupils()
    fr = {}
    for key, pupil in (("rear", None), ("exit", (pp["exit_z_mm"], 1.1 * pp["exit_r_mm"]))):
        n = cfg["width_px"] * cfg["height_px"] * 16
        d = plt.rays_to_device(R.gen_rays(C.dof_law(0.0, 16, pupil), cfg["seed"], 0, n))
        h = plt.alloc_hits(n)
        plt.trace_rays(lens, lens.all_t_id(), d, h, direction=plt.BACKWARD)
        torch.cuda.synchronize()
        fr[key] = float(unpack_mask(h["mask_bits"].cpu().numpy(), n).mean())
    print(fr)
    assert fr["exit"] > 5 * fr["rear"] and fr["exit"] > 0.5


def test_pupil_weights_make_sampling_strategies_agree(gpu_lib):
    """With the Eq. 9 pupil-sampling weights (render_dof(pupil_disc=...)), rays aimed at the
    rear clear aperture and rays aimed at 1.2x the paraxial exit pupil estimate the SAME
    image (the pixel integral), although their ray averages differ several-fold."""
    import torch
    from paper_2605_04017_b200.render import render_dof
    plt = gpu_lib
    cfg = C.CONFIGS["C3_DOF"]
    lens = plt.Lens(C.lens_text("C3_DOF"), **cfg["opts"])
    pp = lens.pupils()
    law0 = C.dof_law(0.0, 64)
    px = cfg["width_px"] * cfg["height_px"]
    imgs = {}
    for key, disc in (("rear", (law0["pupil_z"], law0["pupil_r"])),
                      ("exit", (pp["exit_z_mm"], 1.2 * pp["exit_r_mm"]))):
        n = px * 64
        d = plt.rays_to_device(R.gen_rays(C.dof_law(0.0, 64, disc), cfg["seed"], 0, n))
        fw, fu = (torch.zeros(px, dtype=torch.int64, device="cuda") for _ in range(2))
        render_dof(lens, d, cfg["scene"], fw, 64, cfg["opts"]["backward_exit_z_mm"], weight_scale=1.0 / 64,
                   pupil_disc=disc)
        render_dof(lens, d, cfg["scene"], fu, 64, cfg["opts"]["backward_exit_z_mm"], weight_scale=1.0 / 64)
        torch.cuda.synchronize()
        imgs[key] = (fw.cpu().numpy().astype(np.float64), fu.cpu().numpy().astype(np.float64))
    (wr, ur), (we, ue) = imgs["rear"], imgs["exit"]
    ratio_w, ratio_u = we.sum() / wr.sum(), ue.sum() / ur.sum()
    # 16x16-pixel bins: the weighted images agree to Monte-Carlo noise (the rear-aperture
    # rays are only ~7 % valid: ~1,200 valid rays per bin)
    b = lambda f: f.reshape(cfg["height_px"] // 16, 16, cfg["width_px"] // 16, 16).sum((1, 3))
    rel = np.abs(b(we) - b(wr)).sum() / b(wr).sum()
    print({"weighted_energy_ratio": ratio_w, "unweighted_energy_ratio": ratio_u, "rel_l1_bin16": rel})
    assert abs(ratio_w - 1.0) < 0.03 and abs(ratio_u - 1.0) > 0.5
    assert rel < 0.05


CARDS = [{"z_mm": -400.0, "period_mm": 8.0, "contrast": 0.2, "x0_mm": -60.0, "x1_mm": 0.0, "y0_mm": -40.0,
          "y1_mm": 40.0},
         {"z_mm": -1000.0, "period_mm": 20.0, "contrast": 0.1, "x0_mm": -200.0, "x1_mm": 200.0, "y0_mm": -150.0,
          "y1_mm": 150.0},
         {"z_mm": -2500.0, "period_mm": 60.0, "contrast": 0.4, "x0_mm": 0.0, "x1_mm": 900.0, "y0_mm": -600.0,
          "y1_mm": 600.0}]


@pytest.mark.parametrize("weighted", [False, True])
def test_shade_cards_bit_exact_on_trace_hits(gpu_lib, weighted):
    """plt_shade_cards (scene of three cards at 0.4 / 1 / 2.5 m, partly overlapping, plus
    background) on backward trace hits of the 24 mm camera: bit-identical to the oracle."""
    import torch
    plt = gpu_lib
    cfg = C.CONFIGS["C3_DOF"]
    lens = plt.Lens(C.lens_text("C3_DOF"), **cfg["opts"])
    pp = lens.pupils()
    spp = 16
    n = cfg["width_px"] * cfg["height_px"] * spp
    d = plt.rays_to_device(R.gen_rays(C.dof_law(0.0, spp, (pp["exit_z_mm"], 1.1 * pp["exit_r_mm"])), 9, 0, n))
    h = plt.alloc_hits(n)
    plt.trace_rays(lens, lens.all_t_id(), d, h, direction=plt.BACKWARD)
    px = cfg["width_px"] * cfg["height_px"]
    film = torch.zeros(px, dtype=torch.int64, device="cuda")
    in_dz = d["dz"] if weighted else None
    plt.shade_cards(CARDS, 0.05, cfg["opts"]["backward_exit_z_mm"], h, film, spp, weight_scale=1.0 / spp,
                    in_dz=in_dz)
    torch.cuda.synchronize()
    hh = {k: h[k].cpu().numpy() for k in plt.HIT_KEYS}
    valid = unpack_mask(h["mask_bits"].cpu().numpy(), n)
    ref = oracle.shade_cards(CARDS, 0.05, cfg["opts"]["backward_exit_z_mm"], valid, hh["px"], hh["py"], hh["dx"],
                             hh["dy"], hh["dz"], hh["throughput"], spp=spp, pixels=px, scale=1.0 / spp,
                             in_dz=None if in_dz is None else in_dz.cpu().numpy())
    assert valid.mean() > 0.3
    assert np.array_equal(film.cpu().numpy(), ref)
    assert len(np.unique(ref)) > 100          # cards, checkers and background all present
