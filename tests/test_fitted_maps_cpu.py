"""CPU checks of the map-blob writer and the committed fitted maps (maps/*.pltmap):
well-formed PLTMAP01 blobs with the architecture of PAPER.md:391-392, consistent with
their lens, loadable through the C-ABI without a GPU."""
import glob
import os

import numpy as np
import pytest

import oracle
from plt_inputs import configs as C
from plt_inputs import rays as R

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
MAPS = sorted(glob.glob(os.path.join(ROOT, "maps", "*.pltmap")))


def test_writer_round_trips_a_parsed_blob():
    nm = C.CONFIGS["C2"]["map_norm"]
    for plane in (None, -5.0):
        blob = R.make_map_blob(1024, 0, 77, nm["in_lo"], nm["in_hi"], nm["out_mid"], nm["out_half"], plane_z=plane)
        p = oracle.parse_map_blob(blob)
        assert p["version"] == (1 if plane is None else 2) and p["plane_z"] == plane
        layers = lambda h: [(W.astype(np.float32), b.astype(np.float32)) for W, b in zip(h["W"], h["b"])]
        again = R.write_map_blob(p["path_id"], p["direction"], p["norm"][0:4], p["norm"][4:8], p["norm"][8:14],
                                 p["norm"][14:20], layers(p["classifier"]), layers(p["regressor"]), plane_z=p["plane_z"])
        assert again == blob


def test_map_plane_is_enforced_by_oracle():
    """Version-2 blobs record the input plane of their training rays: the
    oracle's map query refuses rays on another plane (the library does too, plt.h)."""
    blob = C.map_blob("C2", 1 << 10)
    assert oracle.parse_map_blob(blob)["plane_z"] == -5.0
    rays = R.gen_rays(C.CONFIGS["C2"]["law"], 3, 0, 64)
    oracle.map_eval(blob, rays)
    with pytest.raises(ValueError):
        oracle.map_eval(blob, dict(rays, plane_z=-4.0))


def test_writer_rounds_weights_to_nearest_bf16():
    W = np.array([[1.0 + 2 ** -8, 1.0 + 3 * 2 ** -9, -2.0 - 2 ** -9, 3e-3]], np.float32)  # ties -> even
    blob = R.write_map_blob(1, 0, np.zeros(4), np.ones(4), np.zeros(6), np.ones(6),
                            [(W, np.zeros(1))], [(W, np.zeros(1))])
    got = oracle.parse_map_blob(blob)["classifier"]["W"][0][0]
    assert got[0] == 1.0 and got[1] == 1.0 + 2 ** -7 and got[2] == -2.0
    assert abs(got[3] - 3e-3) <= 3e-3 * 2 ** -8


@pytest.mark.parametrize("path", MAPS, ids=[os.path.basename(p) for p in MAPS])
def test_committed_map_is_consistent(path):
    import paper_2605_04017_b200 as plt
    cfg_name, pid = os.path.basename(path)[:-7].rsplit("_", 1)
    cfg = C.CONFIGS[cfg_name]
    blob = open(path, "rb").read()
    p = oracle.parse_map_blob(blob)
    assert p["classifier"]["dims"] == list(R.CLASSIFIER_DIMS)
    assert p["regressor"]["dims"] == list(R.REGRESSOR_DIMS)
    assert p["direction"] == cfg["direction"]
    lo, hi, half = p["norm"][0:4], p["norm"][4:8], p["norm"][14:20]
    assert np.all(hi > lo) and np.all(half > 0)
    assert np.isfinite(np.concatenate([w.ravel() for h in ("classifier", "regressor") for w in p[h]["W"]])).all()
    lens = plt.Lens(C.lens_text(cfg_name), **cfg["opts"])
    want = lens.all_t_id() if int(pid) == 0 else int(pid)
    assert p["path_id"] == want
    if int(pid):
        ids, _ = lens.enumerate_ghosts(2)
        assert want in ids
    plt.Map(blob, lens=lens)      # host-side validation through the C-ABI (no GPU needed)


FLARE = sorted(glob.glob(os.path.join(ROOT, "maps", "flare", "*", "*.pltmap")))


def test_flare_maps_belong_to_their_lens():
    """maps/flare/<config>/<path id>.pltmap (tests/fit_flare_maps.py): every blob is a
    well-formed network for a two-bounce ghost of that config's lens."""
    import paper_2605_04017_b200 as plt
    if not FLARE:
        pytest.skip("no flare maps committed")
    by_cfg = {}
    for path in FLARE:
        by_cfg.setdefault(os.path.basename(os.path.dirname(path)), []).append(path)
    for cfg_name, paths in by_cfg.items():
        cfg = C.CONFIGS[cfg_name]
        lens = plt.Lens(C.lens_text(cfg_name), **cfg["opts"])
        ids, _ = lens.enumerate_ghosts(2)
        ghosts = set(int(i) for i in ids) - {lens.all_t_id()}
        for path in paths:
            p = oracle.parse_map_blob(open(path, "rb").read())
            assert p["path_id"] == int(os.path.basename(path)[:-7]) and p["path_id"] in ghosts
            assert p["classifier"]["dims"] == list(R.CLASSIFIER_DIMS)
            assert p["regressor"]["dims"] == list(R.REGRESSOR_DIMS)
