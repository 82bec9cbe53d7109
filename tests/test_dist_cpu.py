"""Multi-rank host logic on CPU (gloo, world size 2): chunk-aligned ray sharding is
identical to the unsharded batch, and the int64 film all-reduce of per-rank splats
equals the single-process film bit for bit (the exchange step of SURVEY §8(e))."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

FILM = {"width_px": 96, "height_px": 64, "channels": 1, "sensor_w_mm": 36.0, "sensor_h_mm": 24.0,
        "center_x_mm": 0.0, "center_y_mm": 0.0}
N_PER_RANK = 1 << 12


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _film_for(rank, n):
    import sys
    sys.path.insert(0, ROOT)
    import oracle
    import bench
    from plt_inputs import configs as C
    cfg, rays = bench.make_workload(rank, n)
    lens = oracle.load_lens(C.lens_text("C2"), cfg["opts"])
    t = oracle.trace(lens, 1 << lens.n_optical, 0, rays)
    film, _ = oracle.splat(FILM, t["valid"], t["px"].astype(np.float32), t["py"].astype(np.float32),
                           t["dz"].astype(np.float32), t["I"].astype(np.float32), None, 1.0 / n)
    return rays, film


def _worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rays, film = _film_for(rank, N_PER_RANK)
    t = torch.from_numpy(film.reshape(-1).copy())
    dist.all_reduce(t)                         # exact int64 SUM
    np.save(os.path.join(out_dir, f"film_{rank}.npy"), t.numpy())
    np.save(os.path.join(out_dir, f"ox_{rank}.npy"), rays["ox"])
    dist.barrier()
    dist.destroy_process_group()


def test_shards_union_equals_global_batch():
    import sys
    sys.path.insert(0, ROOT)
    import bench
    _, whole = bench.make_workload(0, 4 * (1 << 20))
    for ws in (2, 4):
        n = 4 * (1 << 20) // ws
        parts = [bench.make_workload(r, n)[1] for r in range(ws)]
        assert all("dz" not in p for p in parts)   # unit directions, dz completed by the query
        for k in ("ox", "dx", "lambda_nm"):
            assert np.array_equal(np.concatenate([p[k] for p in parts]), whole[k])


def test_gloo_film_allreduce_matches_single_process(tmp_path):
    port = _free_port()
    mp.spawn(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    f0 = np.load(tmp_path / "film_0.npy")
    f1 = np.load(tmp_path / "film_1.npy")
    assert np.array_equal(f0, f1)
    # single process over both shards' rays: same total film
    _, fa = _film_for(0, N_PER_RANK)
    _, fb = _film_for(1, N_PER_RANK)
    assert np.array_equal(f0, (fa + fb).reshape(-1))
    assert f0.sum() > 0
    assert not np.array_equal(np.load(tmp_path / "ox_0.npy"), np.load(tmp_path / "ox_1.npy"))


@pytest.mark.parametrize("ws", [1, 2, 3, 4, 8])
def test_flare_partition_covers_the_image_once(ws):
    """bench.flare_partition: the ranks' segments tile the (channel, ghost,
    ray) sequence exactly once, each rank's share is within one ray of total / ws, and every
    trace group is one (channel, ray range) with the ghosts of its segments."""
    import sys
    sys.path.insert(0, ROOT)
    import bench
    ghosts, nch, npc = [11, 22, 33, 44, 55], 3, 1000
    seen = np.zeros((nch, len(ghosts), npc), np.int32)
    for r in range(ws):
        segs, groups = bench.flare_partition(ghosts, nch, npc, r, ws)
        total = sum(cnt for *_, cnt in segs)
        assert abs(total - len(ghosts) * nch * npc / ws) <= 1
        for g, c, i0, cnt in segs:
            seen[c, ghosts.index(g), i0:i0 + cnt] += 1
        assert sorted((g, c, i0, cnt) for c, i0, cnt, gs in groups for g in gs) == sorted(segs)
        assert len({(c, i0, cnt) for c, i0, cnt, _ in groups}) == len(groups)
        if ws == 1:
            assert len(groups) == nch and all(gs == ghosts for *_, gs in groups)
    assert (seen == 1).all()
