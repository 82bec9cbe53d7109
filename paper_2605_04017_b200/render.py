"""Forward flare rendering (Listing 1; Eq. 8).

For every transport path P of the lens (the ghosts of §4.2) and every colour
channel, the rays of that channel are pushed through P -- by the path's factorised map
when one is given (eval_map), otherwise by the exact trace -- and the valid exit rays are
splatted into an int64 film inside the same kernel (plt_*_splat).  The film is the exact
integer sum of all contributions, so the image does not depend on the order of paths,
channels or GPUs.  Orchestration only: every step runs in the library's kernels.
"""
from __future__ import annotations

from . import BACKWARD, FP32, FP64, eval_map, propagate_rays, shade_plane, splat_sensor, trace_paths, trace_rays


def render_flare(lens, path_ids, channel_rays, film_desc: dict, film, maps: dict | None = None,
                 precision: int = FP64, weight_scale: float = 1.0, direction: int = 0, per_path: dict | None = None,
                 stream=None, hits=None, side_streams: int = 2):
    """Accumulate the flare image of `path_ids` into `film` (device int64, C*H*W, not cleared;
    may be None when per_path is given).

    channel_rays: list (one per film channel) of device ray dicts (plt_inputs layout);
    maps: {path_id: Map} -- paths in it are evaluated by the network, the others traced
    (precision: PLT_FP64 is binding for ghosts, A22); per_path: optional
    {path_id: film tensor} receiving each path's own contribution instead of `film`
    (for per-path comparisons); hits: optional scratch hits dict of >= max rays.
    side_streams: the (path, channel) launches are independent -- exact int64 atomics into
    one film, order-free -- so they go round-robin over this many streams forked from
    `stream` (each with its own hit buffer; one launch's tail overlaps the next one's
    start: 9-10 % faster images, bit-identical films); 1 = all on `stream`.
    Returns the list of (path_id, "map" | "trace") actually used.
    """
    import torch
    from . import alloc_hits
    used = []
    dev = channel_rays[0]["ox"].device
    nmax = max(int(r["ox"].numel()) for r in channel_rays)
    h = hits if hits is not None else alloc_hits(nmax, device=dev)
    chan = [torch.full((int(r["ox"].numel()),), c, dtype=torch.uint8, device=dev)
            for c, r in enumerate(channel_rays)]
    base = stream if stream is not None else torch.cuda.current_stream(dev)
    k = max(1, int(side_streams))
    sides = [torch.cuda.Stream(device=dev) for _ in range(k)] if k > 1 else [base]
    hs = [h] + [alloc_hits(nmax, device=dev) for _ in range(len(sides) - 1)]
    if len(sides) > 1:
        fork = torch.cuda.Event()
        fork.record(base)
        for sd in sides:
            sd.wait_event(fork)
    j = 0
    # traced paths that all splat into `film`: one plt_trace_paths call per channel (in
    # float64 their common all-T prefix is traced once; same film bit for bit)
    # (per_path films: the shared trace writes every path's hits, then one plt_splat_sensor per
    # path and channel -- the film the fused splat would give, bit for bit)
    traced = [int(p) for p in path_ids if not (maps and maps.get(int(p)) is not None)]
    shared = len(traced) > 1
    if shared:
        ph = [alloc_hits(nmax, device=dev) for _ in traced] if per_path is not None else None
        for c, rays in enumerate(channel_rays):
            n = int(rays["ox"].numel())
            sd, hh = sides[j % len(sides)], hs[j % len(sides)]
            j += 1
            if per_path is None:
                spl = {"film_desc": film_desc, "film": film, "channel": chan[c], "weight_scale": weight_scale}
                trace_paths(lens, traced, rays, [hh] * len(traced), direction=direction, precision=precision, n=n,
                            stream=sd, splat=spl)
                continue
            trace_paths(lens, traced, rays, ph, direction=direction, precision=precision, n=n, stream=sd)
            for pid, hp in zip(traced, ph):
                splat_sensor(film_desc, per_path[pid], hp, channel=chan[c], weight_scale=weight_scale, n=n, stream=sd)
            if len(sides) > 1:   # the next channel may run on another stream: it reuses ph
                e = torch.cuda.Event()
                e.record(sd)
                sides[j % len(sides)].wait_event(e)
    for pid in path_ids:
        target = per_path[pid] if per_path is not None else film
        m = maps.get(int(pid)) if maps else None
        if m is None and shared:
            used.append((int(pid), "trace"))
            continue
        for c, rays in enumerate(channel_rays):
            n = int(rays["ox"].numel())
            sd, hh = sides[j % len(sides)], hs[j % len(sides)]
            j += 1
            spl = {"film_desc": film_desc, "film": target, "channel": chan[c], "weight_scale": weight_scale}
            if m is not None:
                eval_map(m, rays, hh, n=n, stream=sd, splat=spl)
            else:
                trace_rays(lens, int(pid), rays, hh, direction=direction, precision=precision, n=n, stream=sd,
                           splat=spl)
        used.append((int(pid), "map" if m is not None else "trace"))
    if len(sides) > 1:   # the caller's stream continues after every launch
        for sd in sides:
            e = torch.cuda.Event()
            e.record(sd)
            base.wait_event(e)
        # buffers used on the side streams stay reserved until those streams' work is done
        extra = [t for hh in (ph or []) for t in hh.values() if torch.is_tensor(t)] if shared else []
        for sd in sides:
            for t in [t for hh in hs for t in hh.values() if torch.is_tensor(t)] + chan + extra:
                t.record_stream(sd)
    return used


def render_dof(lens, rays: dict, scene: dict, film, spp: int, z_exit_mm: float, m=None, map_plane_z: float | None = None,
               weight_scale: float = 1.0, hits=None, scratch_rays=None, stream=None, pupil_disc: tuple | None = None):
    """Backward depth-of-field image (the camera integrator of
    P:422-427, Eq. 9): pixel-stratified sensor rays (e.g. the sensor_grid law, ray i in
    pixel i // spp) go through the lens -- by the exact all-T trace, or by the map `m`
    after free-space propagation to the map's input plane `map_plane_z` (focusing by a
    sensor shift needs no retraining) -- and their exit rays (on z = z_exit_mm,
    the lens's backward exit plane) are shaded on the checkerboard scene plane into `film`
    (device int64, one entry per pixel, not cleared).  pupil_disc = (z_mm, radius_mm) of
    the disc the sensor rays' directions were sampled through (e.g. the exit pupil of
    plt_lens_pupils): each ray then carries the Eq. 9 estimator weight
    (pi r^2 / dz^2) cos^4(theta) (plt_shade_plane_weighted), making the image an unbiased
    estimate of the pixel integral rather than of the ray average.
    """
    from . import alloc_hits
    import torch
    n = int(rays["ox"].numel())
    h = hits if hits is not None else alloc_hits(n, device=rays["ox"].device)
    if m is None:
        trace_rays(lens, lens.all_t_id(), rays, h, direction=BACKWARD, precision=FP32, stream=stream)
    else:
        src = rays
        if map_plane_z is not None and float(map_plane_z) != float(rays["plane_z"]):
            # rays without dz (A32) keep that form: the scratch gets no dz array either
            dst = scratch_rays if scratch_rays is not None else {
                k: (torch.empty_like(rays[k]) if rays.get(k) is not None else None)
                for k in ("ox", "oy", "dx", "dy", "dz", "lambda_nm")}
            propagate_rays(rays, dst, map_plane_z, direction=BACKWARD, stream=stream)
            src = dst
        eval_map(m, src, h, stream=stream)
    in_dz = None
    if pupil_disc is not None:
        if rays.get("dz") is None:
            raise ValueError("pupil weighting needs the sensor rays' dz")
        from . import pupil_weight
        weight_scale = weight_scale * pupil_weight(rays["plane_z"], pupil_disc[0], pupil_disc[1])
        in_dz = rays["dz"]
    if "cards" in scene:   # several cards at different depths (plt_shade_cards)
        from . import shade_cards
        shade_cards(scene["cards"], scene.get("background", 0.0), z_exit_mm, h, film, spp, weight_scale=weight_scale,
                    n=n, stream=stream, in_dz=in_dz)
    else:
        shade_plane(scene, z_exit_mm, h, film, spp, weight_scale=weight_scale, n=n, stream=stream, in_dz=in_dz)


def path_energies(lens, path_ids, rays, direction: int = 0, precision: int = FP64, stream=None, hits=None):
    """Flux each path carries for the ray batch `rays` (higher-order
    ghost pruning on the GPU).  Every path is traced and its valid hits are splatted, in
    the trace kernel, into a ONE-pixel film covering the whole output plane: the film entry
    is the exact int64 sum of llrint(I * |w_z| * 2^32) over the path's valid rays (Eq. 8
    with G = |w_z|, weight scale 1), so energies are deterministic and need no extra kernel.
    Returns a list of floats (sum of I |w_z| per path, same order as path_ids); one
    device-to-host copy at the end."""
    import torch
    from . import alloc_hits
    dev = rays["ox"].device
    n = int(rays["ox"].numel())
    h = hits if hits is not None else alloc_hits(n, device=dev)
    films = torch.zeros(len(path_ids), dtype=torch.int64, device=dev)
    whole = {"width_px": 1, "height_px": 1, "channels": 1, "sensor_w_mm": 1e9, "sensor_h_mm": 1e9}
    for k, pid in enumerate(path_ids):
        trace_rays(lens, int(pid), rays, h, direction=direction, precision=precision, n=n, stream=stream,
                   splat={"film_desc": whole, "film": films[k:k + 1], "weight_scale": 1.0})
    return [float(v) / 4294967296.0 for v in films.cpu().tolist()]


def prune_paths(lens, path_ids, rays, min_fraction: float, direction: int = 0, precision: int = FP64,
                stream=None):
    """Keep the paths whose measured flux (path_energies) is at least `min_fraction` of the
    all-transmission path's flux on the same rays -- the GPU counterpart of the host's
    normal-incidence prune (plt_enumerate_ghosts min_throughput), measured on real rays
    through real apertures instead of one paraxial ray.  Returns (kept ids, energies dict)."""
    ids = [int(p) for p in path_ids]
    all_t = lens.all_t_id()
    e = path_energies(lens, [all_t] + ids, rays, direction, precision, stream)
    ref = e[0]
    energies = dict(zip(ids, e[1:]))
    return [p for p in ids if ref > 0 and energies[p] >= min_fraction * ref], energies
