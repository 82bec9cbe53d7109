#!/usr/bin/env python3
"""Benchmark of the batched per-ray lens transport query on B200 (one process per GPU).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl plt|reference]

One STEP = one pass of the whole hot path over one batch of the
workload; by default the C2 workload (BASELINE.json configs[1]: 50 mm double-Gauss,
2^24 rays per GPU, lambda uniform 400-700 nm, synthetic seeded rays):
  a8  enumerate_ghosts (host; lists the lens's transport paths)
  a6-a7 trace_rays  -- exact sequential all-T trace (fp32 + fp64 guard-band refine)
  a1-a5 eval_map    -- fused classifier-gated regressor (tcgen05/TMEM)
  a9  splat_sensor  -- both results splatted into an int64 film (768x512, 36x24 mm); by
        default fused into the trace / regressor epilogues (plt_*_splat, bit-identical
        film); --splat separate runs plt_splat_sensor on the hits instead
  a10 film all-reduce over NCCL (N > 1)
Every ray is queried both ways, so value = rays per step (all ranks) / step time.
Scaling is weak: each rank owns its own chunk-aligned slice of the global index range.

--config selects the other BASELINE.json workloads (SURVEY.md §8(e) partitioning):
  C3     805,306,368 backward camera rays (192x128 px x 32768 spp), generated on the
         device; strong scaling, each rank owns 128/N pixel rows; trace + map.
  C4_22 / C4_59  flare image: every ghost x 3 channels x 2^20 rays, fp64 trace + per-ghost
         map, splatted in-kernel; strong scaling over contiguous (channel, ghost, ray)
         ranges, one NCCL int64 film all-reduce per image.
  C5     the throughput sweep (--rays 2^20 .. 2^30 per GPU, device-generated), as C2.

Rank 0 prints ONE JSON line.  `--impl reference` times the float64 CPU oracle
(oracle/, test infrastructure) on the host cores over a bounded sample instead.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "M rays/s lens-map eval & exact trace"
UNIT = "M rays/s"
FILM = {"width_px": 768, "height_px": 512, "channels": 1, "sensor_w_mm": 36.0, "sensor_h_mm": 24.0,
        "center_x_mm": 0.0, "center_y_mm": 0.0}
TANH_PER_RAY_CLS, TANH_PER_RAY_REG = 64, 160      # 2x32 classifier, 5x32 regressor hidden units
MAC_CLS, MAC_REG = 4 * 32 + 32 * 32 + 32, 4 * 32 + 4 * 32 * 32 + 32 * 6
IO_BYTES_PER_RAY = 5 * 4 + 6 * 4 + 1.0 / 8        # SoA in (ox oy dx dy lambda) + SoA out + 1 mask bit
MUFU_PER_CLK_PER_SM = 16                           # B200 nominal SFU rate (DESIGN.md roofline)
FP32_LANES_PER_SM = 128                            # FFMA lanes per SM (DESIGN.md roofline)


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    """SM clock + throttle reasons sampled every ~5 ms (NVML) while the timed region runs.

    Samples are kept only between mark_start() and mark_stop() (host wall clock around the
    device-timed region), so the reported median is the clock under load."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, index: int):
        import threading
        self.index = index
        self.samples = []          # (t, sm_mhz, reasons_mask)
        self.t0 = self.t1 = None
        self.stop_ev = threading.Event()
        self.thread = None
        self.ok = False
        self.max_mhz = None

    def _run(self, h, nv):
        while not self.stop_ev.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                try:
                    rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                except Exception:
                    rs = nv.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                self.samples.append((time.perf_counter(), sm, rs))
            except Exception:
                pass
            time.sleep(0.005)

    def start(self):
        import threading
        try:
            import pynvml as nv
            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            return
        self.thread = threading.Thread(target=self._run, args=(h, nv), daemon=True)
        self.thread.start()

    def mark_start(self):
        self.t0 = time.perf_counter()

    def mark_stop(self):
        self.t1 = time.perf_counter()

    def stop(self) -> dict:
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"], "samples": 0}
        self.stop_ev.set()
        self.thread.join(timeout=2)
        inside = [x for x in self.samples if self.t0 is not None and self.t0 <= x[0] <= (self.t1 or 1e30)]
        use = inside or self.samples
        reasons = sorted({k for _, _, rs in use for k, bit in self.REASONS.items() if rs & bit})
        return {"sm_mhz": float(np.median([x[1] for x in use])) if use else None,
                "sm_max_mhz": float(self.max_mhz), "reasons": reasons, "samples": len(inside)}


# ---------------------------------------------------------------------------------------
def bind_numa_local(dev: int) -> str:
    """Pin this process to the CPU cores NVML reports as closest to GPU `dev` (its NUMA
    node), so the pinned host buffers of the e2e leg are first-touched in that node's memory
    and each rank's host->device copies of a multi-GPU run use the local socket's memory
    bandwidth.  Best effort: returns a note, never raises."""
    try:
        import pynvml
        import torch
        pr = torch.cuda.get_device_properties(dev)
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByPciBusId(f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0")
        words = pynvml.nvmlDeviceGetCpuAffinity(h, (os.cpu_count() + 63) // 64)
        cpus = {64 * i + b for i, w in enumerate(words) for b in range(64) if (w >> b) & 1}
        cpus &= set(os.sched_getaffinity(0))   # within the cores this process may use
        if not cpus:
            return "cpu affinity unchanged (no GPU-local core available)"
        os.sched_setaffinity(0, cpus)
        return f"bound to the {len(cpus)} cores local to the GPU"
    except Exception as ex:   # no NVML / no affinity support: keep the default placement
        return f"cpu affinity unchanged ({type(ex).__name__})"


def dist_setup(args):
    import torch
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # functional-test knob only (never for timing): PLT_BENCH_SHARE_GPU=1 maps every rank
    # onto the visible GPUs round-robin and uses gloo, so the multi-rank code path can be
    # exercised on a one-GPU box (the ranks' kernels never wait on each other)
    share = os.environ.get("PLT_BENCH_SHARE_GPU") == "1"
    if args.impl == "plt":
        if share:
            local = local % torch.cuda.device_count()
        torch.cuda.set_device(local)
        if not share and ws > 1:   # N = 1 keeps every core (the oracle baseline uses them)
            args.numa = bind_numa_local(local)
    if ws > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        nccl = args.impl == "plt" and not share
        if nccl:   # the communicator's init lines (rank count, NVLS/ring choice) go to stderr
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist.init_process_group("nccl" if nccl else "gloo",
                                device_id=torch.device("cuda", local) if nccl else None)
    return ws, rank, local


def ncu_traffic(kernel: str):
    """DRAM bytes per launch of `kernel` from the newest committed ncu --set full capture
    (profiles/*_ncu_traffic.json); None if there is none.  Never runs ncu itself."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "*_ncu_traffic.json")))
    if not files:
        return None
    with open(files[-1]) as f:
        k = json.load(f)["kernels"].get(kernel)
    return None if k is None else k["dram_read"] + k["dram_write"]


def workload_config(n: int, ws: int, pid: int) -> dict:
    """The `config` object shared by both arms (same workload, metric and unit)."""
    size = f"2^{n.bit_length() - 1}" if n & (n - 1) == 0 else str(n)
    return {"workload": f"C2: 50 mm double-Gauss (Kolb/pbrt stand-in), {size} rays per GPU, lambda U[400,700] nm, "
                        "all-T trace + factorised map (fitted weights maps/C2_0.pltmap) + splat"
                        + (" + NCCL film all-reduce" if ws > 1 else ""),
            "rays_per_gpu": n, "lens": "dgauss50", "path_id": pid, "film": "768x512 int64",
            "rays": "(x, y, omega_x, omega_y, lambda) float32 SoA, omega in S^2_+ (P:180; dz completed in-kernel)",
            "l2": (f"inputs {20 * n / 1e6:.0f} MB/GPU > 126 MB L2 (no flush needed)" if 20 * n > 126e6
                   else f"inputs {20 * n / 1e6:.0f} MB/GPU fit in L2 (not a contract workload size)"),
            "parallelism": f"dp{ws} over rays"}


def make_workload(rank: int, n_per_rank: int):
    from plt_inputs import configs as C
    from plt_inputs import rays as R
    cfg = C.CONFIGS["C2"]
    rays = R.gen_rays(cfg["law"], cfg["seed"], rank * n_per_rank, n_per_rank)
    return cfg, unit_rays(rays)


def unit_rays(rays: dict) -> dict:
    """The workload's rays in the paper's parameterisation (omega in S^2_+): dz is not
    stored, the query completes it (include/plt.h) -- 20 B per ray on the wire and in HBM."""
    return {k: v for k, v in rays.items() if k != "dz"}


def oracle_step(olens, blob, rays, pid, threads):
    """The oracle doing one step's work on `rays`: trace + map + splat (float64 CPU)."""
    import oracle
    t = oracle.trace(olens, pid, 0, rays, threads=threads)
    m = oracle.map_eval(blob, rays, threads=threads)
    f1, _ = oracle.splat(FILM, t["valid"], t["px"], t["py"], t["dz"], t["I"], None, 1.0)
    f2, _ = oracle.splat(FILM, m["valid"], m["px"], m["py"], m["dz"], m["I"], None, 1.0)
    return f1, f2


def cpu_baseline(target_s: float = 12.0):
    """Oracle throughput on this host's cores over a bounded sample of the C2 workload:
    consecutive 2^20-ray chunks of the C2 batch until ~target_s seconds of CPU work."""
    import oracle
    from plt_inputs import configs as C
    from plt_inputs import rays as R
    cfg = C.CONFIGS["C2"]
    olens = oracle.load_lens(C.lens_text("C2"), cfg["opts"])
    pid = 1 << olens.n_optical
    blob = C.fitted_map_blob("C2")
    threads = oracle.host_threads()
    chunk = 1 << 20
    done, busy, c = 0, 0.0, 0
    while busy < target_s and c < 64:
        rays = unit_rays(R.gen_rays(cfg["law"], cfg["seed"], c * chunk, chunk))
        t0 = time.perf_counter()
        oracle_step(olens, blob, rays, pid, threads)
        busy += time.perf_counter() - t0
        done += chunk
        c += 1
    return {"value": done / busy / 1e6, "unit": UNIT, "cores": threads, "kind": "oracle",
            "sample": f"first {done} rays of the C2 batch ({c} chunks of 2^20; all-T trace + map + splat "
                      f"in float64), {busy:.1f} s of CPU time"}


# ---------------------------------------------------------------------------------------
def run_reference(args, ws, rank):
    """--impl reference: the float64 oracle, as it stands, on host cores (rank 0 only)."""
    if rank != 0:
        return
    import oracle
    from plt_inputs import configs as C
    from plt_inputs import rays as R
    cfg = C.CONFIGS["C2"]
    olens = oracle.load_lens(C.lens_text("C2"), cfg["opts"])
    pid = 1 << olens.n_optical
    blob = C.fitted_map_blob("C2")
    threads = oracle.host_threads()
    n = args.ref_rays
    rays = unit_rays(R.gen_rays(cfg["law"], cfg["seed"], 0, n))
    for _ in range(args.warmup):
        oracle_step(olens, blob, {k: (v[:4096] if k != "plane_z" else v) for k, v in rays.items()}, pid, threads)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle_step(olens, blob, rays, pid, threads)
    dt = time.perf_counter() - t0
    val = n * args.steps / dt / 1e6
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": workload_config(args.rays or (1 << 24), ws, pid),
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": threads, "kind": "oracle",
                             "sample": f"each step = the first {n} rays of the C2 batch (bounded sample of the "
                                       f"2^24 rays per GPU of the GPU arm), float64 trace + map + splat"},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------------------
CONFIGS = ("C2", "C3", "C4_22", "C4_59", "C5")
FP64_LANES_PER_SM = 64                             # B200 FP64 FMA lanes per SM (nominal; DESIGN.md roofline)


with open(os.path.join(ROOT, "profiles", "trace_flops.json")) as _f:
    _tf = json.load(_f)
TRACE_FLOPS_STEP = _tf["flops_per_step"]          # per step kind (tools/trace_flops.py)
TRACE_FLOPS_INIT = _tf["flops_per_step"]["init"]
del _tf


def flare_partition(ghosts, n_channels, npc, rank, ws):
    """SURVEY §8(e) for the flare image: the (channel, ghost, ray) sequence -- channel-major,
    so a rank's ghosts of one channel are consecutive -- cut into ws contiguous ranges.
    Returns this rank's segments [(ghost, channel, first ray, count)] and its trace groups
    [(channel, first ray, count, [ghosts])]: the segments over the same (channel, ray range),
    traced by one plt_trace_paths call (fp64: the ghosts' common all-T prefix once)."""
    total = len(ghosts) * n_channels * npc
    lo_q, hi_q = rank * total // ws, (rank + 1) * total // ws
    segs, q = [], lo_q
    while q < hi_q:
        item, i0 = divmod(q, npc)
        c, g = item // len(ghosts), ghosts[item % len(ghosts)]
        cnt = min(npc - i0, hi_q - q)
        segs.append((g, c, i0, cnt))
        q += cnt
    groups = {}
    for g, c, i0, cnt in segs:
        groups.setdefault((c, i0, cnt), []).append(g)
    return segs, [(c, i0, cnt, gs) for (c, i0, cnt), gs in groups.items()]


def trace_flops_table():
    """profiles/trace_flops.json: algorithmic FLOPs per ray per (config, path), written by
    tools/trace_flops.py from the oracle's step bookkeeping (a stored value; bench never runs
    the oracle outside its cpu_baseline / reference legs)."""
    with open(os.path.join(ROOT, "profiles", "trace_flops.json")) as f:
        return json.load(f)["configs"]


def timed_steps(step, args, dist, local, stream):
    """W untimed steps, then K steps bracketed by barrier + synchronize and CUDA events on the
    launching stream, NVML clocks sampled during the region.  Returns (seconds, clocks)."""
    import torch
    for _ in range(args.warmup):
        step(None)
    torch.cuda.synchronize()
    sampler = ClockSampler(local)
    sampler.start()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    sampler.mark_start()
    t0.record(stream)
    for k in range(args.steps):
        step(k)
    t1.record(stream)
    torch.cuda.synchronize()
    sampler.mark_stop()
    if dist is not None:
        dist.barrier()
    return t0.elapsed_time(t1) / 1e3, sampler.stop()


class Events:
    """Per-kernel-group durations inside the timed steps (CUDA events on the launching stream)."""

    def __init__(self, names, steps, stream):
        import torch
        self.names, self.stream = names, stream
        self.ev = [[torch.cuda.Event(enable_timing=True) for _ in range(len(names) + 1)] for _ in range(steps)]

    def mark(self, k, i):
        if k is not None:
            self.ev[k][i].record(self.stream)

    def per_step_ms(self):
        out = {n: 0.0 for n in self.names}
        for ev in self.ev:
            for i, n in enumerate(self.names):
                out[n] += ev[i].elapsed_time(ev[i + 1])
        return {n: v / len(self.ev) for n, v in out.items()}


def mask_valid_frac(h, n):
    w = h["mask_bits"][: (n + 31) // 32].cpu().numpy().view(np.uint32)
    bits = np.unpackbits(w.view(np.uint8), bitorder="little")[:n]
    return float(bits.sum()) / max(n, 1)


def map_roofline(rays, v, secs, sm_max):
    """eval_map: MUFU tanh roofline -- 64 classifier + 160 regressor tanh per valid ray."""
    tanh = rays * (TANH_PER_RAY_CLS + TANH_PER_RAY_REG * v)
    peak = MUFU_PER_CLK_PER_SM * 148 * sm_max * 1e6 / 1e9
    ach = tanh / secs / 1e9
    return {"bound": "alu", "achieved": ach, "peak": peak, "unit": "Gtanh/s", "frac": ach / peak,
            "peak_source": "16 MUFU/clk/SM x 148 SMs x sm_max_mhz (DESIGN.md)", "tanh_per_ray": tanh / rays}


def trace_roofline(flops, secs, sm_max, fp64=False):
    """trace_rays: algorithmic FLOPs (profiles/trace_flops.json) against the FP32 (or FP64) peak."""
    lanes = FP64_LANES_PER_SM if fp64 else FP32_LANES_PER_SM
    peak = lanes * 2 * 148 * sm_max * 1e6 / 1e12
    ach = flops / secs / 1e12
    return {"bound": "alu", "achieved": ach, "peak": peak, "unit": "TFLOP/s", "frac": ach / peak,
            "peak_source": f"{lanes} {'FP64' if fp64 else 'FP32'} lanes x 2 x 148 SMs x sm_max_mhz (DESIGN.md)"}


def run_plt(args, ws, rank, local):
    import torch
    import paper_2605_04017_b200 as plt
    from plt_inputs import configs as C
    from plt_inputs import philox as PX

    plt.load()
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream()
    dist = None
    if ws > 1:
        import torch.distributed as dist
    peaks, peaks_src = load_peaks()
    sm_max = float(peaks.get("sm_max_mhz", 1965.0))
    flops_tab = trace_flops_table()
    name = args.config
    fused = args.splat == "fused"
    e2e = None
    extra_cfg = {}
    cpu_base = None

    if name in ("C2", "C5"):
        # ---- batch workloads (weak scaling): every ray traced + mapped + splatted ----------
        n = args.rays if args.rays else (1 << 24 if name == "C2" else max(C.CONFIGS["C5"]["sizes"]))
        cfg = C.CONFIGS[name]
        lens = plt.Lens(C.lens_text(name), **cfg["opts"])
        pid = lens.all_t_id()
        m = plt.Map(C.fitted_map_blob("C2"), lens=lens)           # C5 = the C2 lens, law and plane
        if name == "C2":
            _, rays_np = make_workload(rank, n)
            keys = [k for k in plt.RAY_KEYS if k in rays_np]
            host = {k: torch.from_numpy(rays_np[k]).pin_memory() for k in keys}
            d_rays = {k: host[k].to(dev) for k in keys}
            d_rays["dz"] = None
            d_rays["plane_z"] = rays_np["plane_z"]
        else:   # device-generated (Philox), the rank's slice of the global index range
            d_rays = plt.gen_rays(PX.law_constants(cfg["law"]), cfg["seed"], rank * n, n, with_dz=False)
        h_trace, h_map = plt.alloc_hits(n, dev), plt.alloc_hits(n, dev)
        npx = FILM["channels"] * FILM["height_px"] * FILM["width_px"]
        film = torch.zeros(npx, dtype=torch.int64, device=dev)
        ev = Events(["trace_rays", "eval_map", "splat_sensor", "film_allreduce"], args.steps, stream)

        def step(k):
            lens.enumerate_ghosts(0)                                   # a8 (host)
            film.zero_()
            ev.mark(k, 0)
            spl = {"film_desc": FILM, "film": film, "weight_scale": 1.0 / n} if fused else None
            plt.trace_rays(lens, pid, d_rays, h_trace, stream=stream, splat=spl)        # a6-a7 (+a9)
            ev.mark(k, 1)
            plt.eval_map(m, d_rays, h_map, stream=stream, splat=spl)                    # a1-a5 (+a9)
            ev.mark(k, 2)
            if not fused:
                plt.splat_sensor(FILM, film, h_trace, weight_scale=1.0 / n, stream=stream)   # a9
                plt.splat_sensor(FILM, film, h_map, weight_scale=1.0 / n, stream=stream)
            ev.mark(k, 3)
            if dist is not None:
                dist.all_reduce(film)                                  # a10
            ev.mark(k, 4)

        elapsed, clocks = timed_steps(step, args, dist, local, stream)
        if name == "C2":
            e2e = e2e_query_host(args, plt, lens, pid, m, host, rays_np["plane_z"], film, n, dist, stream, dev)
        v_map, v_trace = mask_valid_frac(h_map, n), mask_valid_frac(h_trace, n)
        per = {k: v / 1e3 for k, v in ev.per_step_ms().items()}
        fl = flops_tab[name][str(pid)]["flops_per_ray"]
        kernels = {
            "trace_rays": {"ms": per["trace_rays"] * 1e3, "M_rays_s": n / per["trace_rays"] / 1e6, "valid_frac": v_trace,
                           "kernel": plt.trace_kernel(lens, pid),
                           "roofline": dict(trace_roofline(n * fl, per["trace_rays"], sm_max), flops_per_ray=fl),
                           "hbm_GBs": n * IO_BYTES_PER_RAY / per["trace_rays"] / 1e9},
            "eval_map": {"ms": per["eval_map"] * 1e3, "M_rays_s": n / per["eval_map"] / 1e6, "valid_frac": v_map,
                         "roofline": map_roofline(n, v_map, per["eval_map"], sm_max),
                         "tensor_frac": 2.0 * n * (MAC_CLS + MAC_REG * v_map) / per["eval_map"] / 1e12
                         / float(peaks["bf16_tflops"]),
                         "hbm_GBs": n * IO_BYTES_PER_RAY / per["eval_map"] / 1e9},
            "splat_sensor": {"ms": per["splat_sensor"] * 1e3,
                             "mode": "fused into trace_rays / eval_map epilogues" if fused else "separate kernel"},
            "film_allreduce": {"ms": per["film_allreduce"] * 1e3},
        }
        rays_per_rank, scaling, launches = n, "weak", 3 if fused else 5
        dtype = "f32 trace (+f64 refine), bf16xbf16->f32 map"
        if name == "C2":
            cfg_line = workload_config(n, ws, pid)
        else:
            size = f"2^{n.bit_length() - 1}" if n & (n - 1) == 0 else str(n)
            cfg_line = {"workload": f"C5: throughput sweep point, C2 lens and law, {size} rays per GPU generated on "
                                    "the device (plt_gen_rays, Philox keyed by global index), all-T trace + fitted map"
                                    " + fused splat" + (" + NCCL film all-reduce" if ws > 1 else ""),
                        "rays_per_gpu": n, "lens": "dgauss50", "path_id": pid,
                        "l2": f"inputs {20 * n / 1e6:.0f} MB/GPU" + (" > 126 MB L2" if 20 * n > 126e6 else " (fit in L2)"),
                        "parallelism": f"dp{ws} over rays"}
        if ws == 1 and not args.no_cpu_baseline and name == "C2":
            cpu_base = cpu_baseline()
    elif name == "C3":
        # ---- backward camera batch at the 32768-spp scale (strong scaling by pixel rows) ----
        cfg = C.CONFIGS[name]
        total = cfg["n"]
        rows = 128
        if rows % ws:
            raise SystemExit("C3 shards 128 pixel rows: world size must divide 128")
        n = total // ws                                   # rows/ws pixel rows x 192 px x 32768 spp
        lens = plt.Lens(C.lens_text(name), **cfg["opts"])
        pid = lens.all_t_id()
        m = plt.Map(C.fitted_map_blob("C3"), lens=lens)
        d_rays = plt.gen_rays(PX.law_constants(cfg["law"]), cfg["seed"], rank * n, n, with_dz=False)
        h_trace, h_map = plt.alloc_hits(n, dev), plt.alloc_hits(n, dev)
        ev = Events(["trace_rays", "eval_map"], args.steps, stream)

        def step(k):
            ev.mark(k, 0)
            plt.trace_rays(lens, pid, d_rays, h_trace, direction=plt.BACKWARD, stream=stream)
            ev.mark(k, 1)
            plt.eval_map(m, d_rays, h_map, stream=stream)
            ev.mark(k, 2)

        elapsed, clocks = timed_steps(step, args, dist, local, stream)
        v_map, v_trace = mask_valid_frac(h_map, n), mask_valid_frac(h_trace, n)
        per = {k: v / 1e3 for k, v in ev.per_step_ms().items()}
        fl = flops_tab[name][str(pid)]["flops_per_ray"]
        kernels = {
            "trace_rays": {"ms": per["trace_rays"] * 1e3, "M_rays_s": n / per["trace_rays"] / 1e6, "valid_frac": v_trace,
                           "kernel": plt.trace_kernel(lens, pid, plt.BACKWARD),
                           "roofline": dict(trace_roofline(n * fl, per["trace_rays"], sm_max), flops_per_ray=fl)},
            "eval_map": {"ms": per["eval_map"] * 1e3, "M_rays_s": n / per["eval_map"] / 1e6, "valid_frac": v_map,
                         "roofline": map_roofline(n, v_map, per["eval_map"], sm_max)},
        }
        rays_per_rank, scaling, launches = n, "strong", 3
        dtype = "f32 trace (+f64 refine), bf16xbf16->f32 map"
        cfg_line = {"workload": "C3: 24 mm wide-angle (Nakamura x1.0897 stand-in), backward camera batch at the "
                                "32768-spp scale: 192x128 px x 32768 spp = 805,306,368 rays generated on the device "
                                "(plt_gen_rays), all-T backward trace + fitted backward map (maps/C3_0.pltmap)",
                    "rays_total": total, "rays_per_gpu": n, "lens": "wide24", "path_id": pid,
                    "l2": f"inputs {20 * n / 1e9:.1f} GB/GPU > 126 MB L2",
                    "parallelism": f"{ws} ranks x {rows // ws} pixel rows (strong scaling)"}
    else:
        # ---- flare image: every two-bounce ghost x 3 channels x 2^20 rays (strong scaling over
        # (channel, ghost, ray) ranges), fp64 trace + per-ghost map, both splatted in-kernel,
        # one NCCL int64 film all-reduce per image (Eq. 8) --------------------------
        cfg = C.CONFIGS[name]
        lens = plt.Lens(C.lens_text(name), **cfg["opts"])
        ids, _ = lens.enumerate_ghosts(2)
        ghosts = [int(g) for g in ids[1:]]
        npc = cfg["n_per_channel"]
        fd = cfg["film"]
        maps, fitted = {}, 0
        for g in ghosts:
            path = os.path.join(ROOT, "maps", "flare", name, f"{g}.pltmap")
            if os.path.exists(path):
                maps[g] = plt.Map(open(path, "rb").read(), lens=lens)
                fitted += 1
            else:   # the few paths too rare to fit (maps/README.md): seeded weights
                maps[g] = plt.Map(C.map_blob(name, g, seed=g % 100000), lens=lens)
        K = {c: PX.law_constants(dict(cfg["law"], lam=lam)) for c, lam in enumerate(cfg["channels"])}
        chans = [plt.gen_rays(K[c], cfg["seed"] * 16 + c, 0, npc) for c in range(3)]
        chan_ids = [torch.full((npc,), c, dtype=torch.uint8, device=dev) for c in range(3)]
        total = len(ghosts) * 3 * npc
        segs, tgroups = flare_partition(ghosts, 3, npc, rank, ws)
        h = plt.alloc_hits(npc, dev)
        film = torch.zeros(fd["channels"] * fd["height_px"] * fd["width_px"], dtype=torch.int64, device=dev)
        ev = Events(["trace_rays", "eval_map", "film_allreduce"], args.steps, stream)
        # the image's (ghost, channel) launches are independent (int64 atomics into one film:
        # order-free, bit-identical), so they go round-robin over a few side streams, each with
        # its own hit buffer: one launch's tail overlaps the next one's start
        n_side = max(1, args.flare_streams)
        sides = [torch.cuda.Stream(device=dev) for _ in range(n_side)] if n_side > 1 else [stream]
        hs = [h] + [plt.alloc_hits(npc, dev) for _ in range(len(sides) - 1)]
        fork_ev = [torch.cuda.Event() for _ in range(2)]
        join_ev = [[torch.cuda.Event() for _ in sides] for _ in range(2)]

        def view(d, i0, cnt):
            return {k: (v[i0:i0 + cnt] if k != "plane_z" and v is not None else v) for k, v in d.items()}

        def fan_out(phase, launch, items):
            if len(sides) > 1:
                fork_ev[phase].record(stream)
                for sd in sides:
                    sd.wait_event(fork_ev[phase])
            for j, seg in enumerate(items):
                launch(seg, sides[j % len(sides)], hs[j % len(sides)])
            if len(sides) > 1:
                for sd, e in zip(sides, join_ev[phase]):
                    e.record(sd)
                    stream.wait_event(e)

        def step(k):
            film.zero_()
            ev.mark(k, 0)

            def tr(grp, sd, hh):
                c, i0, cnt, gs = grp
                spl = {"film_desc": fd, "film": film, "channel": chan_ids[c][i0:i0 + cnt], "weight_scale": 1.0 / npc}
                plt.trace_paths(lens, gs, view(chans[c], i0, cnt), [hh] * len(gs), precision=plt.FP64, n=cnt,
                                stream=sd, splat=spl)

            def mp(seg, sd, hh):
                g, c, i0, cnt = seg
                spl = {"film_desc": fd, "film": film, "channel": chan_ids[c][i0:i0 + cnt], "weight_scale": 1.0 / npc}
                plt.eval_map(maps[g], view(chans[c], i0, cnt), hh, n=cnt, stream=sd, splat=spl)
            fan_out(0, tr, tgroups)
            ev.mark(k, 1)
            fan_out(1, mp, segs)
            ev.mark(k, 2)
            if dist is not None:
                dist.all_reduce(film)
            ev.mark(k, 3)

        elapsed, clocks = timed_steps(step, args, dist, local, stream)
        if args.dump_film and rank == 0:
            np.save(args.dump_film, film.cpu().numpy())
        per = {k: v / 1e3 for k, v in ev.per_step_ms().items()}
        n = sum(cnt for *_, cnt in segs)
        # algorithmic FLOPs of the shared-prefix trace (plt_trace_paths): per group, the all-T
        # prefix up to the deepest first reflection once per ray, plus every ghost's own steps
        # from its first reflection on (profiles/trace_flops.json, tools/trace_flops.py)
        tab, allt = flops_tab[name], flops_tab[name][str(int(ids[0]))]
        fl = 0.0
        for c, i0, cnt, gs in tgroups:
            dmax = max(tab[str(g)]["first_R_step"] for g in gs)
            pre = TRACE_FLOPS_INIT + sum(a * TRACE_FLOPS_STEP[kd] for a, kd in
                                         list(zip(allt["alive_before_step"], allt["steps"]))[:dmax])
            fl += cnt * (pre + sum(tab[str(g)]["suffix_flops_per_ray"] for g in gs))
        # valid fraction of this rank's map queries (for the tanh count): re-run outside the timing
        vm_rays = 0
        for g, c, i0, cnt in segs:
            plt.eval_map(maps[g], view(chans[c], i0, cnt), h, n=cnt, stream=stream)
            vm_rays += mask_valid_frac(h, cnt) * cnt
        v_map = vm_rays / max(n, 1)
        kernels = {
            "trace_rays": {"ms": per["trace_rays"] * 1e3, "M_rays_s": n / per["trace_rays"] / 1e6,
                           "precision": "fp64 (binding for ghosts, A22)", "call": "plt_trace_paths per channel",
                           "roofline": dict(trace_roofline(fl, per["trace_rays"], sm_max, fp64=True),
                                            flops_per_ray=fl / max(n, 1))},
            "eval_map": {"ms": per["eval_map"] * 1e3, "M_rays_s": n / per["eval_map"] / 1e6, "valid_frac": v_map,
                         "roofline": map_roofline(n, v_map, per["eval_map"], sm_max)},
            "film_allreduce": {"ms": per["film_allreduce"] * 1e3, "bytes": film.numel() * 8},
        }
        # per trace group: the prefix kernel + (zero-fill, resume) per ghost; one eval_map per segment
        rays_per_rank, scaling, launches = n, "strong", sum(1 + 2 * len(gs) for *_, gs in tgroups) + len(segs)
        dtype = "f64 trace, bf16xbf16->f32 map"
        cfg_line = {"workload": f"{name}: {'22 mm Nakamura @15 deg' if name == 'C4_22' else '59 mm double-Gauss @10 deg'} "
                                f"flare image, {len(ghosts)} two-bounce ghosts x 3 channels x 2^20 rays "
                                f"= {total:,} queries, each traced (fp64; plt_trace_paths: the ghosts' common all-T "
                                f"prefix traced once per channel) and mapped ({fitted} fitted per-ghost maps, "
                                f"{len(ghosts) - fitted} seeded), splatted in-kernel into a 768x512x3 int64 film"
                                + (", one NCCL film all-reduce per image" if ws > 1 else ""),
                    "rays_total": total, "rays_per_gpu": n, "lens": cfg["lens"], "ghosts": len(ghosts),
                    "l2": "rays 3 x 2^20 x 24 B = 75 MB, re-read per ghost (L2-resident by design)",
                    "parallelism": f"{ws} ranks x contiguous (channel, ghost, ray) ranges (strong scaling)"}
        extra_cfg["segments_rank0"] = len(segs)

    # ---- one JSON line (max over ranks) ------------------------------------------------------
    step_s = elapsed / args.steps
    vals = torch.tensor([step_s, e2e["s"] if e2e else 0.0], dtype=torch.float64, device=dev)
    if dist is not None:
        dist.all_reduce(vals, op=dist.ReduceOp.MAX)
    step_s, e2e_s = vals.tolist()
    if rank != 0:
        return
    dominant = max((k for k in kernels if "roofline" in kernels[k]), key=lambda k: kernels[k]["ms"])
    roof = dict(kernels[dominant]["roofline"])
    roof["kernel"] = dominant
    roof["traffic"] = ncu_traffic(dominant) if name == "C2" else None
    rays_all = rays_per_rank * ws if scaling == "weak" else (cfg_line.get("rays_total") or rays_per_rank * ws)
    line = {
        "metric": METRIC, "value": rays_all / step_s / 1e6, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": step_s * 1e3, "higher_is_better": True, "scaling": scaling,
        "vs_baseline": None, "dtype": dtype, "data": "synthetic",
        "config": dict(cfg_line, name=name, **extra_cfg,
                       **({"host_affinity": args.numa} if getattr(args, "numa", None) else {})),
        "roofline": roof,
        "kernels": kernels,
        "e2e": ({"value": rays_all / e2e_s / 1e6, "unit": UNIT, "h2d_bytes_per_step": e2e["h2d"],
                 "d2h_bytes_per_step": e2e["d2h"], "path": "plt_query_host (C-ABI, host buffers)",
                 "h2d_GBs": e2e["h2d"] / e2e_s / 1e9, "pinned_h2d_GBs_measured": e2e["h2d_peak"],
                 "frac_of_pinned_h2d": e2e["h2d"] / e2e_s / 1e9 / e2e["h2d_peak"]} if e2e else
                {"value": None, "note": "inputs are generated on the device for this config (plt_gen_rays)"}),
        "gpu_launches": args.steps * launches,
        "clocks": clocks,
        "peaks_source": peaks_src,
    }
    if cpu_base is not None:
        line["cpu_baseline"] = cpu_base
    print(json.dumps(line), flush=True)


def pinned_h2d_gbs(dev, nbytes=1 << 30):
    """Measured host->device bandwidth from pinned memory: the best of 5 trials of one 1 GiB
    copy and of 16 back-to-back 64 MiB copies (a single trial of one form varies by ~7 %)."""
    import torch
    src = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    dst = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    best = 0.0
    for parts in (1, 16):
        step = nbytes // parts
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for k in range(parts):
                dst[k * step:(k + 1) * step].copy_(src[k * step:(k + 1) * step], non_blocking=True)
            b.record()
            torch.cuda.synchronize()
            best = max(best, nbytes / (a.elapsed_time(b) / 1e3) / 1e9)
    return best


def e2e_query_host(args, plt, lens, pid, m, host, plane_z, film, n, dist, stream, dev):
    """The same step end to end through the C-ABI host-buffer call plt_query_host: the rays'
    host -> device copies (chunked, on the library's copy stream, overlapping the kernels),
    trace + map + fused splat, and the film back to pinned host memory, every step."""
    import torch
    fused = args.splat == "fused"
    host_rays = dict(host, plane_z=plane_z)
    film_host = torch.empty(film.numel(), dtype=torch.int64).pin_memory()
    steps = max(3, min(args.steps, 10))

    def e2e_step():
        lens.enumerate_ghosts(0)
        film.zero_()
        plt.query_host(lens, pid, m, host_rays, FILM, film, None if dist is not None else film_host,
                       weight_scale=1.0 / n, chunk=args.e2e_chunk, stream=stream)
        if dist is not None:
            dist.all_reduce(film)
            film_host.copy_(film, non_blocking=True)

    if not fused:
        return None
    e2e_step()
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        e2e_step()
    e1.record(stream)
    torch.cuda.synchronize()
    h2d = sum(int(v.numel()) * 4 for k, v in host.items() if k != "plane_z")
    return {"s": e0.elapsed_time(e1) / 1e3 / steps, "h2d": h2d, "d2h": film.numel() * 8,
            "h2d_peak": pinned_h2d_gbs(dev)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["plt", "reference"], default="plt")
    ap.add_argument("--config", choices=CONFIGS, default="C2",
                    help="BASELINE.json workload: C2 (default, the N=1 headline), C3, C4_22, C4_59, C5")
    ap.add_argument("--rays", type=int, default=0, help="rays per GPU per step (C2: 2^24, C5: 2^30 by default)")
    ap.add_argument("--dump-film", default=None, help="(C4) save rank 0's final film (.npy) -- for tests")
    ap.add_argument("--flare-streams", type=int, default=2,
                    help="(C4) side streams the image's independent (ghost, channel) launches go round-robin over")
    ap.add_argument("--ref-rays", type=int, default=1 << 15, help="rays per oracle step (--impl reference)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-chunk", type=int, default=1 << 21, help="rays per H2D chunk of the e2e leg")
    ap.add_argument("--splat", choices=["fused", "separate"], default="fused",
                    help="splat in the query kernels' epilogues (default) or as a separate kernel")
    args = ap.parse_args()
    ws, rank, local = dist_setup(args)
    try:
        if args.impl == "reference":
            run_reference(args, ws, rank)
        else:
            run_plt(args, ws, rank, local)
    finally:
        if ws > 1:
            import torch.distributed as dist
            if dist.is_initialized():
                dist.destroy_process_group()


if __name__ == "__main__":
    main()
