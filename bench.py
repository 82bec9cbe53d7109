#!/usr/bin/env python3
"""Benchmark of the batched per-ray lens transport query on B200 (one process per GPU).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl plt|reference]

One STEP = one pass of the whole hot path over one batch of the
C2 workload (BASELINE.json configs[1]: 50 mm double-Gauss, 2^24 rays per GPU,
lambda uniform 400-700 nm, synthetic seeded rays):
  a8  enumerate_ghosts (host; lists the lens's transport paths)
  a6-a7 trace_rays  -- exact sequential all-T trace (fp32 + fp64 guard-band refine)
  a1-a5 eval_map    -- fused classifier-gated regressor (tcgen05/TMEM)
  a9  splat_sensor  -- both results splatted into an int64 film (768x512, 36x24 mm); by
        default fused into the trace / regressor epilogues (plt_*_splat, bit-identical
        film); --splat separate runs plt_splat_sensor on the hits instead
  a10 film all-reduce over NCCL (N > 1)
Every ray is queried both ways, so value = rays per step (all ranks) / step time.
Scaling is weak: each rank owns its own chunk-aligned slice of the global index range.

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
# Algorithmic FP32 FLOPs of the exact trace (counted from the O1-O8
# formulas, add/mul/div/sqrt = 1 FLOP): per spherical interaction step 77, per stop 13,
# output plane 6, input normalisation 9; weighted by the measured survival fraction at
# each step of the C2 path (rays stop costing work once vignetted).
TRACE_FLOPS_STEP, TRACE_FLOPS_STOP, TRACE_FLOPS_OUT, TRACE_FLOPS_INIT = 77, 13, 6, 9
C2_ALIVE_BEFORE_STEP = (1.0, 0.837, 0.837, 0.781, 0.781, 0.738, 0.614, 0.561, 0.498, 0.441, 0.388)  # stop = 6th
C2_ALIVE_AT_OUTPUT = 0.371


def trace_flops_per_ray_c2() -> float:
    f = TRACE_FLOPS_INIT + C2_ALIVE_AT_OUTPUT * TRACE_FLOPS_OUT
    for k, a in enumerate(C2_ALIVE_BEFORE_STEP):
        f += a * (TRACE_FLOPS_STOP if k == 5 else TRACE_FLOPS_STEP)
    return f


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
    if ws > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        nccl = args.impl == "plt" and not share
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
            "config": workload_config(args.rays, ws, pid),
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": threads, "kind": "oracle",
                             "sample": f"each step = the first {n} rays of the C2 batch (bounded sample of the "
                                       f"2^24 rays per GPU of the GPU arm), float64 trace + map + splat"},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------------------
def run_plt(args, ws, rank, local):
    import torch
    import paper_2605_04017_b200 as plt
    from plt_inputs import configs as C

    plt.load()
    fused = args.splat == "fused"
    dev = torch.device("cuda", local)
    n = args.rays
    cfg, rays_np = make_workload(rank, n)
    lens = plt.Lens(C.lens_text("C2"), **cfg["opts"])
    pid = lens.all_t_id()
    m = plt.Map(C.fitted_map_blob("C2"), lens=lens)
    stream = torch.cuda.current_stream()

    # inputs resident in HBM (device-timed value); pinned host copies for e2e
    keys = [k for k in plt.RAY_KEYS if k in rays_np]
    host = {k: torch.from_numpy(rays_np[k]).pin_memory() for k in keys}
    d_rays = {k: host[k].to(dev) for k in keys}
    d_rays["dz"] = None
    d_rays["plane_z"] = rays_np["plane_z"]
    h_trace = plt.alloc_hits(n, dev)
    h_map = plt.alloc_hits(n, dev)
    npx = FILM["channels"] * FILM["height_px"] * FILM["width_px"]
    film = torch.zeros(npx, dtype=torch.int64, device=dev)
    film_host = torch.empty(npx, dtype=torch.int64).pin_memory()
    dist = None
    if ws > 1:
        import torch.distributed as dist

    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(args.steps)]
    t_kern = {"trace_rays": 0.0, "eval_map": 0.0, "splat_sensor": 0.0, "film_allreduce": 0.0}

    def step(ev=None):
        lens.enumerate_ghosts(0)                       # a8 (host)
        film.zero_()
        if ev:
            ev[0].record(stream)
        spl = {"film_desc": FILM, "film": film, "weight_scale": 1.0 / n} if fused else None
        plt.trace_rays(lens, pid, d_rays, h_trace, stream=stream, splat=spl)          # a6-a7 (+a9 fused)
        if ev:
            ev[1].record(stream)
        plt.eval_map(m, d_rays, h_map, stream=stream, splat=spl)                      # a1-a5 (+a9 fused)
        if ev:
            ev[2].record(stream)
        if not fused:
            plt.splat_sensor(FILM, film, h_trace, weight_scale=1.0 / n, stream=stream)   # a9
            plt.splat_sensor(FILM, film, h_map, weight_scale=1.0 / n, stream=stream)
        if ev:
            ev[3].record(stream)
        if dist is not None:
            dist.all_reduce(film)                                          # a10
        if ev:
            ev[4].record(stream)

    for _ in range(args.warmup):
        step()
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
        step(evs[k])
    t1.record(stream)
    torch.cuda.synchronize()
    sampler.mark_stop()
    if dist is not None:
        dist.barrier()
    clocks = sampler.stop()
    elapsed = t0.elapsed_time(t1) / 1e3
    for ev in evs:   # per-kernel durations, CUDA events on the launching stream
        t_kern["trace_rays"] += ev[0].elapsed_time(ev[1])
        t_kern["eval_map"] += ev[1].elapsed_time(ev[2])
        t_kern["splat_sensor"] += ev[2].elapsed_time(ev[3])
        t_kern["film_allreduce"] += ev[3].elapsed_time(ev[4])
    step_s = elapsed / args.steps

    # ---------------- e2e: host buffers -> device -> step -> film back to host ----------
    e2e_steps = max(3, min(args.steps, 10))

    from paper_2605_04017_b200.pipeline import query_host_batch
    host_rays = dict(host, plane_z=rays_np["plane_z"])
    copy_stream = torch.cuda.Stream(device=dev)
    chunk = args.e2e_chunk
    copy_done = [torch.cuda.Event() for _ in range((n + chunk - 1) // chunk)]

    def e2e_step():
        # the public host-batch path: chunked H2D on a copy stream overlapping the kernels
        lens.enumerate_ghosts(0)
        film.zero_()
        query_host_batch(lens, pid, m, host_rays, d_rays, h_trace, h_map, FILM, film, None,
                         weight_scale=1.0 / n, chunk=chunk, compute_stream=stream, copy_stream=copy_stream,
                         copy_done=copy_done, fused=fused)
        if dist is not None:
            dist.all_reduce(film)
        film_host.copy_(film, non_blocking=True)

    e2e_step()
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(e2e_steps):
        e2e_step()
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_s = e0.elapsed_time(e1) / 1e3 / e2e_steps

    # valid fractions (for the algorithmic tanh count) -- outside the timed region
    def valid_frac(h):
        w = h["mask_bits"].cpu().numpy().view(np.uint32)
        return float(np.unpackbits(w.view(np.uint8)).sum()) / n

    v_map, v_trace = valid_frac(h_map), valid_frac(h_trace)

    vals = torch.tensor([step_s, e2e_s, elapsed], dtype=torch.float64, device=dev)
    if dist is not None:
        dist.all_reduce(vals, op=dist.ReduceOp.MAX)
    step_s, e2e_s, elapsed = vals.tolist()
    if rank != 0:
        return

    peaks, peaks_src = load_peaks()
    sm_max = float(peaks.get("sm_max_mhz", 1965.0))
    per_step = {k: v / args.steps / 1e3 for k, v in t_kern.items()}
    # eval_map roofline: MUFU (tanh) bound; algorithmic tanh = 64 per ray + 160 per valid ray
    tanh_per_launch = n * (TANH_PER_RAY_CLS + TANH_PER_RAY_REG * v_map)
    mufu_peak = MUFU_PER_CLK_PER_SM * 148 * sm_max * 1e6 / 1e9       # G tanh/s
    map_ach = tanh_per_launch / per_step["eval_map"] / 1e9
    flops_map = 2.0 * n * (MAC_CLS + MAC_REG * v_map)
    fp32_peak = FP32_LANES_PER_SM * 2 * 148 * sm_max * 1e6 / 1e12         # TFLOP/s
    trace_tflops = n * trace_flops_per_ray_c2() / per_step["trace_rays"] / 1e12
    trace_bytes = n * IO_BYTES_PER_RAY
    kernels = {
        "eval_map": {"ms": per_step["eval_map"] * 1e3, "M_rays_s": n / per_step["eval_map"] / 1e6,
                     "valid_frac": v_map,
                     "roofline": {"bound": "alu", "achieved": map_ach, "peak": mufu_peak, "unit": "Gtanh/s",
                                  "frac": map_ach / mufu_peak,
                                  "peak_source": "16 MUFU/clk/SM x 148 SMs x sm_max_mhz (DESIGN.md)"},
                     "tensor_TFLOPs": flops_map / per_step["eval_map"] / 1e12,
                     "tensor_frac": flops_map / per_step["eval_map"] / 1e12 / float(peaks["bf16_tflops"]),
                     "hbm_GBs": trace_bytes / per_step["eval_map"] / 1e9},
        "trace_rays": {"ms": per_step["trace_rays"] * 1e3, "M_rays_s": n / per_step["trace_rays"] / 1e6,
                       "valid_frac": v_trace,
                       "roofline": {"bound": "alu", "achieved": trace_tflops, "peak": fp32_peak,
                                    "unit": "TFLOP/s", "frac": trace_tflops / fp32_peak,
                                    "peak_source": "128 FP32 lanes x 2 x 148 SMs x sm_max_mhz (DESIGN.md)",
                                    "flops_per_ray": trace_flops_per_ray_c2()},
                       "hbm_GBs": trace_bytes / per_step["trace_rays"] / 1e9,
                       "hbm_frac": trace_bytes / per_step["trace_rays"] / 1e9 / float(peaks["hbm_gbs"])},
        "splat_sensor": {"ms": per_step["splat_sensor"] * 1e3,
                         "mode": "fused into trace_rays / eval_map epilogues" if fused else "separate kernel"},
        "film_allreduce": {"ms": per_step["film_allreduce"] * 1e3},
    }
    dominant = max(("eval_map", "trace_rays"), key=lambda k: kernels[k]["ms"])
    roof = dict(kernels[dominant]["roofline"])
    roof["kernel"] = dominant
    roof["traffic"] = ncu_traffic(dominant)
    value = ws * n / step_s / 1e6
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": step_s * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32 trace (+f64 refine), bf16xbf16->f32 map", "data": "synthetic",
        "config": workload_config(n, ws, pid),
        "roofline": roof,
        "kernels": kernels,
        "e2e": {"value": ws * n / e2e_s / 1e6, "unit": UNIT,
                "h2d_bytes_per_step": 4 * len(keys) * n, "d2h_bytes_per_step": npx * 8},
        "gpu_launches": args.steps * (3 if fused else 5),
        "clocks": clocks,
        "peaks_source": peaks_src,
    }
    if ws == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline()
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["plt", "reference"], default="plt")
    ap.add_argument("--rays", type=int, default=1 << 24, help="rays per GPU per step")
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
