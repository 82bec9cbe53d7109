"""Summarise a tools/refresh_evidence.sh run (gpurun_out/<tag>_*) into profiles/:
the bench and reference-arm lines, the launch-list shares, the ncu --set full summary and
the per-launch DRAM traffic bench.py reports as roofline.traffic.

    python tools/refresh_profiles.py r01
"""
import csv
import io
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))


def last_json_line(path):
    with open(path) as f:
        lines = [l for l in f if l.strip().startswith("{")]
    return json.loads(lines[-1]) if lines else None


def traffic(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, data = rows[0], rows[2:]
    name, rd, wr = h.index("Kernel Name"), h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum")
    unit = rows[1][rd]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[unit]
    res = {}
    for r in data:
        k = "trace_rays" if "plt_trace_jit" in r[name] else "eval_map" if "eval_map" in r[name] else \
            "refine" if "refine" in r[name] else None
        if k and k not in res:
            res[k] = {"dram_read": int(float(r[rd].replace(",", "")) * scale),
                      "dram_write": int(float(r[wr].replace(",", "")) * scale)}
    return res


def main(tag):
    g, p = os.path.join(ROOT, "gpurun_out"), os.path.join(ROOT, "profiles")
    for kind in ("bench", "reference_arm", "configs"):
        src = os.path.join(g, f"{tag}_{kind}.json")
        if os.path.exists(src) and os.path.getsize(src) > 0:
            if kind == "configs":
                shutil.copy(src, os.path.join(p, f"{tag}_configs.json"))
            else:
                line = last_json_line(src)
                with open(os.path.join(p, f"{tag}_{kind}.json"), "w") as f:
                    json.dump(line, f, indent=1)
                    f.write("\n")
    for f in sorted(os.listdir(g)):   # flare / dof images and reports
        if f.startswith(f"{tag}_flare_") or f.startswith(f"{tag}_dof"):
            if f.endswith(".json") or f.endswith(".png"):
                shutil.copy(os.path.join(g, f), os.path.join(p, f))
    launches = os.path.join(g, f"{tag}_bench_launches.csv")
    if os.path.exists(launches):
        shutil.copy(launches, os.path.join(p, f"{tag}_bench_launches.csv"))
        txt = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "launch_summary.py"), launches,
                              "python bench.py --steps 2 --warmup 1 --no-cpu-baseline"],
                             capture_output=True, text=True).stdout
        with open(os.path.join(p, f"{tag}_bench_launches_summary.txt"), "w") as f:
            f.write(txt)
    rep = os.path.join(g, f"{tag}_full.ncu-rep")
    if os.path.exists(rep):
        txt = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), rep],
                             capture_output=True, text=True).stdout
        with open(os.path.join(p, f"{tag}_ncu_full_summary.txt"), "w") as f:
            f.write("# ncu --set full --clock-control none of python bench.py --steps 1 --warmup 0 "
                    "--no-cpu-baseline (one capture each: plt_trace_jit, refine_kernel, eval_map_kernel<8>)\n")
            f.write(txt)
        t = traffic(rep)
        n = 1 << 24
        alg = {"eval_map": n * (20 + 24) + n // 8, "trace_rays": n * (20 + 24) + n // 8}
        for k in t:
            if k in alg:
                t[k]["algorithmic"] = alg[k]
        with open(os.path.join(p, f"{tag}_ncu_traffic.json"), "w") as f:
            json.dump({"source": f"profiles/{tag}_ncu_full_summary.txt (ncu --set full --clock-control none, "
                                 "python bench.py --steps 1 --warmup 0 --no-cpu-baseline, one B200)",
                       "unit": "bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum), 2^24 rays; "
                               "algorithmic = 20 B in (no dz, A32) + 24 B out + 1/8 B mask per ray",
                       "kernels": t}, f, indent=1)
            f.write("\n")
    print("profiles refreshed for", tag)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r01")
