"""Summarise an ncu --set full report: key throughput metrics, stall reasons, top SASS stall sites."""
import csv
import io
import subprocess
import sys
from collections import Counter

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__cycles_elapsed.avg.per_second", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def main(rep, top=25, which=None):
    h, u, data = raw(rep)
    for kidx, r in enumerate(data):
        if which is not None and kidx != which:
            continue
        print("kernel[%d]:" % kidx, r[h.index("Kernel Name")][:100])
        for k in KEYS:
            if k in h:
                print(f"  {k:70s} {r[h.index(k)]:>16s} {u[h.index(k)]}")
        stalls = [(k, float(r[i])) for i, k in enumerate(h)
                  if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")
                  and r[i] not in ("", "n/a")]
        stalls.sort(key=lambda x: -x[1])
        print("  stalls/issue:", ", ".join(f"{k[34:-23]}={v:.2f}" for k, v in stalls[:8]))
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    # split into per-kernel sections (each starts with a "Kernel Name" row then a header row)
    sections, cur = [], None
    for row in rows:
        if row and row[0] == "Kernel Name":
            cur = {"name": row[1] if len(row) > 1 else "", "rows": []}
            sections.append(cur)
        elif cur is not None:
            cur["rows"].append(row)
    seen = set()
    for sidx, sec in enumerate(sections):
        if which is not None and sidx != which:
            continue
        if sec["name"] in seen and which is None:
            continue
        seen.add(sec["name"])
        hh, d = sec["rows"][0], sec["rows"][1:]
        si, src, ex = hh.index("Warp Stall Sampling (All Samples)"), hh.index("Source"), hh.index("Instructions Executed")
        tot = sum(float(x[si] or 0) for x in d) or 1.0
        print(f"== {sec['name'][:80]}: top stall sites (of {tot:.0f} samples):")
        for x in sorted(d, key=lambda x: -float(x[si] or 0))[:top]:
            print(f"   {float(x[si] or 0) / tot * 100:5.1f}%  {x[src].strip()[:80]}")
        c = Counter()
        for x in d:
            t = x[src].strip().split()
            if not t:
                continue
            op = t[1] if t[0].startswith("@") and len(t) > 1 else t[0]
            c[op.split(".")[0]] += float(x[ex] or 0)
        tot_i = sum(c.values()) or 1.0
        print("  instruction mix:", ", ".join(f"{k}={v / tot_i * 100:.1f}%" for k, v in c.most_common(16)))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25,
         int(sys.argv[3]) if len(sys.argv) > 3 else None)
