"""Per-kernel shares of an ncu launch list (`ncu --metrics gpu__time_duration.sum --csv`).
    python tools/launch_summary.py launches.csv [title]"""
import csv
import re
import sys
from collections import defaultdict


def short(name: str) -> str:
    name = re.sub(r"\(.*$", "", name)                      # drop the argument list
    name = re.sub(r"^void\s+", "", name)
    name = name.replace("plt::<unnamed>::", "").replace("(anonymous namespace)::", "")
    if name.startswith("at::") or "at::native" in name:
        return "torch:" + name.split("::")[-1][:40]
    return name


def main(path, title=""):
    rows = []
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        us = v / 1000.0 if unit in ("ns", "nsecond") else v if unit in ("us", "usecond") else v * 1000.0
        rows.append((short(r["Kernel Name"]), us))
    agg = defaultdict(lambda: [0, 0.0])
    for k, us in rows:
        agg[k][0] += 1
        agg[k][1] += us
    tot = sum(v[1] for v in agg.values())
    if title:
        print(f"# {title}")
    print("# gpu__time_duration.sum per launch, --clock-control none; ncu serialises launches (cold caches):")
    print("# compare SHARES with the bench's event timings, not absolutes.")
    print(f"{'kernel':40s} {'launches':>8s} {'mean_us':>10s} {'total_us':>10s} {'share':>7s}")
    for k, (c, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k:40s} {c:8d} {us / c:10.1f} {us:10.1f} {100 * us / tot:6.1f}%")


if __name__ == "__main__":
    main(sys.argv[1], " ".join(sys.argv[2:]))
