# Developer A/B of eval_map variants on a GPU box (one call): alternating runs of
# tools/map_time_probe.py (C2 fitted map, 2^24 rays, fused splat) per library.
#   gpurun -- 'bash tools/ab_map.sh TAG lib1.so lib2.so ...'
set -u
tag=$1; shift
o=gpurun_out/$tag
for r in 1 2 3; do
  for lib in "$@"; do
    PLT_LIB=$lib timeout 120 python tools/map_time_probe.py --tag $(basename $lib .so) >> $o.jsonl 2>&1
    PLT_LIB=$lib timeout 120 python tools/map_time_probe.py --map C3 --rays 16777216 --tag $(basename $lib .so) >> $o.jsonl 2>&1
  done
done
python - "$o.jsonl" <<'PY'
import json, collections, sys
d = collections.defaultdict(list)
for l in open(sys.argv[1]):
    if l.startswith("{"):
        j = json.loads(l); d[(j["map"], j["rays"], j["tag"])].append(round(j["ms"], 4))
for k in sorted(d): print(k, d[k])
PY
