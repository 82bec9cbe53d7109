# Developer A/B on a GPU box (one call); see DESIGN.md for the recorded outcomes.
set -u
o=gpurun_out/ab41
for r in 1 2; do
  for lib in variants/libplt_prev.so paper_2605_04017_b200/libplt.so; do
    t=$(basename $lib .so)
    PLT_LIB=$lib timeout 120 python tools/map_time_probe.py --tag $t >> $o.jsonl 2>&1
    for n in 262144 1048576 4194304; do
      PLT_LIB=$lib timeout 120 python tools/map_time_probe.py --map C4_22 --ghost 65616 --rays $n --tag $t >> $o.jsonl 2>&1
      PLT_LIB=$lib timeout 120 python tools/map_time_probe.py --map C4_59 --ghost 16404 --rays $n --tag $t >> $o.jsonl 2>&1
    done
  done
done
timeout 1200 python -m pytest tests/test_gpu_map_splat.py tests/test_gpu_fitted_maps.py tests/test_gpu_fused_splat.py tests/test_gpu_flare_render.py tests/test_gpu_edge_cases.py -q -x > $o.tests.log 2>&1; echo "exit $?" >> $o.tests.log
python - <<'PY'
import json, collections
d = collections.defaultdict(list)
for l in open("gpurun_out/ab41.jsonl"):
    if l.startswith("{"):
        j = json.loads(l); d[(j["map"], j.get("ghost", 0), j["rays"], j["tag"])].append(round(j["ms"], 4))
for k in sorted(d): print(k, d[k])
PY
tail -n 2 $o.tests.log
