# Developer A/B on a GPU box (one call); see DESIGN.md for the recorded outcomes.
set -u
o=gpurun_out/ab28
for r in 1 2 3; do
  timeout 120 python tools/map_time_probe.py --tag iterwait >> $o.jsonl 2>&1
  PLT_LIB=variants/libplt_prev.so timeout 120 python tools/map_time_probe.py --tag clockwait >> $o.jsonl 2>&1
done
timeout 120 python tools/map_time_probe.py --map C3 --rays 67108864 --tag iterwait >> $o.jsonl 2>&1
PLT_LIB=variants/libplt_prev.so timeout 120 python tools/map_time_probe.py --map C3 --rays 67108864 --tag clockwait >> $o.jsonl 2>&1
timeout 600 python -m pytest tests/test_gpu_map_splat.py tests/test_gpu_fitted_maps.py tests/test_gpu_graph.py -q > $o.tests.log 2>&1; echo "exit $?" >> $o.tests.log
python - <<'PY'
import json
for l in open("gpurun_out/ab28.jsonl"):
    if l.startswith("{"):
        d = json.loads(l); print(d["tag"], d.get("config", d.get("map")), round(d["ms"], 4))
    else: print(l[:200])
PY
tail -n 2 $o.tests.log
