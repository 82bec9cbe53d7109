# Developer A/B on a GPU box (one call); see DESIGN.md for the recorded outcomes.
set -u
o=gpurun_out/ab27
for r in 1 2; do
  timeout 120 python tools/trace_time_probe.py --config C2 --tag new >> $o.jsonl 2>&1
  PLT_LIB=variants/libplt_prev.so timeout 120 python tools/trace_time_probe.py --config C2 --tag prev >> $o.jsonl 2>&1
  timeout 120 python tools/map_time_probe.py --tag new >> $o.jsonl 2>&1
  PLT_LIB=variants/libplt_prev.so timeout 120 python tools/map_time_probe.py --tag prev >> $o.jsonl 2>&1
  timeout 120 python tools/splat_probe.py >> $o.splat.log 2>&1
  PLT_LIB=variants/libplt_prev.so timeout 120 python tools/splat_probe.py >> $o.splat.log 2>&1
done
timeout 900 python -m pytest tests/test_gpu_map_splat.py tests/test_gpu_fused_splat.py tests/test_gpu_flare_render.py tests/test_gpu_determinism.py tests/test_gpu_query_host.py tests/test_gpu_edge_cases.py -q > $o.tests.log 2>&1; echo "exit $?" >> $o.tests.log
python - <<'PY'
import json
for l in open("gpurun_out/ab27.jsonl"):
    if l.startswith("{"):
        d = json.loads(l); print(d["tag"], d.get("config", d.get("map")), round(d["ms"], 4))
    else: print(l[:200])
PY
cat $o.splat.log | tail -8; tail -n 2 $o.tests.log
