# Developer A/B on a GPU box (one call); see DESIGN.md for the recorded outcomes.
set -u
mkdir -p gpurun_out
o=gpurun_out/ab19
timeout 300 python -m pytest tests/test_gpu_map_splat.py -q -x > $o.tests0.log 2>&1; echo "exit $?" >> $o.tests0.log; tail -n 3 $o.tests0.log
for r in 1 2 3; do
  timeout 120 python tools/map_time_probe.py --tag db >> $o.jsonl 2>&1
  PLT_MAP_DB=0 timeout 120 python tools/map_time_probe.py --tag base >> $o.jsonl 2>&1
done
timeout 120 python tools/map_time_probe.py --map C3 --rays 67108864 --tag db >> $o.jsonl 2>&1
PLT_MAP_DB=0 timeout 120 python tools/map_time_probe.py --map C3 --rays 67108864 --tag base >> $o.jsonl 2>&1
timeout 300 python tools/logit_err_probe.py > $o.err.jsonl 2>&1
timeout 600 python -m pytest tests/test_gpu_fitted_maps.py tests/test_gpu_map_splat.py tests/test_gpu_fused_splat.py tests/test_gpu_edge_cases.py tests/test_gpu_graph.py tests/test_gpu_flare_render.py -q > $o.tests.log 2>&1; echo "exit $?" >> $o.tests.log
python - <<'PY'
import json
for l in open("gpurun_out/ab19.jsonl"):
    if l.startswith("{"):
        d = json.loads(l); print(d["tag"], d["map"], round(d["ms"], 4))
    else: print(l[:300])
PY
cat $o.err.jsonl; tail -n 2 $o.tests.log
