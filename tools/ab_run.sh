# Developer A/B on a GPU box (one call); see DESIGN.md for the recorded outcomes.
set -u
o=gpurun_out/ab30
for r in 1 2; do
  timeout 120 python tools/trace_time_probe.py --config C3 --rays 67108864 --tag back-2 >> $o.jsonl 2>&1
  PLT_TRACE_SPLIT_DELTA=2 timeout 120 python tools/trace_time_probe.py --config C3 --rays 67108864 --tag stop >> $o.jsonl 2>&1
  timeout 120 python tools/trace_time_probe.py --config C3 --rays 67108864 --fp64 --tag back-2 >> $o.jsonl 2>&1
  PLT_TRACE_SPLIT_DELTA=2 timeout 120 python tools/trace_time_probe.py --config C3 --rays 67108864 --fp64 --tag stop >> $o.jsonl 2>&1
  timeout 120 python tools/trace_time_probe.py --config C2 --tag fwd >> $o.jsonl 2>&1
done
timeout 900 python -m pytest tests/test_gpu_trace.py tests/test_gpu_camera.py tests/test_gpu_full_range.py tests/test_gpu_unit_dirs.py tests/test_gpu_asphere.py -q > $o.tests.log 2>&1; echo "exit $?" >> $o.tests.log
python - <<'PY'
import json
for l in open("gpurun_out/ab30.jsonl"):
    if l.startswith("{"):
        d = json.loads(l); print(d["tag"], d["config"], d["fp64"], round(d["ms"], 4))
    else: print(l[:200])
PY
tail -n 2 $o.tests.log
