# Developer A/B on a GPU box (one call); see DESIGN.md for the recorded outcomes.
set -u
mkdir -p gpurun_out
o=gpurun_out/ab16
for r in 1 2; do
  python tools/trace_time_probe.py --config C2 --tag idx32 >> $o.jsonl 2>&1
  python tools/trace_time_probe.py --config C3 --rays 67108864 --tag idx32 >> $o.jsonl 2>&1
  PLT_TRACE_JIT=0 python tools/trace_time_probe.py --config C2 --tag idx32-generic >> $o.jsonl 2>&1
done
timeout 900 python -m pytest tests/test_gpu_trace.py tests/test_gpu_trace_jit.py tests/test_gpu_fused_splat.py tests/test_gpu_edge_cases.py tests/test_gpu_unit_dirs.py tests/test_gpu_full_range.py tests/test_gpu_graph.py -q > $o.tests.log 2>&1; echo "exit $?" >> $o.tests.log
python - <<'PY'
import json
for l in open("gpurun_out/ab16.jsonl"):
    if l.startswith("{"):
        d = json.loads(l); print(d["tag"], d["config"], d["path"], round(d["ms"], 4), d["flagged_frac"])
PY
tail -n 3 $o.tests.log
