# Developer A/B on a GPU box (one call); see DESIGN.md for the recorded outcomes.
set -u
o=gpurun_out/ab25
for r in 1 2; do
  for c in C2 C3; do
    extra=""; [ $c = C3 ] && extra="--rays 67108864"
    timeout 120 python tools/trace_time_probe.py --config $c $extra --tag early >> $o.jsonl 2>&1
    PLT_TRACE_NO_EARLY=1 timeout 120 python tools/trace_time_probe.py --config $c $extra --tag none >> $o.jsonl 2>&1
    PLT_TRACE_JIT=0 timeout 120 python tools/trace_time_probe.py --config $c $extra --tag early-generic >> $o.jsonl 2>&1
    PLT_TRACE_JIT=0 PLT_TRACE_NO_EARLY=1 timeout 120 python tools/trace_time_probe.py --config $c $extra --tag none-generic >> $o.jsonl 2>&1
  done
done
timeout 600 python -m pytest tests/test_gpu_trace.py tests/test_gpu_trace_jit.py tests/test_gpu_fused_splat.py tests/test_gpu_edge_cases.py tests/test_gpu_full_range.py tests/test_gpu_camera.py tests/test_gpu_determinism.py -q > $o.tests.log 2>&1; echo "exit $?" >> $o.tests.log
PLT_TRACE_JIT=0 timeout 600 python -m pytest tests/test_gpu_trace.py tests/test_gpu_edge_cases.py tests/test_gpu_fuzz_lenses.py -q > $o.tests_g.log 2>&1; echo "exit $?" >> $o.tests_g.log
python - <<'PY'
import json
for l in open("gpurun_out/ab25.jsonl"):
    if l.startswith("{"):
        d = json.loads(l); print(d["tag"], d["config"], round(d["ms"], 4), d["flagged_frac"])
    else: print(l[:200])
PY
tail -n 2 $o.tests.log $o.tests_g.log
