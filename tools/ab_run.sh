# Developer A/B on a GPU box (one call); see DESIGN.md for the recorded outcomes.
set -u
o=gpurun_out/ab37
for r in 1 2; do
  for lib in variants/libplt_prev.so paper_2605_04017_b200/libplt.so; do
    t=$(basename $lib .so)
    PLT_LIB=$lib timeout 120 python tools/trace_time_probe.py --config C4_22 --path 65616 --fp64 --rays 1048576 --tag $t >> $o.jsonl 2>&1
    PLT_LIB=$lib timeout 120 python tools/trace_time_probe.py --config C4_59 --path 16404 --fp64 --rays 1048576 --tag $t >> $o.jsonl 2>&1
    PLT_LIB=$lib timeout 120 python tools/trace_time_probe.py --config C2 --fp64 --tag $t >> $o.jsonl 2>&1
  done
done
timeout 900 python -m pytest tests/test_gpu_trace.py tests/test_gpu_flare_render.py tests/test_gpu_asphere.py tests/test_gpu_fuzz_lenses.py tests/test_gpu_path_pruning.py -q > $o.tests.log 2>&1; echo "exit $?" >> $o.tests.log
python - <<'PY'
import json
for l in open("gpurun_out/ab37.jsonl"):
    if l.startswith("{"):
        d = json.loads(l); print(d["tag"], d["config"], d["path"], round(d["ms"], 4))
PY
tail -n 2 $o.tests.log
