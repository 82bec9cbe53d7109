# Developer A/B on a GPU box (one call); see DESIGN.md for the recorded outcomes.
set -u
mkdir -p gpurun_out
o=gpurun_out/ab15
V=paper_2605_04017_b200
for r in 1 2; do
  for lib in $V/libplt_plt_fp64_full_newton.so $V/libplt.so; do
    t=$(basename $lib .so)
    PLT_LIB=$lib python tools/trace_time_probe.py --config C4_22 --path 65616 --fp64 --rays 1048576 --tag $t >> $o.jsonl 2>&1
    PLT_LIB=$lib python tools/trace_time_probe.py --config C4_59 --path 16404 --fp64 --rays 1048576 --tag $t >> $o.jsonl 2>&1
    PLT_LIB=$lib python tools/trace_time_probe.py --config C2 --fp64 --tag $t >> $o.jsonl 2>&1
    PLT_LIB=$lib python tools/trace_time_probe.py --config C2 --tag $t >> $o.jsonl 2>&1
  done
done
timeout 900 python -m pytest tests/test_gpu_trace.py tests/test_gpu_flare_render.py tests/test_gpu_path_pruning.py tests/test_gpu_asphere.py tests/test_gpu_edge_cases.py tests/test_gpu_fuzz_lenses.py tests/test_gpu_unit_dirs.py tests/test_gpu_camera.py -q > $o.tests.log 2>&1; echo "exit $?" >> $o.tests.log
python - <<'PY'
import json
for l in open("gpurun_out/ab15.jsonl"):
    if l.startswith("{"):
        d = json.loads(l); print(d["tag"], d["config"], d["path"], d["fp64"], round(d["ms"], 4))
PY
tail -n 3 $o.tests.log
