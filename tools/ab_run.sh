# Developer A/B on a GPU box (one call); see DESIGN.md for the recorded outcomes.
set -u
mkdir -p gpurun_out
o=gpurun_out/ab18
for r in 1 2 3; do
  python tools/map_time_probe.py --tag preissue >> $o.jsonl 2>&1
  PLT_LIB=variants/libplt_rational.so python tools/map_time_probe.py --tag base >> $o.jsonl 2>&1
done
python tools/logit_err_probe.py > $o.err.jsonl 2>&1
timeout 600 python -m pytest tests/test_gpu_fitted_maps.py tests/test_gpu_map_splat.py tests/test_gpu_fused_splat.py -q > $o.tests.log 2>&1; echo "exit $?" >> $o.tests.log
python - <<'PY'
import json
for l in open("gpurun_out/ab18.jsonl"):
    if l.startswith("{"):
        d = json.loads(l); print(d["tag"], d["map"], round(d["ms"], 4))
    else: print(l[:300])
PY
cat $o.err.jsonl; tail -n 2 $o.tests.log
