# Developer A/B on a GPU box (one call); see DESIGN.md for the recorded outcomes.
set -u
mkdir -p gpurun_out
o=gpurun_out/ab20
V=paper_2605_04017_b200
for r in 1 2 3; do
  PLT_LIB=$V/libplt_plt_map_bias_d.so timeout 120 python tools/map_time_probe.py --tag bias-d >> $o.jsonl 2>&1
  timeout 120 python tools/map_time_probe.py --tag base >> $o.jsonl 2>&1
done
PLT_LIB=$V/libplt_plt_map_bias_d.so timeout 300 python tools/logit_err_probe.py > $o.err.jsonl 2>&1
PLT_LIB=$V/libplt_plt_map_bias_d.so timeout 600 python -m pytest tests/test_gpu_fitted_maps.py tests/test_gpu_map_splat.py tests/test_gpu_fused_splat.py -q > $o.tests.log 2>&1; echo "exit $?" >> $o.tests.log
python - <<'PY'
import json
for l in open("gpurun_out/ab20.jsonl"):
    if l.startswith("{"):
        d = json.loads(l); print(d["tag"], d["map"], round(d["ms"], 4))
    else: print(l[:300])
PY
cat $o.err.jsonl; tail -n 2 $o.tests.log
