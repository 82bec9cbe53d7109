# Developer A/B on a GPU box (one call); see DESIGN.md for the recorded outcomes.
set -u
mkdir -p gpurun_out
o=gpurun_out/ab17
V=paper_2605_04017_b200
for r in 1 2 3; do
  python tools/map_time_probe.py --tag rational >> $o.jsonl 2>&1
  PLT_LIB=$V/libplt_plt_map_acc_ex2.so python tools/map_time_probe.py --tag ex2 >> $o.jsonl 2>&1
done
python tools/logit_err_probe.py --flare > $o.err.jsonl 2>&1
PLT_LIB=$V/libplt_plt_map_acc_ex2.so python tools/logit_err_probe.py --flare > $o.err_ex2.jsonl 2>&1
python - <<'PY'
import json
for l in open("gpurun_out/ab17.jsonl"):
    if l.startswith("{"):
        d = json.loads(l); print(d["tag"], d["map"], round(d["ms"], 4))
PY
echo rational; cat $o.err.jsonl; echo ex2; cat $o.err_ex2.jsonl
