# Developer A/B on a GPU box (one call); see DESIGN.md for the recorded outcomes.
set -u
mkdir -p gpurun_out
o=gpurun_out/ab8
V=paper_2605_04017_b200
for r in 1 2 3; do
  python tools/map_time_probe.py --tag duty-claim-ahead >> $o.jsonl 2>&1
  PLT_LIB=variants/libplt_duty.so python tools/map_time_probe.py --tag duty >> $o.jsonl 2>&1
done
PLT_LIB=$V/libplt_plt_map_profile.so python tools/map_time_probe.py --tag profile > $o.profile.log 2>&1
python tools/logit_err_probe.py > $o.err.jsonl 2>&1
python - <<'PY'
import json
for l in open("gpurun_out/ab8.jsonl"):
    if l.startswith("{"):
        d = json.loads(l); print(d["tag"], round(d["ms"], 4))
PY
grep "PROF blk0" $o.profile.log | tail -8; cat $o.err.jsonl
