# Developer A/B on a GPU box (one call); see DESIGN.md for the recorded outcomes.
set -u
mkdir -p gpurun_out
o=gpurun_out/ab22
V=paper_2605_04017_b200
for r in 1 2 3; do
  timeout 120 python tools/map_time_probe.py --tag k0 >> $o.jsonl 2>&1
  for k in 1 2 3; do
    PLT_LIB="$V/libplt_plt_map_fma_tanh_pairs=$k.so" timeout 120 python tools/map_time_probe.py --tag k$k >> $o.jsonl 2>&1
  done
done
PLT_LIB="$V/libplt_plt_map_fma_tanh_pairs=2.so" timeout 300 python tools/logit_err_probe.py > $o.err2.jsonl 2>&1
python - <<'PY'
import json
for l in open("gpurun_out/ab22.jsonl"):
    if l.startswith("{"):
        d = json.loads(l); print(d["tag"], d["map"], round(d["ms"], 4))
    else: print(l[:200])
PY
cat $o.err2.jsonl
