# Developer A/B on a GPU box (one call): trace variants.
set -u
mkdir -p gpurun_out
o=gpurun_out/ab3
TORCH_NVRTC=/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/cuda_nvrtc/lib/libnvrtc.so.12
for r in 1 2; do
  for c in C2 C3; do
    extra=""; [ $c = C3 ] && extra="--rays 67108864"
    PLT_TRACE_QUEUE=0 python tools/trace_time_probe.py --config $c $extra --tag block >> $o.jsonl 2>&1
    PLT_TRACE_QUEUE=1 python tools/trace_time_probe.py --config $c $extra --tag queue >> $o.jsonl 2>&1
    PLT_TRACE_QUEUE=0 PLT_JIT_DEFINES="#define PLT_NEAR_UNGATED 1" python tools/trace_time_probe.py --config $c $extra --tag block-ungated >> $o.jsonl 2>&1
    PLT_TRACE_QUEUE=0 PLT_NVRTC=$TORCH_NVRTC python tools/trace_time_probe.py --config $c $extra --tag block-nvrtc128 >> $o.jsonl 2>&1
  done
done
PLT_TRACE_QUEUE=0 timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > $o.bench.json 2>&1
python - <<'PY'
import json
for l in open("gpurun_out/ab3.jsonl"):
    if l.startswith("{"):
        d = json.loads(l); print(d["tag"], d["config"], round(d["ms"], 4), d["kernel"], d["flagged_frac"])
PY
tail -c 300 $o.bench.json
