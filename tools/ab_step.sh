# Developer A/B of whole bench steps (C2, fused splat) across libraries: alternating
# `bench.py --steps 100` runs (device time per step; no CPU baseline, no e2e).
#   gpurun -- 'bash tools/ab_step.sh TAG lib1.so lib2.so ...'
set -u
tag=$1; shift
o=gpurun_out/$tag
for r in 1 2 3; do
  for lib in "$@"; do
    PLT_LIB=$lib timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -n 1 | \
      python -c "import sys,json; j=json.loads(sys.stdin.read()); print(json.dumps({'tag': '$(basename $lib .so)', 'ms_per_step': j['ms_per_step'], 'trace_ms': j['kernels']['trace_rays']['ms'], 'map_ms': j['kernels']['eval_map']['ms']}))" >> $o.jsonl
  done
done
cat $o.jsonl
