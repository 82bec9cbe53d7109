set -u
o=gpurun_out/guard
for r in 1 2 3; do
  for lib in variants/libplt_base.so paper_2605_04017_b200/libplt.so; do
    PLT_LIB=$lib timeout 120 python tools/trace_time_probe.py --tag $(basename $lib .so) >> $o.jsonl 2>&1
  done
done
timeout 1200 python -m pytest tests/test_gpu_map_splat.py tests/test_gpu_fused_splat.py tests/test_gpu_flare_render.py tests/test_gpu_determinism.py tests/test_gpu_camera.py tests/test_gpu_trace_paths.py -q -x > $o.tests.log 2>&1; echo "exit $?" >> $o.tests.log
grep -h '^{' $o.jsonl | python -c "
import sys,json,collections
d=collections.defaultdict(list)
for l in sys.stdin:
    j=json.loads(l); d[j.get('tag')].append(round(j['ms'],4))
print(dict(d))"
tail -n 3 $o.tests.log
