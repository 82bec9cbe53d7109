# Developer A/B on a GPU box (one call); see DESIGN.md for the recorded outcomes.
set -u
o=gpurun_out/ab40
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/pipemix tools/pipe_mix_bench.cu && /tmp/pipemix > $o.pipemix.json 2>&1
for r in 1 2 3; do
  for lib in paper_2605_04017_b200/libplt.so variants/libplt_ef.so variants/libplt_el.so variants/libplt_efel.so; do
    PLT_LIB=$lib timeout 120 python tools/map_time_probe.py >> $o.jsonl 2>&1
  done
done
for lib in paper_2605_04017_b200/libplt.so variants/libplt_ef.so variants/libplt_el.so variants/libplt_efel.so; do
  t=$(basename $lib .so)
  PLT_LIB=$lib timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_write.sum,lts__t_sectors_srcunit_tex_op_read.sum \
    -k regex:eval_map -c 2 --csv python tools/map_time_probe.py --tag $t > $o.ncu_$t.csv 2>&1
done
python - <<'PY'
import json, collections
d = collections.defaultdict(list)
for l in open("gpurun_out/ab40.jsonl"):
    if l.startswith("{"):
        j = json.loads(l); d[j["tag"]].append(round(j["ms"], 4))
for k, v in d.items(): print(k, v)
PY
cat $o.pipemix.json
