#!/usr/bin/env bash
# Re-measure the round's evidence on a GPU box (one B200); outputs land in gpurun_out/ and
# are summarised into profiles/ by tools/refresh_profiles.py on the build host.
#   gpurun --timeout 1800 -- 'bash tools/refresh_evidence.sh r01'
set -u
tag=${1:-r01}
out=gpurun_out
mkdir -p $out
timeout 600 python bench.py > $out/${tag}_bench.json 2> $out/${tag}_bench.err || echo "bench failed"
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > $out/${tag}_reference_arm.json 2>> $out/${tag}_bench.err || echo "reference arm failed"
# launch list (cold-cache, serialised: shares, not absolute times)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/${tag}_bench_launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $out/${tag}_ncu_launches.log 2>&1 || echo "launch list failed"
# one full capture of each kernel of the step
timeout 900 ncu --set full --clock-control none --import-source on \
    -k 'regex:plt_trace_jit|refine_kernel|eval_map_kernel' -c 3 -o $out/${tag}_full \
    python bench.py --steps 1 --warmup 0 --no-cpu-baseline > $out/${tag}_ncu_full.log 2>&1 || echo "ncu full failed"
timeout 900 python tools/configs_bench.py > $out/${tag}_configs.json 2> $out/${tag}_configs.err || echo "configs failed"
# NEXT-2 flare images and NEXT-3 depth of field (timings + image agreement)
for c in C4_22 C4_59; do
    timeout 600 python tools/flare_compare.py --config $c --out $out/${tag}_flare_$c.json --png $out/${tag}_flare_$c \
        > $out/${tag}_flare_$c.log 2>&1 || echo "flare $c failed"
done
timeout 900 python tools/dof_compare.py --spp 1024 --out $out/${tag}_dof.json --png $out/${tag}_dof > $out/${tag}_dof.log 2>&1 || echo "dof failed"
tail -c 400 $out/${tag}_bench.json
