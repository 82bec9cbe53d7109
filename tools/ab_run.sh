# Developer A/B on a GPU box (one call); see DESIGN.md for the recorded outcomes.
set -u
mkdir -p gpurun_out
o=gpurun_out/ab23
for c in C4_22 C4_59; do
  for fs in 1 2 4 8; do
    timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --flare-streams $fs --dump-film gpurun_out/film_${c}_$fs.npy 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$c', $fs, round(d['ms_per_step'],3), {k:round(v['ms'],3) for k,v in d['kernels'].items()})"
  done
  python -c "
import numpy as np
a=[np.load('gpurun_out/film_${c}_%d.npy'%f) for f in (1,2,4,8)]
print('films identical:', all(np.array_equal(a[0], x) for x in a[1:]))"
done
