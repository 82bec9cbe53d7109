# Developer A/B on a GPU box (one call); see DESIGN.md for the recorded outcomes.
set -u
o=gpurun_out/ab33
for v in base both; do
  case $v in base) D="";; both) D="#define PLT_TRACE_COST_FAST 1
#define PLT_TRACE_T1_FAST 1";; esac
  PLT_JIT_DEFINES="$D" timeout 900 python -m pytest tests/test_gpu_trace.py tests/test_gpu_full_range.py tests/test_gpu_fuzz_lenses.py -q -s -k "c1_ or c2_ or c3_ or ragged or full_range or fuzz" 2>&1 | grep -E "^compare_trace|passed|failed" | sed "s/^/$v /" >> $o.log
done
python - <<'PY'
import ast, collections
mx = collections.defaultdict(lambda: {'max_dp':0,'max_dw':0,'max_dI':0, 'n':0})
for l in open("gpurun_out/ab33.log"):
    v, rest = l.split(" ", 1)
    if rest.startswith("compare_trace"):
        d = ast.literal_eval(rest[len("compare_trace "):].strip())
        if d.get("n", 0) >= 4096:
            m = mx[v]
            for k in ('max_dp','max_dw','max_dI'): m[k] = max(m[k], d.get(k, 0))
            m['n'] += 1
    else: print(v, rest.strip())
for v, m in mx.items(): print(v, m)
PY
