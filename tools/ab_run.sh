# Developer A/B on a GPU box (one call); see DESIGN.md for the recorded outcomes.
set -u
o=gpurun_out/ab36
for v in base disc out both pre; do
  case $v in base) D="";; disc) D="#define PLT_TRACE_DISC_FAST 1";; out) D="#define PLT_TRACE_OUT_FAST 1";; both) D="#define PLT_TRACE_DISC_FAST 1
#define PLT_TRACE_OUT_FAST 1";; pre) D="";; esac
  if [ $v = pre ]; then PLT_LIB=variants/libplt_prev.so timeout 600 python tools/trace_err_probe.py 2>/dev/null | tail -1 >> $o.jsonl
  else PLT_JIT_DEFINES="$D" timeout 600 python tools/trace_err_probe.py 2>/dev/null | tail -1 >> $o.jsonl; fi
done
cat $o.jsonl
