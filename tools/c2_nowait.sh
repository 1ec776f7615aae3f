# C2 loop: the math alone (PF_QNOWAIT: no TMA waits/refills) vs the stream alone (PF_QTRIVIAL) vs both
for d in "" "PF_QNOWAIT" "PF_QTRIVIAL" "PF_QMAX_INT" "PF_QNOWAIT;PF_QMAX_INT"; do
  echo "== $d"
  PFB200_DEFINES="PF_EVENT_TRACE;$d" python tools/trace_fused.py C2 2>&1 | grep -E "setup done|loop done|finalize"
  PFB200_DEFINES="$d" python bench.py --config C2 --steps 30 --warmup 5 --no-fit --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('step %.1f us kernel %.1f us value %r' % (d['ms_per_step']*1e3, d['roofline']['kernel_ms']*1e3, d['metric_value']))"
done
