# C2 loop: is the 1024-entry table gather (6-way bank conflicts) on the critical path?
for d in "" "PF_QNOTABLE" "PF_QNOWAIT" "PF_QNOWAIT;PF_QNOTABLE"; do
  echo "== $d"
  PFB200_DEFINES="PF_EVENT_TRACE;$d" python tools/trace_fused.py C2 2>&1 | grep -E "setup done|loop done"
  PFB200_DEFINES="$d" python bench.py --config C2 --steps 30 --warmup 5 --no-fit --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('step %.1f us kernel %.1f us value %r' % (d['ms_per_step']*1e3, d['roofline']['kernel_ms']*1e3, d['metric_value']))"
done
