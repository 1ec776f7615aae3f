# C2 QFAST loop variants: unroll depth (instruction-fetch stalls) and max(d,0) on the integer pipe
run() { echo "== $1"; shift; env "$@" python bench.py --config C2 --steps 30 --warmup 5 --no-fit --no-cpu-baseline 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    l=l.strip()
    if l.startswith('{'):
        d=json.loads(l); print('step %.1f us  kernel %.1f us  e2e %.1f us  value %r' % (d['ms_per_step']*1e3, d['roofline']['kernel_ms']*1e3, d['e2e']['ms_per_step']*1e3, d['metric_value']))
    elif 'Error' in l or 'error' in l: print(l)
"; }
run default X=1
run u1 PFB200_DEFINES="PF_QUNROLL=1"
run u2 PFB200_DEFINES="PF_QUNROLL=2"
run u4 PFB200_DEFINES="PF_QUNROLL=4"
run maxint PFB200_DEFINES="PF_QMAX_INT"
run u2_maxint PFB200_DEFINES="PF_QUNROLL=2;PF_QMAX_INT"
run u4_maxint PFB200_DEFINES="PF_QUNROLL=4;PF_QMAX_INT"
run default_again X=1
