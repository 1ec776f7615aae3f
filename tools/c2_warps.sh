# C2: active warps per SM through the chunk size (EPT x NSUB x 32 events): 11 (default), 14.7, 16
run() { echo "== $1"; shift; env "$@" python bench.py --config C2 --steps 30 --warmup 5 --no-fit --no-cpu-baseline 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    l=l.strip()
    if l.startswith('{'):
        d=json.loads(l); print('step %.1f us  kernel %.1f us  e2e %.1f us  value %r %s' % (d['ms_per_step']*1e3, d['roofline']['kernel_ms']*1e3, d['e2e']['ms_per_step']*1e3, d['metric_value'], d['roofline'].get('kernel')))
    elif 'Error' in l or 'error' in l: print(l)
"; }
run default X=1
run ept22_nsub3 PFB200_EPT=22 PFB200_NSUB=3
run ept18_nsub4 PFB200_EPT=18 PFB200_NSUB=4
run ept22_nsub3_maxint PFB200_EPT=22 PFB200_NSUB=3 PFB200_DEFINES=PF_QMAX_INT
run default_again X=1
for e in "PFB200_EPT=22 PFB200_NSUB=3" "X=1"; do env $e PFB200_DEFINES="PF_EVENT_TRACE" python tools/trace_fused.py C2 2>&1 | tail -7; done
