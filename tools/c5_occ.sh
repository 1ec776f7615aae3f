# C5 event kernel: resident 2-warp blocks per SM (register cap) 8 / 10 / 12 / 16
run() { echo "== $1"; shift; env "$@" timeout 300 python bench.py --config C5 --steps 20 --warmup 5 --no-fit --no-cpu-baseline 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    l=l.strip()
    if l.startswith('{'):
        d=json.loads(l); print('step %.1f us  kernel %.1f us  value %r' % (d['ms_per_step']*1e3, d['roofline']['kernel_ms']*1e3, d['metric_value']))
    elif 'Error' in l or 'error' in l: print(l)
"; }
run default X=1
run b10 PFB200_EV_BLOCKS=10 PFB200_DEFINES=PF_EVENT_MIN_BLOCKS=10
run b12 PFB200_EV_BLOCKS=12 PFB200_DEFINES=PF_EVENT_MIN_BLOCKS=12
run b16 PFB200_EV_BLOCKS=16 PFB200_DEFINES=PF_EVENT_MIN_BLOCKS=16
