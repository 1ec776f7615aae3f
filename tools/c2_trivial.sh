# is C2's event loop bound by its math or by the stream?  (PF_QTRIVIAL: one add per event)
run() { echo "== $1 $3"; env $2 python bench.py --config C2 --steps 30 --warmup 5 --no-fit --no-cpu-baseline $3 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    l=l.strip()
    if l.startswith('{'):
        d=json.loads(l); print('step %.1f us  kernel %.1f us  value %r' % (d['ms_per_step']*1e3, d['roofline']['kernel_ms']*1e3, d['metric_value']))
    elif 'Error' in l or 'error' in l: print(l)
"; }
run default X=1
run trivial PFB200_DEFINES=PF_QTRIVIAL
run trivial PFB200_DEFINES=PF_QTRIVIAL --diag-no-flush
for d in "" "PF_QTRIVIAL"; do echo "== trace $d"; PFB200_DEFINES="PF_EVENT_TRACE;$d" python tools/trace_fused.py C2 2>&1 | tail -8; done
