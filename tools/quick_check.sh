# quick A/B after a kernel change: C1-C3 step times, the C2 timeline, the parity tests
for c in C2 C1 C3; do
  python bench.py --config $c --steps 30 --warmup 5 --no-fit --no-cpu-baseline 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    l=l.strip()
    if l.startswith('{'):
        d=json.loads(l); print('$c step %.1f us  kernel %.1f us  e2e %.1f us  value %r' % (d['ms_per_step']*1e3, d['roofline']['kernel_ms']*1e3, d['e2e']['ms_per_step']*1e3, d['metric_value']))
    elif 'Error' in l or 'error' in l: print(l)
"
done
PFB200_DEFINES="PF_SETUP_TRACE" python tools/trace_fused.py C2 2>&1 | tail -9 | head -8
PFB200_DEFINES="PF_EVENT_TRACE" python tools/trace_fused.py C2 2>&1 | tail -9
python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -3
