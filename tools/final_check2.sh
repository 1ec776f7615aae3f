# the whole GPU suite at HEAD, smoke, and C1-C5 bench lines (MMIO publish)
timeout 1200 python -m pytest tests -q -m gpu 2>&1 | tail -3
python __graft_entry__.py smoke 2>&1 | tail -1
for c in C2 C1 C3 C4 C5 C5TI; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-fit --no-cpu-baseline 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    l=l.strip()
    if l.startswith('{'):
        d=json.loads(l); print('$c step %.1f us  kernel %.1f us  e2e %.1f us  value %r frac %.3f' % (d['ms_per_step']*1e3, d['roofline']['kernel_ms']*1e3, d['e2e']['ms_per_step']*1e3, d['metric_value'], d['roofline']['frac']))
    elif 'Error' in l or 'error' in l: print(l)
"
done
timeout 300 python tools/e2e_probe.py 2>&1 | tail -4
