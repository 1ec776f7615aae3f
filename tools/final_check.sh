# the whole GPU suite at HEAD, then C5 / C5TI with and without the grid column tables
timeout 1200 python -m pytest tests -q -m gpu 2>&1 | tail -3
run() { echo "== $1"; shift; env "$@" timeout 300 python bench.py --config $C --steps 30 --warmup 5 --no-fit --no-cpu-baseline 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    l=l.strip()
    if l.startswith('{'):
        d=json.loads(l); print('step %.1f us  kernel %.1f us  value %r' % (d['ms_per_step']*1e3, d['roofline']['kernel_ms']*1e3, d['metric_value']))
    elif 'Error' in l or 'error' in l: print(l)
"; }
for C in C5TI C5; do
  echo "#### $C"
  run table X=1
  run per_point PFB200_NOTDDPTAB=1
done
python __graft_entry__.py smoke 2>&1 | tail -1
