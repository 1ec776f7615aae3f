# C5 / C5TI: the norm kernel's column table (channel A per column) vs per point (PFB200_NOTDDPTAB)
timeout 600 python -m pytest tests -q -m gpu -x -k "tddp or TDDP or dalitz or C5 or golden or generate" 2>&1 | tail -2
run() { echo "== $1"; shift; env "$@" timeout 300 python bench.py --config $C --steps 20 --warmup 5 --no-fit --no-cpu-baseline 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    l=l.strip()
    if l.startswith('{'):
        d=json.loads(l); print('step %.1f us  kernel %.1f us  value %r' % (d['ms_per_step']*1e3, d['roofline']['kernel_ms']*1e3, d['metric_value']))
    elif 'Error' in l or 'error' in l: print(l)
"; }
for C in C5 C5TI; do
  echo "#### $C"
  run table X=1
  run per_point PFB200_NOTDDPTAB=1
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"pf_" --csv --log-file gpurun_out/c5t.csv python bench.py --config C5 --steps 2 --warmup 3 --no-cpu-baseline --no-fit > /dev/null 2>&1
python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/c5t.csv')) if len(r)>10]
h=rows[0]; ik=h.index('Kernel Name'); iv=h.index('Metric Value')
print([(r[ik][:16], r[iv]) for r in rows[1:]][-3:])
PY
