# C5 after the mixing-factor change: TDDP tests, the bench line, the launch list
timeout 900 python -m pytest tests -q -x -m gpu -k "tddp or TDDP or C5 or dalitz or generate" 2>&1 | tail -3
for c in C5 C5TI; do
timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-fit --no-cpu-baseline 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    l=l.strip()
    if l.startswith('{'):
        d=json.loads(l); print('$c step %.1f us  kernel %.1f us  e2e %.1f us  value %r  %s frac %.3f' % (d['ms_per_step']*1e3, d['roofline']['kernel_ms']*1e3, d['e2e']['ms_per_step']*1e3, d['metric_value'], d['roofline'].get('kernel'), d['roofline']['frac']))
    elif 'Error' in l or 'error' in l: print(l)
"
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"pf_" --csv --log-file gpurun_out/c5_launches2.csv python bench.py --config C5 --steps 2 --warmup 3 --no-cpu-baseline --no-fit > /dev/null 2>&1
python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/c5_launches2.csv')) if len(r)>10]
h=rows[0]; ik=h.index('Kernel Name'); iv=h.index('Metric Value')
for r in rows[1:][-6:]: print(r[ik][:40], r[iv])
PY
