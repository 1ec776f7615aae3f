# C5 norm kernel with and without the column table: launch durations (ncu, cold) and bench steps, alternated
for rep in 1 2; do
for v in "X=1" "PFB200_NOTDDPTAB=1"; do
  env $v timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"pf_norm" --csv --log-file gpurun_out/c5t.csv python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline --no-fit > /dev/null 2>&1
  python - "$v" <<'PY'
import csv,sys
rows=[r for r in csv.reader(open('gpurun_out/c5t.csv')) if len(r)>10]
h=rows[0]; iv=h.index('Metric Value')
print(sys.argv[1], 'norm us', [round(float(r[iv])/1000,1) for r in rows[1:]][-4:])
PY
  env $v timeout 300 python bench.py --config C5 --steps 30 --warmup 5 --no-fit --no-cpu-baseline 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    l=l.strip()
    if l.startswith('{'):
        d=json.loads(l); print('   step %.1f us' % (d['ms_per_step']*1e3))
"
done
done
