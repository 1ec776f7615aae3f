# C5 norm kernel: run length (points per thread run) 32 / 16 / 8 at 2 blocks per SM
for r in 64 48; do
  echo "== run $r"
  PFB200_NORM_RUN=$r PFB200_DEFINES="PF_NORM_RUN=$r" timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"pf_" --csv --log-file gpurun_out/c5n.csv python bench.py --config C5 --steps 2 --warmup 3 --no-cpu-baseline --no-fit > /dev/null 2>&1
  python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/c5n.csv')) if len(r)>10]
h=rows[0]; ik=h.index('Kernel Name'); iv=h.index('Metric Value')
print([(r[ik][:16], r[iv]) for r in rows[1:]][-3:])
PY
  PFB200_NORM_RUN=$r PFB200_DEFINES="PF_NORM_RUN=$r" timeout 300 python bench.py --config C5 --steps 20 --warmup 5 --no-fit --no-cpu-baseline 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    l=l.strip()
    if l.startswith('{'):
        d=json.loads(l); print('step %.1f us  kernel %.1f us  value %r' % (d['ms_per_step']*1e3, d['roofline']['kernel_ms']*1e3, d['metric_value']))
"
done
