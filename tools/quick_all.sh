# after a kernel change: the parity/golden/fuzz suites, then C1-C5 step times and the C4/C5 launch lists
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_fuzz.py -q -x 2>&1 | tail -2
for c in C2 C1 C4 C5; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-fit --no-cpu-baseline 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    l=l.strip()
    if l.startswith('{'):
        d=json.loads(l); print('$c step %.1f us  kernel %.1f us  e2e %.1f us  value %r' % (d['ms_per_step']*1e3, d['roofline']['kernel_ms']*1e3, d['e2e']['ms_per_step']*1e3, d['metric_value']))
    elif 'Error' in l or 'error' in l: print(l)
"
done
for c in C4 C5; do
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"pf_" --csv --log-file gpurun_out/q_$c.csv python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-fit > /dev/null 2>&1
python - $c <<'PY'
import csv,sys
rows=[r for r in csv.reader(open('gpurun_out/q_%s.csv' % sys.argv[1])) if len(r)>10]
h=rows[0]; ik=h.index('Kernel Name'); iv=h.index('Metric Value')
print(sys.argv[1], [(r[ik][:16], r[iv]) for r in rows[1:]][-3:])
PY
done
