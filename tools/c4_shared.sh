# C4: warp-shared convolution window products vs per-lane (PFB200_NOCONVSHARED), the conv tests, the launch list
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_golden.py tests/test_gpu_sizes.py -q -x -k "conv or C4 or golden or bw" 2>&1 | tail -3
run() { echo "== $1"; shift; env "$@" timeout 300 python bench.py --config C4 --steps 20 --warmup 5 --no-fit --no-cpu-baseline 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    l=l.strip()
    if l.startswith('{'):
        d=json.loads(l); print('step %.1f us  kernel %.1f us  e2e %.1f us  value %r  %s frac %.3f' % (d['ms_per_step']*1e3, d['roofline']['kernel_ms']*1e3, d['e2e']['ms_per_step']*1e3, d['metric_value'], d['roofline'].get('kernel'), d['roofline']['frac']))
    elif 'Error' in l or 'error' in l: print(l)
"; }
run shared X=1
run per_lane PFB200_NOCONVSHARED=1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"pf_" --csv --log-file gpurun_out/c4_launches.csv python bench.py --config C4 --steps 2 --warmup 3 --no-cpu-baseline --no-fit > /dev/null 2>&1
python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/c4_launches.csv')) if len(r)>10]
h=rows[0]; ik=h.index('Kernel Name'); iv=h.index('Metric Value')
for r in rows[1:][-6:]: print(r[ik][:40], r[iv])
PY
