# C4 event pass: shared-memory copy of S or not, 8 or 16 two-warp blocks per SM; the norm kernel's S copy
run() { echo "== $1"; shift; env "$@" python bench.py --config C4 --steps 20 --warmup 5 --no-fit --no-cpu-baseline 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    l=l.strip()
    if l.startswith('{'):
        d=json.loads(l); print('step %.1f us  kernel %.1f us  e2e %.1f us  value %r  %s frac %.3f' % (d['ms_per_step']*1e3, d['roofline']['kernel_ms']*1e3, d['e2e']['ms_per_step']*1e3, d['metric_value'], d['roofline'].get('kernel'), d['roofline']['frac']))
    elif 'Error' in l or 'error' in l: print(l[:300])
"; }
run A_default X=1
run B_s_global PFB200_EVENT_S_SMEM=0
run C_s_global_16 PFB200_EVENT_S_SMEM=0 PFB200_EV_BLOCKS=16 PFB200_DEFINES=PF_EVENT_MIN_BLOCKS=16
run D_16 PFB200_EV_BLOCKS=16 PFB200_DEFINES=PF_EVENT_MIN_BLOCKS=16
run E_s_global_12 PFB200_EVENT_S_SMEM=0 PFB200_EV_BLOCKS=12 PFB200_DEFINES=PF_EVENT_MIN_BLOCKS=12
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"pf_" --csv --log-file gpurun_out/c4_launches2.csv python bench.py --config C4 --steps 2 --warmup 3 --no-cpu-baseline --no-fit > /dev/null 2>&1
python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/c4_launches2.csv')) if len(r)>10]
h=rows[0]; ik=h.index('Kernel Name'); iv=h.index('Metric Value')
for r in rows[1:][-6:]: print(r[ik][:40], r[iv])
PY
python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_golden.py tests/test_gpu_sizes.py -q -k "conv or C4 or golden or bw" 2>&1 | tail -3
