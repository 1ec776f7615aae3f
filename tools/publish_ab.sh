# record publish: volatile stores + system-scope release (default) vs uncached MMIO stores, no fence
run() { echo "== $1"; shift; env "$@" timeout 300 python bench.py --config C2 --steps 30 --warmup 5 --no-fit --no-cpu-baseline 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    l=l.strip()
    if l.startswith('{'):
        d=json.loads(l); print('step %.1f us  kernel %.1f us  e2e %.1f us (mean %.1f)  value %r' % (d['ms_per_step']*1e3, d['roofline']['kernel_ms']*1e3, d['e2e']['ms_per_step']*1e3, d['e2e']['ms_per_step_mean']*1e3, d['metric_value']))
    elif 'Error' in l or 'error' in l: print(l)
"; }
for rep in 1 2; do
  run release X=1
  run mmio PFB200_DEFINES=PF_PUBLISH_MMIO
done
PFB200_DEFINES=PF_PUBLISH_MMIO timeout 300 python tools/e2e_probe.py 2>&1 | tail -4
PFB200_DEFINES=PF_PUBLISH_MMIO timeout 600 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2
