# C5 / C5TI: parameters, constants and S in the event pass's shared memory (PF_PC_SMEM) vs global (PFB200_NOPCSMEM)
timeout 600 python -m pytest tests -q -m gpu -x -k "tddp or TDDP or dalitz or C5 or golden" 2>&1 | tail -2
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
  run pc_smem X=1
  run global PFB200_NOPCSMEM=1
done
