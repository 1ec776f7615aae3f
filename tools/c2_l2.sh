for f in "" "--diag-no-flush"; do
  python bench.py --config C2 --steps 30 --warmup 5 --no-fit --no-cpu-baseline $f 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('flag=$f step %.1f us kernel %.1f us' % (d['ms_per_step']*1e3, d['roofline']['kernel_ms']*1e3))"
  python bench.py --config C2 --events 2000000 --steps 30 --warmup 5 --no-fit --no-cpu-baseline $f 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('2e6 flag=$f step %.1f us kernel %.1f us' % (d['ms_per_step']*1e3, d['roofline']['kernel_ms']*1e3))"
done
