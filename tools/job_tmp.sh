python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-fit > gpurun_out/c2e.json 2> gpurun_out/c2e.err; python -c "import json; d=json.load(open('gpurun_out/c2e.json')); print('C2', d['ms_per_step'], d['e2e'])"; tail -2 gpurun_out/c2e.err
