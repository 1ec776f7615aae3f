python -m pytest tests -m gpu -q 2>&1 | tail -4
timeout 900 python bench.py --config C5 --steps 10 --warmup 3 > gpurun_out/c5.json 2> gpurun_out/c5.err; python -c "import json; d=json.load(open('gpurun_out/c5.json')); print('C5', d['ms_per_step'], d['value'], d['metric_value'], d['roofline']['frac'], d.get('cpu_baseline'))"; tail -3 gpurun_out/c5.err
