./paper_1311_1753_b200/_build/drop_in_test 2>&1 | tail -20
python -m pytest tests -m gpu -q 2>&1 | tail -8
timeout 600 python bench.py --config C3 --steps 10 --warmup 3 > gpurun_out/c3.json 2> gpurun_out/c3.err; tail -c 1800 gpurun_out/c3.json; tail -3 gpurun_out/c3.err
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/c2.json 2> gpurun_out/c2.err; python -c "import json; d=json.load(open('gpurun_out/c2.json')); print(d['ms_per_step'], d['fit'])"; tail -3 gpurun_out/c2.err
