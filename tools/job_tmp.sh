python -m pytest tests -m gpu -q 2>&1 | tail -3
python bench.py > gpurun_out/r1d_c2.json 2> gpurun_out/r1d_c2.err; python -c "import json; d=json.load(open('gpurun_out/r1d_c2.json')); print('C2', d['ms_per_step'], d['value'], d['e2e'], d.get('fit'), d.get('cpu_baseline'))"; tail -2 gpurun_out/r1d_c2.err
python bench.py --impl reference > gpurun_out/r1d_c2_ref.json 2> gpurun_out/r1d_c2_ref.err; cat gpurun_out/r1d_c2_ref.json | cut -c1-300
python __graft_entry__.py smoke 2>&1 | tail -2
