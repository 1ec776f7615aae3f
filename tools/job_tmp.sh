python -m pytest tests -m gpu -q 2>&1 | tail -3
BENCH_ARGS="--config C3" bash tools/variants.sh "" "PFB200_EV_BLOCKS=10 PFB200_DEFINES=PF_EVENT_MIN_BLOCKS=10" 2>&1
bash tools/variants.sh "" 2>&1
python bench.py --config C1 --steps 50 --no-cpu-baseline > gpurun_out/c1.json 2>gpurun_out/c1.err; tail -c 900 gpurun_out/c1.json; tail -2 gpurun_out/c1.err
