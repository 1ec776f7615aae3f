python -m pytest tests -m gpu -q 2>&1 | tail -3
BENCH_ARGS="--config C4" bash tools/variants.sh "" "PFB200_NSUB=4" 2>&1
