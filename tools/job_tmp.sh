BENCH_ARGS="--config C3" bash tools/variants.sh "" "PFB200_EV_BLOCKS=10 PFB200_DEFINES=PF_EVENT_MIN_BLOCKS=10" "PFB200_NSUB=8" "PFB200_DEFINES=PF_UNROLL=4" 2>&1
BENCH_ARGS="--config C4" bash tools/variants.sh "" "PFB200_NSUB=4" "PFB200_EV_BLOCKS=4" 2>&1
bash tools/variants.sh "" 2>&1
