python -m pytest tests -m gpu -q 2>&1 | tail -3
bash tools/trace_event.sh 2>&1 | head -3
bash tools/variants.sh "" "PFB200_SETUP_CLUSTER=4" "" 2>&1
