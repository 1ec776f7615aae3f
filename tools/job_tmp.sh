python -m pytest tests -m gpu -q 2>&1 | tail -3
bash tools/trace_event.sh 2>&1 | head -3
bash tools/variants.sh "" "PFB200_DEFINES=PF_PUBLISH_FENCE" "" "PFB200_DEFINES=PF_PUBLISH_FENCE" 2>&1
