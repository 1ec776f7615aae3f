# setup phases traced twice in one kernel: the second pass runs from warm instruction caches
PFB200_DEFINES="PF_SETUP_TRACE;PF_SETUP_TWICE" python tools/trace_fused.py C2 2>&1 | grep "^setup" | tail -18
PFB200_DEFINES="PF_SETUP_TRACE;PF_SETUP_TWICE" python tools/trace_fused.py C1 2>&1 | grep "^setup" | tail -18
