for v in "X=1"; do
  echo "== $v (setup phases, cycles)"
  env $v PFB200_DEFINES="PF_EVENT_TRACE;PF_SETUP_TRACE" python tools/trace_fused.py C2 2>&1 | grep "^setup" | tail -9
  echo "== $v (timeline)"
  env $v PFB200_DEFINES="PF_EVENT_TRACE" python tools/trace_fused.py C2 2>&1 | tail -14
done
