# setup phases (clock64, CTA 0) with the grid points split over a 2-CTA cluster
for cl in 1 2; do
  echo "== cluster $cl"
  PFB200_SETUP_CLUSTER=$cl PFB200_DEFINES="PF_SETUP_TRACE" python tools/trace_fused.py C2 2>&1 | grep "^setup" | tail -9
done
