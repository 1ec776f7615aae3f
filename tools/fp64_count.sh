# FP64 instruction counts of each config's dominant kernel (ncu SASS op
# counters, one launch), for the FP64 roofline of bench.py: flops per unit =
# (DADD + DMUL + 2 DFMA) thread instructions / units.  Plain run first (ncu
# only profiles a command that has just exited 0 without it).
TAG=${1:-r2}
M=sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__sass_thread_inst_executed_op_dfma_pred_on.sum,gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum
for spec in "C2 pf_fused_kernel 10000000" "C4 pf_event_kernel 1000000" "C5 pf_event_kernel 1000000" "C5TI pf_event_kernel 1000000"; do
  set -- $spec
  CMD="python bench.py --config $1 --events $3 --steps 2 --warmup 2 --no-fit --no-cpu-baseline"
  $CMD > gpurun_out/fp64_plain_$1.log 2>&1 && \
  ncu --metrics $M --clock-control none -k regex:$2 -s 3 -c 1 --csv --log-file gpurun_out/${TAG}_fp64_$1.csv $CMD > gpurun_out/fp64_ncu_$1.log 2>&1
done
