for v in "X=1" "PFB200_DEFINES=PF_NO_L2_PREFETCH"; do
  echo "== $v (timeline)"
  env $v python -c "import os; os.environ['PFB200_DEFINES']=(os.environ.get('PFB200_DEFINES','')+';PF_EVENT_TRACE').strip(';'); import runpy, sys; sys.argv=['t','C2']; runpy.run_path('tools/trace_fused.py', run_name='__main__')" 2>&1 | tail -14
done
