# C4 normalisation kernel: grid points per block (PFB200_CONV_NORM_PER)
for per in 1 8 32 256; do
  echo "== per $per"
  PFB200_CONV_NORM_PER=$per ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"pf_norm" --csv --log-file gpurun_out/c4n_$per.csv python bench.py --config C4 --steps 2 --warmup 3 --no-cpu-baseline --no-fit > /dev/null 2>&1
  python - $per <<'PY'
import csv,sys
rows=[r for r in csv.reader(open('gpurun_out/c4n_%s.csv' % sys.argv[1])) if len(r)>10]
h=rows[0]; iv=h.index('Metric Value')
print([r[iv] for r in rows[1:]][-4:])
PY
done
