#!/bin/bash
# One complete measurement round: GPU tests, every BASELINE config's bench line
# and reference arm, ncu launch list + full captures, exchange paths, smoke.
# Usage (on the GPU box): bash tools/final_round.sh TAG   -> gpurun_out/TAG_*
T=${1:-r2}
O=gpurun_out
nproc > $O/${T}_host.txt; lscpu | grep -E "Model name|Thread|Core|Socket" >> $O/${T}_host.txt
python __graft_entry__.py smoke > $O/${T}_smoke.txt 2>&1
python -m pytest tests -m gpu -q > $O/${T}_pytest_gpu.txt 2>&1
python bench.py --steps 20 --warmup 5 > $O/${T}_c2.json 2> $O/${T}_c2.err
python bench.py --impl reference --steps 20 --warmup 5 > $O/${T}_c2_ref.json 2> $O/${T}_c2_ref.err
for c in C1 C3 C4 C5 C5TI; do
  python bench.py --config $c --steps 20 > $O/${T}_${c,,}.json 2> $O/${T}_${c,,}.err
  python bench.py --config $c --impl reference --steps 3 --warmup 1 > $O/${T}_${c,,}_ref.json 2> $O/${T}_${c,,}_ref.err
done
for ex in p2p nccl; do
  python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29515 \
    bench.py --force-exchange --exchange $ex --steps 30 --warmup 3 --no-fit --no-cpu-baseline 2> $O/${T}_x_$ex.err | tail -1 > $O/${T}_x_$ex.json
done
python -m paper_1311_1753_b200 bench --workload C2 --gpus 1 2 --repetitions 3 > $O/${T}_cli_bench.txt 2>&1
CMD="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-fit"
$CMD > $O/${T}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"pf_" --csv --log-file $O/${T}_launches.csv $CMD > $O/${T}_ncu_l.log 2>&1
for spec in "C1 pf_fused" "C2 pf_fused" "C3 pf_fused" "C4 pf_event" "C5 pf_event"; do
  set -- $spec
  CMD="python bench.py --config $1 --steps 2 --warmup 3 --no-cpu-baseline --no-fit"
  $CMD > $O/${T}_plain_${1,,}.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"$2" -s 3 -c 1 -o $O/${T}_${1,,}_event \
    --force-overwrite $CMD > $O/${T}_ncu_${1,,}.log 2>&1
done
CMD="python bench.py --config C5 --steps 2 --warmup 3 --no-cpu-baseline --no-fit"
ncu --set full --clock-control none --import-source on -k regex:"pf_norm" -s 1 -c 1 -o $O/${T}_c5_norm \
  --force-overwrite $CMD > $O/${T}_ncu_c5norm.log 2>&1
for c in C4 C5; do
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"pf_" --csv --log-file $O/${T}_${c,,}_launches.csv \
    python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-fit > /dev/null 2>&1
done
python tools/gen_probe.py 10000000 1000000 > $O/${T}_generate_1e7.json 2> $O/${T}_generate.err
bash tools/fp64_count.sh $T > $O/${T}_fp64_count.log 2>&1
PFB200_DEFINES="PF_EVENT_TRACE" python tools/trace_fused.py C2 > $O/${T}_trace_c2.txt 2>&1
python tools/e2e_probe.py > $O/${T}_e2e_probe.txt 2>&1
