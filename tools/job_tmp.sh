python bench.py --config C3 --steps 20 > gpurun_out/r1c_c3.json 2> gpurun_out/r1c_c3.err
python bench.py --config C1 --steps 50 > gpurun_out/r1c_c1.json 2> gpurun_out/r1c_c1.err
ncu --set full --clock-control none --import-source on -k regex:"pf_event" -s 3 -c 1 -o gpurun_out/r1c_c3_event --force-overwrite python bench.py --config C3 --steps 2 --warmup 3 --no-cpu-baseline --no-fit > gpurun_out/r1c_ncu3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"pf_event" -s 3 -c 1 -o gpurun_out/r1c_c1_event --force-overwrite python bench.py --config C1 --steps 2 --warmup 3 --no-cpu-baseline --no-fit > gpurun_out/r1c_ncu1.log 2>&1
