#!/bin/bash
# Reproduce the profiles/ evidence on a B200 (run through gpurun), then
# summarise here with tools/summarize_ncu.py:
#   gpurun --timeout 2700 -- 'TAG=r02 bash tools/profile_round.sh'
#   python tools/summarize_ncu.py full gpurun_out/sweep_c1_$TAG.ncu-rep profiles/${TAG}_sweep_c1_packed --bytes 3319529472
#   python tools/summarize_ncu.py launches gpurun_out/launches_$TAG.csv profiles/${TAG}_launches
TAG=${TAG:-r01c}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -2
python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
cat gpurun_out/bench_$TAG.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$TAG.csv \
    python bench.py --steps 2 --warmup 1 --skip-cpu > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
ncu --set full --import-source on --clock-control none -k regex:rapdb_solver_kernel --launch-skip 2 -c 1 \
    -o gpurun_out/sweep_c1_$TAG python tools/profile_sweep.py C1 1 > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
