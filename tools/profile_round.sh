timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -2
python bench.py > gpurun_out/bench_r01c.json 2> gpurun_out/bench_r01c.err; echo "bench rc=$?"
cat gpurun_out/bench_r01c.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r01c.csv python bench.py --steps 2 --warmup 1 --skip-cpu > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
ncu --set full --import-source on --clock-control none -k regex:rapdb_solver_kernel --launch-skip 2 -c 1 -o gpurun_out/sweep_c1_r01c python tools/profile_sweep.py C1 1 > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
