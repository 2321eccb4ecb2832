python tools/profile_sweep.py C1 30
RAPDB_LAYOUT=rows python tools/profile_sweep.py C1 30
python tools/profile_sweep.py C0 100
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -5
timeout 900 python bench.py --skip-cpu > gpurun_out/bench.json 2> gpurun_out/bench.err; cat gpurun_out/bench.json
