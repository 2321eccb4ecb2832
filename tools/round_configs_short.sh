# smoke + the configs whose sweep dominates (C2, C4 nm) with the current code
mkdir -p gpurun_out
o=gpurun_out/r01g_configs.jsonl; : > $o
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.txt 2>&1; tail -1 gpurun_out/smoke.txt
run() { timeout 600 python tools/measure_configs.py "$@" 2>>gpurun_out/cfg.err | tail -1 >> $o; }
run C1 20000 mono fixed500
run C2 5000 mono fixed500
run C4 400000 nm fixed500
