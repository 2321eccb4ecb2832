mkdir -p gpurun_out
o=gpurun_out/r01f_configs.jsonl; : > $o
run() { timeout 600 python tools/measure_configs.py "$@" 2>>gpurun_out/cfg.err | tail -1 >> $o; }
run C0 50000 nm adaptive
run C1 20000 mono fixed500
run C1 20000 nm fixed500
run C1 20000 mono adaptive
run C1 20000 nm adaptive
run C2 5000 mono fixed500
run C2 5000 nm fixed500
run C3f 30000 mono fixed500
run C4 400000 nm fixed500
run C4 400000 mono fixed500
