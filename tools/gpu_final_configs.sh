timeout 600 python tools/measure_configs.py C0 50000 nm adaptive > gpurun_out/f_c0.json 2>/dev/null
timeout 600 python tools/measure_configs.py C2 3000 mono > gpurun_out/f_c2.json 2>/dev/null
timeout 900 python tools/measure_configs.py C3f 30000 mono > gpurun_out/f_c3f.json 2>/dev/null
timeout 900 python tools/measure_configs.py C4 400000 nm fixed500 > gpurun_out/f_c4.json 2>/dev/null
timeout 600 python tools/measure_configs.py C1 20000 mono adaptive > gpurun_out/f_c1ada.json 2>/dev/null
for f in f_c0 f_c2 f_c3f f_c4 f_c1ada; do python -c "import json; d=json.load(open('gpurun_out/$f.json')); print('$f', d['iterations'], d['converged'], round(d['wall_s'],3), round(d['ms_per_iter'],4))"; done
