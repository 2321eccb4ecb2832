timeout 900 python -m pytest tests/test_gpu_factored.py tests/test_gpu_sharding.py -q -p no:cacheprovider -x 2>&1 | tail -3
python tools/profile_grad.py C3 2
RAPDB_FAC_HOST=0 python tools/profile_grad.py C3 2
timeout 900 python tools/measure_configs.py C3f 30000 mono > gpurun_out/m_c3f.json 2> gpurun_out/m_c3f.err; tail -2 gpurun_out/m_c3f.err; python -c "import json; d=json.load(open('gpurun_out/m_c3f.json')); print(d['iterations'], d['converged'], d['wall_s'], d['ms_per_iter'], d['step_profile_ms'])"
