timeout 900 python -m pytest tests/test_gpu_factored.py -q -p no:cacheprovider -x 2>&1 | grep -E "passed|failed|Error|assert" | head
python tools/profile_grad.py C3 2
timeout 900 python tools/measure_configs.py C3 2000 mono > gpurun_out/m_c3.json 2> gpurun_out/m_c3.err; tail -2 gpurun_out/m_c3.err; cat gpurun_out/m_c3.json
