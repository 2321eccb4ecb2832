timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -3
RAPDB_STEP_PROFILE=1 python tools/step_profile.py C1 | head -9
timeout 600 python tools/measure_configs.py C4 400000 nm fixed500 > gpurun_out/m_c4.json 2> gpurun_out/m_c4.err; cut -c1-400 gpurun_out/m_c4.json
