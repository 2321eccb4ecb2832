timeout 900 python tools/measure_configs.py C3 20000 nm > gpurun_out/m_c3_nm20k.json 2> gpurun_out/m_c3_nm20k.err; cat gpurun_out/m_c3_nm20k.json
timeout 900 python tools/measure_configs.py C3 20000 mono > gpurun_out/m_c3_mono20k.json 2> gpurun_out/m_c3_mono20k.err; cat gpurun_out/m_c3_mono20k.json
