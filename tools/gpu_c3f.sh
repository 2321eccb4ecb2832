timeout 1200 python tools/measure_configs.py C3f 30000 mono > gpurun_out/m_c3f_mono.json 2> gpurun_out/m_c3f_mono.err; cat gpurun_out/m_c3f_mono.json; tail -2 gpurun_out/m_c3f_mono.err
