timeout 600 python tools/measure_configs.py C2 3000 mono > gpurun_out/m_c2_mono.json 2> gpurun_out/m_c2_mono.err; tail -2 gpurun_out/m_c2_mono.err; cat gpurun_out/m_c2_mono.json
timeout 600 python tools/measure_configs.py C0 50000 nm adaptive > gpurun_out/m_c0.json 2> gpurun_out/m_c0.err; tail -2 gpurun_out/m_c0.err; cat gpurun_out/m_c0.json
timeout 900 python tools/measure_configs.py C4 400000 nm fixed500 > gpurun_out/m_c4.json 2> gpurun_out/m_c4.err; tail -2 gpurun_out/m_c4.err; cat gpurun_out/m_c4.json
timeout 900 python tools/measure_configs.py C3 2000 mono > gpurun_out/m_c3.json 2> gpurun_out/m_c3.err; tail -2 gpurun_out/m_c3.err; cat gpurun_out/m_c3.json
