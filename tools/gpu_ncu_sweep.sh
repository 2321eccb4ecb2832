nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -I. -o /tmp/sym_probe tools/sym_probe.cu
ncu --set full --import-source on --clock-control none -k regex:rapdb_solver_kernel -c 1 -o gpurun_out/sweep_c1_packed python tools/profile_sweep.py C1 1 > gpurun_out/ncu_sweep.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:phase_a -c 1 -o gpurun_out/proto_phase_a /tmp/sym_probe 2000 201 1 > gpurun_out/ncu_proto.log 2>&1
ls -la gpurun_out
