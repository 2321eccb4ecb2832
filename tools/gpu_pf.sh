nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -I. -o /tmp/sym_probe tools/sym_probe.cu
/tmp/sym_probe 2000 201 20 0 0 0 | sed -n 2p
for W in 8 16 32; do timeout 60 /tmp/sym_probe 2000 201 20 0 0 0 $W; done
timeout 120 /tmp/sym_probe 4096 513 5 0 0 0 8
