nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -I. -o /tmp/sym_probe tools/sym_probe.cu
/tmp/sym_probe 2000 201 20 0 0 0 | sed -n 2p
for ns in 12 10 8; do timeout 60 /tmp/sym_probe 2000 201 20 0 0 0 -$ns; done
timeout 60 /tmp/sym_probe 200 11 20 0 0 0 -12
timeout 60 /tmp/sym_probe 65 3 20 0 0 0 -12
timeout 60 /tmp/sym_probe 1001 7 20 0 0 0 -12
timeout 120 /tmp/sym_probe 4096 513 5 0 0 0 -11
