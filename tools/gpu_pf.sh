nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -I. -o /tmp/sym_probe tools/sym_probe.cu
for v in 0 3 0 3; do /tmp/sym_probe 2000 201 20 0 0 $v | sed -n 2p; done
for v in 0 3; do /tmp/sym_probe 4096 513 5 0 0 $v | sed -n 2p; done
