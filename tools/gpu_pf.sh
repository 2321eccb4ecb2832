nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -I. -o /tmp/sym_probe tools/sym_probe.cu
for v in 0 2 1; do /tmp/sym_probe 2000 201 20 0 0 $v | sed -n 2p; done
for v in 0 2; do /tmp/sym_probe 2000 201 20 4 0 $v | sed -n 2p; done
