nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -I. -o /tmp/sym_probe tools/sym_probe.cu
for a in "33 2 3" "100 3 3" "200 11 20" "2000 201 20" "2000 201 20 5" "2000 201 20 4" "4096 513 5"; do timeout 300 /tmp/sym_probe $a; done
