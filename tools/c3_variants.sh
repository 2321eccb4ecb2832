#!/bin/bash
# A/B builds of the factored path's standalone kernels (csrc/factored.cuh
# tunables) into scratch/variants/, and their per-kernel times on a B200:
#   bash tools/c3_variants.sh build "name:-DRAPDB_ROWU=10 -DRAPDB_ROWCTAS=4" ...     (here)
#   gpurun -- 'bash tools/c3_variants.sh run name ...'                                (GPU box)
cd "$(dirname "$0")/.."
mode=$1; shift
if [ "$mode" = build ]; then
  mkdir -p scratch/variants
  NCCL_HOME=$(python3 -c "import nvidia.nccl as m; print(list(m.__path__)[0])")
  for spec in "$@"; do
    name=${spec%%:*}; flags=${spec#*:}
    ( nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -Xptxas -v -Xcompiler -fPIC \
        -shared -Iinclude -I$NCCL_HOME/include $flags -o scratch/variants/$name.so paper_2605_29291_b200/csrc/solver.cu \
        -L$NCCL_HOME/lib -Xlinker -rpath=$NCCL_HOME/lib -l:libnccl.so.2 2> scratch/variants/$name.log
      echo "$name [$flags]: $(grep -A2 -E 'fac_row_kernel|fac_grad_kernelILb1' scratch/variants/$name.log | grep -oE '[0-9]+ bytes spill loads|Used [0-9]+ registers' | tr '\n' ' ')" ) &
  done
  wait
else
  for name in "$@"; do
    echo "== $name"
    RAPDB_LIB=$PWD/scratch/variants/$name.so timeout 300 python tools/kernel_times.py C3f 60 2>&1 | grep -E "fac_row|fac_grad_kernel|per eval"
  done
fi
