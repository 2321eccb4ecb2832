#!/bin/bash
# C3f (factored path) check + timing round on one B200:
#   gpurun --timeout 2400 -- 'TAG=r02d bash tools/c3_round.sh'
TAG=${TAG:-r02d}
PARTS=${PARTS:-"tests times kkt"}
mkdir -p gpurun_out
has() { [[ " $PARTS " == *" $1 "* ]]; }
if has tests; then
  timeout 1500 python -m pytest tests/test_gpu_factored.py tests/test_gpu_memcheck.py tests/test_gpu_sharding.py \
      tests/test_gpu_endtoend.py -k "factored or c3f or phases or scipy" -x -q -p no:cacheprovider \
      > gpurun_out/pytest_c3_$TAG.log 2>&1
  echo "pytest rc=$?"; tail -15 gpurun_out/pytest_c3_$TAG.log
fi
if has times; then
  for rows in ${PHASE_ROWS:-8388608 4194304 2097152 1048576}; do
    echo "== RAPDB_RT_PHASE_ROWS=$rows"
    RAPDB_RT_PHASE_ROWS=$rows timeout 600 python tools/kernel_times.py C3f 100 2>&1 | tail -22
  done > gpurun_out/c3_times_$TAG.log 2>&1
  cat gpurun_out/c3_times_$TAG.log
fi
if has kkt; then
  timeout 900 python tools/measure_configs.py C3f 3000 > gpurun_out/c3f_kkt_$TAG.json 2> gpurun_out/c3f_kkt_$TAG.err
  echo "C3f to KKT rc=$?"; cat gpurun_out/c3f_kkt_$TAG.json
fi
if has ncu; then
  NCU="ncu --set full --import-source on --clock-control none"
  timeout 1200 $NCU -k regex:"fac_" --launch-skip 30 -c 8 -o gpurun_out/c3_$TAG \
      python tools/c3_launches.py 6 > gpurun_out/ncu_c3_$TAG.log 2>&1; echo "ncu c3 rc=$?"
  python tools/summarize_ncu.py multi gpurun_out/c3_$TAG.ncu-rep gpurun_out/c3_$TAG > gpurun_out/c3_${TAG}_summary.log 2>&1
  cat gpurun_out/c3_${TAG}_summary.log
  rm -f gpurun_out/c3_$TAG.ncu-rep
fi
