#!/bin/bash
# Round-2 evidence on one B200 (run through gpurun):
#   gpurun --timeout 3600 -- 'TAG=r02c bash tools/profile_r02.sh'
# then summarise here with tools/summarize_ncu.py (full captures) and
# tools/summarize_ncu.py launches (launch list).
# PARTS selects steps (default: all).
TAG=${TAG:-r02c}
PARTS=${PARTS:-"tests smoke bench launches c1 c2 c4 c3"}
mkdir -p gpurun_out
has() { [[ " $PARTS " == *" $1 "* ]]; }
NCU="ncu --set full --import-source on --clock-control none"
LIB=paper_2605_29291_b200/_rapdb_b200.so
# gpurun merges back at most 64 MiB: summarise every full capture on the box
# (raw metrics JSON, details CSV, hottest source lines) and drop the report
summ() {  # summ <name> <algorithmic bytes> [kernel]
  local rep=gpurun_out/$1_$TAG.ncu-rep
  [ -f "$rep" ] || { echo "no report $rep"; return; }
  python tools/summarize_ncu.py full "$rep" gpurun_out/$1_$TAG --bytes "$2" > gpurun_out/$1_${TAG}_summary.log 2>&1
  python tools/ncu_hot.py "$rep" $LIB "${3:-rapdb_solver_kernel}" 40 > gpurun_out/$1_${TAG}_hot.txt 2>&1
  rm -f "$rep"
}
if has tests; then
  timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_$TAG.log 2>&1
  echo "pytest rc=$?"; tail -3 gpurun_out/pytest_$TAG.log
fi
if has smoke; then
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"
  tail -1 gpurun_out/smoke_$TAG.log
fi
if has bench; then
  timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
  cat gpurun_out/bench_$TAG.json
fi
if has launches; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
      --log-file gpurun_out/launches_$TAG.csv \
      python bench.py --steps 2 --warmup 1 --skip-cpu --c2-steps 0 --c3-steps 0 > gpurun_out/ncu_launch_$TAG.log 2>&1
  echo "ncu launches rc=$?"
fi
if has c1; then
  timeout 600 $NCU -k regex:rapdb_solver_kernel --launch-skip 2 -c 1 -o gpurun_out/sweep_c1_$TAG \
      python tools/profile_sweep.py C1 1 > gpurun_out/ncu_c1_$TAG.log 2>&1; echo "ncu c1 rc=$?"
  summ sweep_c1 $(cat gpurun_out/streamed_C1.txt)
fi
if has c2; then
  timeout 900 $NCU -k regex:rapdb_solver_kernel --launch-skip 2 -c 1 -o gpurun_out/sweep_c2_$TAG \
      python tools/profile_sweep.py C2 1 > gpurun_out/ncu_c2_$TAG.log 2>&1; echo "ncu c2 rc=$?"
  summ sweep_c2 $(cat gpurun_out/streamed_C2.txt)
fi
if has c4; then
  timeout 600 $NCU -k regex:rapdb_solver_kernel --launch-skip 2 -c 1 -o gpurun_out/sweep_c4_$TAG \
      python tools/profile_sweep.py C4 1 > gpurun_out/ncu_c4_$TAG.log 2>&1; echo "ncu c4 rc=$?"
  summ sweep_c4 $(cat gpurun_out/streamed_C4.txt)
fi
if has gather; then
  ./tools/gather_probe > gpurun_out/gather_probe_$TAG.json 2> gpurun_out/gather_probe_$TAG.err; echo "gather probe rc=$?"
  tail -c 1500 gpurun_out/gather_probe_$TAG.json
fi
if has c0grid; then
  for g in 148 64 32 16 8; do
    echo "RAPDB_GRID=$g"; RAPDB_GRID=$g python tools/measure_configs.py C0 5000 nm adaptive 2>&1 | tail -12
  done > gpurun_out/c0grid_$TAG.log 2>&1
  cat gpurun_out/c0grid_$TAG.log
fi
if has valc4; then
  timeout 3000 python tools/validate_long.py C4 nm 3000 > gpurun_out/validate_long_c4nm_$TAG.json 2> gpurun_out/validate_long_c4nm_$TAG.err
  echo "validate C4 nm rc=$?"; cut -c1-700 gpurun_out/validate_long_c4nm_$TAG.json
fi
if has valc2; then
  timeout 5400 python tools/validate_long.py C2 mono 600 > gpurun_out/validate_long_c2mono_$TAG.json 2> gpurun_out/validate_long_c2mono_$TAG.err
  echo "validate C2 mono to KKT rc=$?"; cut -c1-700 gpurun_out/validate_long_c2mono_$TAG.json
fi
if has valc2nm; then
  timeout 5400 python tools/validate_full.py C2 200 > gpurun_out/validate_c2_full_$TAG.json 2> gpurun_out/validate_c2_full_$TAG.err
  echo "validate C2 200 rc=$?"; cat gpurun_out/validate_c2_full_$TAG.json
fi
if has c3; then
  # the factored kernels of a few C3f iterations (one of each kind after warm-up)
  timeout 1200 $NCU -k regex:"fac_|rapdb_solver_kernel" --launch-skip 40 -c 12 -o gpurun_out/c3_$TAG \
      python tools/c3_launches.py 6 > gpurun_out/ncu_c3_$TAG.log 2>&1; echo "ncu c3 rc=$?"
  python tools/summarize_ncu.py multi gpurun_out/c3_$TAG.ncu-rep gpurun_out/c3_$TAG > gpurun_out/c3_${TAG}_summary.log 2>&1
  for k in fac_grad_kernel fac_row_kernel; do
    python tools/ncu_hot.py gpurun_out/c3_$TAG.ncu-rep $LIB $k 30 > gpurun_out/c3_${TAG}_hot_$k.txt 2>&1
  done
  rm -f gpurun_out/c3_$TAG.ncu-rep
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/c3_launches_$TAG.csv python tools/c3_launches.py 20 > /dev/null 2>&1
  echo "ncu c3 launches rc=$?"
fi
