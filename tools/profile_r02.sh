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
      python bench.py --steps 2 --warmup 1 --skip-cpu --c2-steps 0 > gpurun_out/ncu_launch_$TAG.log 2>&1
  echo "ncu launches rc=$?"
fi
if has c1; then
  timeout 600 $NCU -k regex:rapdb_solver_kernel --launch-skip 2 -c 1 -o gpurun_out/sweep_c1_$TAG \
      python tools/profile_sweep.py C1 1 > gpurun_out/ncu_c1_$TAG.log 2>&1; echo "ncu c1 rc=$?"
fi
if has c2; then
  timeout 900 $NCU -k regex:rapdb_solver_kernel --launch-skip 2 -c 1 -o gpurun_out/sweep_c2_$TAG \
      python tools/profile_sweep.py C2 1 > gpurun_out/ncu_c2_$TAG.log 2>&1; echo "ncu c2 rc=$?"
fi
if has c4; then
  timeout 600 $NCU -k regex:rapdb_solver_kernel --launch-skip 2 -c 1 -o gpurun_out/sweep_c4_$TAG \
      python tools/profile_sweep.py C4 1 > gpurun_out/ncu_c4_$TAG.log 2>&1; echo "ncu c4 rc=$?"
fi
if has c3; then
  # the factored kernels of a few C3f iterations (one of each kind after warm-up)
  timeout 1200 $NCU -k regex:"fac_|rapdb_solver_kernel" --launch-skip 40 -c 12 -o gpurun_out/c3_$TAG \
      python tools/c3_launches.py 6 > gpurun_out/ncu_c3_$TAG.log 2>&1; echo "ncu c3 rc=$?"
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/c3_launches_$TAG.csv python tools/c3_launches.py 20 > /dev/null 2>&1
  echo "ncu c3 launches rc=$?"
fi
