#!/bin/bash
# compute-sanitizer over every device op (tools/sanitize_cases.py), on a B200:
#   gpurun --timeout 3000 -- 'bash tools/sanitize.sh'
# logs -> gpurun_out/sanitize/<tool>_<case>.log, summary -> gpurun_out/sanitize/summary.txt
mkdir -p gpurun_out/sanitize
out=gpurun_out/sanitize
: > $out/summary.txt
CASES=${CASES:-"run gap early rows factored factored_fused peer comm egm probe"}
TOOLS=${TOOLS:-"memcheck racecheck synccheck initcheck"}
for tool in $TOOLS; do
  for c in $CASES; do
    extra=""
    [ "$tool" = "memcheck" ] && extra="--leak-check full"
    [ "$tool" = "racecheck" ] && extra="--racecheck-report all"
    timeout 900 compute-sanitizer --tool $tool $extra --error-exitcode 9 --target-processes all \
        python tools/sanitize_cases.py $c > $out/${tool}_${c}.log 2>&1
    rc=$?
    errs=$(grep -E "ERROR SUMMARY|RACECHECK SUMMARY|LEAK SUMMARY" $out/${tool}_${c}.log | tr '\n' ' ')
    echo "$tool $c rc=$rc $errs" | tee -a $out/summary.txt
  done
done
