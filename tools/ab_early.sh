#!/bin/bash
# A/B of the packed sweep's early reduction: builds in build/*.so x chunk counts,
# C1 (mono) and C4 (nm) solves; prints the per-solve kernel times and the
# stream / reduce sub-phases.   usage: tools/ab_early.sh build/a.so build/b.so ...
for lib in "$@"; do
  for ch in ${CHUNKS:-0 4 8}; do
    for cfg in "C1" "C4 nm"; do
      echo "== $lib chunks=$ch $cfg"
      RAPDB_LIB=$lib RAPDB_EARLY_CHUNKS=$ch RAPDB_STEP_PROFILE=1 REPS=${REPS:-4} timeout 300 \
        python tools/step_profile.py $cfg 2>&1 | grep -E "^solve|sweep:stream|sweep:reduce"
    done
  done
done
