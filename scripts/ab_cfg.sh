#!/bin/bash
# A/B of the current build against scripts/ab/lib_prev.so on one box, interleaved:
#   bash scripts/ab_cfg.sh c5 3
CFG=${1:-c5}; REPS=${2:-3}
for r in $(seq $REPS); do
  FF_LIB_OVERRIDE=$PWD/scripts/ab/lib_prev.so timeout 300 python scripts/cfg_sustained.py $CFG '{}' ${STEPS:-10} | sed 's/^/prev /'
  timeout 300 python scripts/cfg_sustained.py $CFG '{}' ${STEPS:-10} | sed 's/^/new  /'
done
