#!/bin/bash
# A/B of FF_TRACE cycle counters (clock-independent) between scripts/ab/lib_prev.so and the current build
for c in "$@"; do
  echo "== $c prev"; FF_TRACE=1 FF_LIB_OVERRIDE=$PWD/scripts/ab/lib_prev.so python scripts/run_once.py $c '{}' 2>&1 | grep "ff trace"
  echo "== $c new";  FF_TRACE=1 python scripts/run_once.py $c '{}' 2>&1 | grep "ff trace"
done
