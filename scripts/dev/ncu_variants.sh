#!/bin/bash
# usage: CFG=c4 bash scripts/ncu_variants.sh 'label|ENV=..|{json}' ...   -> one summary line per variant
M=gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second
CFG=${CFG:-c4}
for spec in "$@"; do
  IFS='|' read -r label envs opts <<< "$spec"
  (export $envs; timeout 200 python scripts/run_once.py $CFG "$opts" > /dev/null 2>&1 && \
   timeout 900 ncu $NCU_EXTRA --metrics $M --clock-control none -k regex:ffgemm_tc -c 1 --csv python scripts/run_once.py $CFG "$opts" 2>/dev/null \
   | grep -E '"(gpu__time|dram__bytes|lts__t_sector_hit|sm__pipe_tensor|sm__cycles)' \
   | awk -F'","' -v l="$label" '{printf "%s %s %s\n", l, $(NF-2), $NF}')
done
