#!/bin/bash
# c4: L2 policy bits (FF_HINTS) x raster band: sustained time (interleaved) + ncu DRAM bytes per launch
for rep in 1 2; do
  for h in 3 6 10 2; do
    FF_HINTS=$h timeout 300 python scripts/cfg_sustained.py c4 '{}' 12 | sed "s/^/hints=$h /"
  done
done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed
for h in 3 6 10 2; do
  FF_HINTS=$h timeout 300 ncu --metrics $M --clock-control none -k regex:ffgemm_tc -c 1 --csv python scripts/run_once.py c4 '{}' 2>/dev/null \
    | grep -E '"(gpu__time|dram__bytes|lts__t_sector_hit|sm__pipe_tensor)' | awk -F'","' -v h=$h '{printf "hints=%s %s %s\n", h, $(NF-2), $NF}'
done
