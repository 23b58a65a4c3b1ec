#!/bin/bash
# Sweep raster band / cache hints on c4 (CTA-pair kernel): ncu DRAM bytes + hit rate + tensor active.
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second
for R in 2 4 8 16 32; do for H in 0 3; do
  export FF_RASTER=$R FF_HINTS=$H
  timeout 120 python scripts/run_once.py c4 '{"cta_group":2}' > /dev/null 2>&1 && \
  timeout 300 ncu --metrics $M --clock-control none -k regex:ffgemm_tc -c 1 --csv python scripts/run_once.py c4 '{"cta_group":2}' 2>/dev/null \
    | grep -E '"(gpu__time|dram__bytes|lts__t_sector_hit|sm__pipe_tensor|sm__cycles)' | awk -F'","' -v r=$R -v h=$H '{print "R="r" H="h" "$(NF-2)" "$(NF-1)" "$NF}'
done; done
