#!/bin/bash
# Sweep raster band x k-block length (locality) on a config: ncu DRAM bytes + time + tensor active.
CFG=${CFG:-c4}
M=gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second
for R in ${RS:-8 16}; do for KB in ${KBS:-0 4096 2048 1024}; do
  export FF_RASTER=$R FF_HINTS=${HINTS:-3}
  O="{\"cta_group\":2,\"kb_override\":$KB}"
  timeout 120 python scripts/run_once.py $CFG "$O" > /dev/null 2>&1 && \
  timeout 300 ncu --metrics $M --clock-control none -k regex:ffgemm_tc -c 1 --csv python scripts/run_once.py $CFG "$O" 2>/dev/null \
    | grep -E '"(gpu__time|dram__bytes|lts__t_sector_hit|sm__pipe_tensor|sm__cycles)' | awk -F'","' -v r=$R -v kb=$KB '{printf "R=%s KB=%s %s %s\n", r, kb, $(NF-2), $NF}'
done; done
