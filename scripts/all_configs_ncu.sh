#!/bin/bash
# Per-config ncu summary of the tcgen05 GEMM launches (tensor-pipe
# utilisation, DRAM traffic and rate, SM clock) -> gpurun_out/all_configs_ncu.csv
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__bytes.sum.per_second,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second
for c in c1 c2 c3 c4 c5; do
  timeout 300 python scripts/run_once.py $c '{}' > /dev/null 2>&1
  timeout 900 ncu --metrics $M --clock-control none -k regex:ffgemm_tc --csv python scripts/run_once.py $c '{}' 2>/dev/null \
    | grep -E '"(gpu__time|dram__|lts__t_sector_hit|sm__pipe_tensor|sm__cycles)' | sed "s/^/$c,/" >> gpurun_out/all_configs_ncu.csv
done
