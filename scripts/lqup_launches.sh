#!/bin/bash
# LQUP launch list with DRAM bytes per launch (development aid)
python paper_cs_0601133_b200/build.py > /dev/null || exit 1
N=${1:-8192}
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size --clock-control none --csv \
  --log-file gpurun_out/lqup_launches_$N.csv python scripts/run_lqup_once.py $N > /dev/null 2>&1
ls -la gpurun_out/lqup_launches_$N.csv
