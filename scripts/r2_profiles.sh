#!/bin/bash
# Round-2 ncu evidence: one full capture each of the c4 GEMM, the c5 Winograd products P1/P2
# (CRT), the c1 latency kernel; launch lists of c4 and c5.  Each command runs plain first.
mkdir -p gpurun_out
set -x
python scripts/run_once.py c4 '{}' > /dev/null 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:ffgemm_tc -c 1 -o gpurun_out/r2_c4_full \
      python scripts/run_once.py c4 '{}' > gpurun_out/r2_c4_full.log 2>&1
python scripts/run_once.py c5 '{}' > /dev/null 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:ffgemm_tc -c 2 -o gpurun_out/r2_c5_full \
      python scripts/run_once.py c5 '{}' > gpurun_out/r2_c5_full.log 2>&1
python scripts/run_once.py c1 '{}' > /dev/null 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:lat_gemm -c 1 -o gpurun_out/r2_c1_full \
      python scripts/run_once.py c1 '{}' > gpurun_out/r2_c1_full.log 2>&1
for c in c4 c5 c3 c2 c1; do bash scripts/launch_list.sh $c '{}' r2_$c > gpurun_out/r2_ll_$c.txt 2>&1; done
ls -la gpurun_out/*.ncu-rep
