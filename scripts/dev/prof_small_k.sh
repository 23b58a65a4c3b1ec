#!/bin/bash
python paper_cs_0601133_b200/build.py > /dev/null || exit 1
timeout 300 python scripts/small_k.py | tee gpurun_out/small_k.txt
timeout 600 ncu --set full --import-source on --clock-control none -k regex:ffgemm_tc -c 1 -o gpurun_out/small_k -f python scripts/small_k.py once > gpurun_out/ncu_small_k.log 2>&1
tail -2 gpurun_out/ncu_small_k.log
