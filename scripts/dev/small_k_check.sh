#!/bin/bash
python paper_cs_0601133_b200/build.py > /dev/null || exit 1
timeout 300 python scripts/small_k.py | tee gpurun_out/small_k.txt
timeout 300 python scripts/lqup_time.py 8192 16384 2>&1 | tee -a gpurun_out/small_k.txt
