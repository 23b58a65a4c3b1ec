#!/bin/bash
python paper_cs_0601133_b200/build.py > /dev/null || exit 1
for g in 2 4 6 8; do echo "group $g"; FF_LQUP_GROUP=$g timeout 300 python scripts/lqup_time.py 8192 16384 2>&1; done | tee gpurun_out/group_sweep.txt
