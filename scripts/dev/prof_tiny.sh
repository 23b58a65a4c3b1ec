#!/bin/bash
python paper_cs_0601133_b200/build.py > /dev/null || exit 1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:ffgemm_tc -s 2 -c 1 -o gpurun_out/tiny -f python scripts/tiny_once.py > gpurun_out/ncu_tiny.log 2>&1
FF_TRACE=1 timeout 60 python scripts/tiny_once.py 2>&1 | grep "ff trace" | tail -1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none python scripts/tiny_once.py 2>&1 | grep -E "ffgemm|encode|duration" | head -20
