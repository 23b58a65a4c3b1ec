#!/bin/bash
python paper_cs_0601133_b200/build.py > /dev/null || exit 1
timeout 600 ncu --set full --import-source on --warp-sampling-interval 0 --clock-control none -k regex:panel_spec -s 2 -c 1 -o gpurun_out/panel_spec -f python scripts/run_lqup_once.py 2048 > gpurun_out/ncu_spec.log 2>&1
tail -3 gpurun_out/ncu_spec.log
