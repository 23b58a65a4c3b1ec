#!/bin/bash
# LQUP: tests, then timing (default, no deferral, no speculation).
python paper_cs_0601133_b200/build.py > /dev/null || exit 1
timeout 600 python -m pytest tests/test_gpu_lqup.py -x -q 2>&1 | tail -15 > gpurun_out/pytest_lqup_spec.log
cat gpurun_out/pytest_lqup_spec.log
timeout 300 python scripts/lqup_time.py 4096 8192 16384 2>&1 | tee gpurun_out/lqup_spec_time.txt
FF_LQUP_GROUP=1 timeout 300 python scripts/lqup_time.py 8192 16384 2>&1 | tee -a gpurun_out/lqup_spec_time.txt
