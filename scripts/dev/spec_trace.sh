#!/bin/bash
python paper_cs_0601133_b200/build.py > /dev/null || exit 1
FF_LQUP_TRACE=1 timeout 120 python scripts/run_lqup_once.py 2048 2>&1 | head -40
