#!/bin/bash
python paper_cs_0601133_b200/build.py > /dev/null || exit 1
FF_SMALL=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -x -q 2>&1 | tail -3
FF_SMALL=0 timeout 300 python scripts/small_path_ab.py
FF_SMALL=1 timeout 300 python scripts/small_path_ab.py
