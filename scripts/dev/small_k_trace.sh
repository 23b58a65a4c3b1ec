#!/bin/bash
python paper_cs_0601133_b200/build.py > /dev/null || exit 1
FF_TRACE=1 timeout 300 python scripts/small_k.py once 2>&1 | grep "ff trace" | tail -3
