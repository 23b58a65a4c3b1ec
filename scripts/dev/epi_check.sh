#!/bin/bash
# Epilogue change check: GEMM parity tests, short-K / tiny timings, config timings.
python paper_cs_0601133_b200/build.py > /dev/null || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
timeout 300 python scripts/small_k.py
timeout 300 python scripts/tiny_gemm2.py
timeout 600 python scripts/quick_time.py c1 c2 c3 c4 c5
