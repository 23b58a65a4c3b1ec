#!/bin/bash
# CRT (multi-modular) GEMM on c5 / c2: ncu summary metrics per variant + FF_TRACE cycle counters.
mkdir -p gpurun_out
W='"winograd":-1'
FF_TRACE=1 python scripts/run_once.py c5 "{\"scheme\":3,$W}" > gpurun_out/trace_c5crt.txt 2>&1
FF_TRACE=1 python scripts/run_once.py c5 "{\"scheme\":1,$W}" >> gpurun_out/trace_c5crt.txt 2>&1
FF_TRACE=1 python scripts/run_once.py c2 '{"scheme":3}' >> gpurun_out/trace_c5crt.txt 2>&1
CFG=c5 bash scripts/ncu_variants.sh "crt_R16|FF_RASTER=16|{\"scheme\":3,$W}" "crt_R4|FF_RASTER=4|{\"scheme\":3,$W}" \
  "crt_R8|FF_RASTER=8|{\"scheme\":3,$W}" "limb|FF_RASTER=16|{\"scheme\":1,$W}" > gpurun_out/ncu_c5crt.txt 2>&1
CFG=c2 bash scripts/ncu_variants.sh "c2crt|FF_RASTER=16|{\"scheme\":3}" "c2limb|FF_RASTER=16|{\"scheme\":1}" >> gpurun_out/ncu_c5crt.txt 2>&1
