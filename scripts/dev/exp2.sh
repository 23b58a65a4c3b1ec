#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x -k "crt or encoder" > gpurun_out/pytest_crt.log 2>&1; tail -2 gpurun_out/pytest_crt.log
bash scripts/launch_list.sh c5 '{"winograd":-1}' c5crt_f32enc
bash scripts/launch_list.sh c5 '{}' c5crtw_f32enc
W='"winograd":-1'
CFG=c5 bash scripts/ncu_variants.sh "crt_h3|FF_HINTS=3|{\"scheme\":3,$W}" "crt_h6|FF_HINTS=6|{\"scheme\":3,$W}" "crt_h10|FF_HINTS=10|{\"scheme\":3,$W}" "crt_h2|FF_HINTS=2|{\"scheme\":3,$W}"
CFG=c4 bash scripts/ncu_variants.sh "c4_h3|FF_HINTS=3|{}" "c4_h6|FF_HINTS=6|{}" "c4_h10|FF_HINTS=10|{}" "c4_h2|FF_HINTS=2|{}"
