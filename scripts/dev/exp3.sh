#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x -k "encoder or crt or c3 or winograd_level" > gpurun_out/pytest_enc.log 2>&1; tail -2 gpurun_out/pytest_enc.log
bash scripts/launch_list.sh c3 '{}' c3_pipe
bash scripts/launch_list.sh c4 '{}' c4_pipe
bash scripts/launch_list.sh c5 '{}' c5_pipe
