#!/bin/bash
# Round-end measurement: GPU tests, bench (N=1), ncu launch list of the bench and
# one --set full capture of the c4 GEMM; summaries go to profiles/ via
# scripts/summarize_profiles.py (run here afterwards).
mkdir -p gpurun_out
(time python -m pytest tests -m gpu -q) > gpurun_out/final_pytest_gpu.log 2>&1
tail -3 gpurun_out/final_pytest_gpu.log
python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err
cat gpurun_out/final_bench.json
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/final_bench_ref.json 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/final_c4_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/final_ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ffgemm_tc -c 1 \
  -o gpurun_out/final_c4_gemm python scripts/run_once.py c4 '{}' > gpurun_out/final_ncu_full.log 2>&1
bash scripts/launch_list.sh c5 '{}' final_c5 > gpurun_out/final_c5_list.txt 2>&1
python scripts/quick_time.py > gpurun_out/final_quick_all.txt 2>&1
cat gpurun_out/final_quick_all.txt
