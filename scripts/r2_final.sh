#!/bin/bash
# round-2 closing evidence: GPU suite, full bench (c4 + per-config + e2e + cpu), ncu of c5 P1/P6 and c1
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/r2f_gputest.log 2>&1; tail -2 gpurun_out/r2f_gputest.log
python bench.py > gpurun_out/r2f_bench.json 2> gpurun_out/r2f_bench.err; echo "bench rc=$?"
python scripts/run_once.py c5 '{}' > /dev/null 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:ffgemm_tc -c 3 -o gpurun_out/r2f_c5_full \
      python scripts/run_once.py c5 '{}' > gpurun_out/r2f_c5_full.log 2>&1
python scripts/run_once.py c1 '{}' > /dev/null 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:lat_gemm -c 1 -o gpurun_out/r2f_c1_full \
      python scripts/run_once.py c1 '{}' > gpurun_out/r2f_c1_full.log 2>&1
for c in c5 c1; do bash scripts/launch_list.sh $c '{}' r2f_$c > gpurun_out/r2f_ll_$c.txt 2>&1; done
ls gpurun_out/r2f_*
# the bench command's own launch list (contract: kernel share of the step)
python bench.py --steps 3 --warmup 3 --no-per-config --no-e2e --no-cpu --no-verify > /dev/null 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2f_bench_launches.csv \
      python bench.py --steps 3 --warmup 3 --no-per-config --no-e2e --no-cpu --no-verify > gpurun_out/r2f_bench_ncu.log 2>&1
echo "bench ncu rc=$?"
