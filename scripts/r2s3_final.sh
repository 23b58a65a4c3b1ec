#!/bin/bash
# Round-2 closing evidence of the final code (session 3): GPU suite, default bench line,
# the bench command's own launch list, a --set full capture of the c4 GEMM (roofline.traffic),
# launch lists of one default call per config.  Each ncu command runs plain first.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/f3_gputest.log 2>&1; tail -2 gpurun_out/f3_gputest.log
timeout 900 python bench.py > gpurun_out/f3_bench.json 2> gpurun_out/f3_bench.err; echo "bench rc=$?"
python bench.py --steps 3 --warmup 3 --no-per-config --no-e2e --no-cpu --no-verify > /dev/null 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f3_bench_launches.csv \
      python bench.py --steps 3 --warmup 3 --no-per-config --no-e2e --no-cpu --no-verify > gpurun_out/f3_bench_ncu.log 2>&1
echo "bench ncu rc=$?"
python scripts/run_once.py c4 '{}' > /dev/null 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:ffgemm_tc -c 1 -o gpurun_out/f3_c4_full \
      python scripts/run_once.py c4 '{}' > gpurun_out/f3_c4_full.log 2>&1
echo "c4 full rc=$?"
for c in c1 c2 c3 c4 c5; do bash scripts/launch_list.sh $c '{}' f3_$c > gpurun_out/f3_ll_$c.txt 2>&1; done
ls gpurun_out/f3_*
