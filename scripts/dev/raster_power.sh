#!/bin/bash
# c4 bench under raster / L2-hint variants: ms/step, SM clock, power (the GEMM is power-capped)
python paper_cs_0601133_b200/build.py > /dev/null || exit 1
for v in "FF_RASTER=16" "FF_RASTER=8" "FF_RASTER=4" "FF_HINTS=11" "FF_RASTER=8 FF_HINTS=11" "FF_RASTER=16"; do
  env $v python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); c=d['clocks']
print('%-26s %7.2f ms/step  frac %.3f  clock-frac %.3f  sm %s MHz  %s W' % ('$v', d['ms_per_step'], d['roofline']['frac'], d['roofline']['frac_of_clock_peak'], c['sm_mhz'], c.get('power_w_max')))"
done
