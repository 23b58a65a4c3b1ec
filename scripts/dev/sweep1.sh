mkdir -p gpurun_out
python scripts/quick_time.py > gpurun_out/quick_all.txt 2>&1
for R in 4 8 16 32; do CFG=c4 bash scripts/ncu_variants.sh "c4_R$R|FF_RASTER=$R|{}"; done > gpurun_out/sweep_c4.txt 2>&1
for R in 4 8 16; do CFG=c5 bash scripts/ncu_variants.sh "c5w0_R$R|FF_RASTER=$R|{\"winograd\":0}"; done > gpurun_out/sweep_c5.txt 2>&1
CFG=c3 bash scripts/ncu_variants.sh "c3|FF_RASTER=16|{}" >> gpurun_out/sweep_c5.txt 2>&1
