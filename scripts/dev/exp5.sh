mkdir -p gpurun_out
CFG=c4 bash scripts/ncu_variants.sh "c4_T0|FF_THROTTLE=0|{}" "c4_T1|FF_THROTTLE=1|{}" "c4_T2|FF_THROTTLE=2|{}" "c4_T4|FF_THROTTLE=4|{}"
W='"winograd":-1'
CFG=c5 bash scripts/ncu_variants.sh "c5_T0|FF_THROTTLE=0|{$W}" "c5_T1|FF_THROTTLE=1|{$W}" "c5_T2|FF_THROTTLE=2|{$W}"
for T in 0 1 2; do FF_THROTTLE=$T python scripts/ab_test.py c4 '{}' 2>&1 | tail -1; done
