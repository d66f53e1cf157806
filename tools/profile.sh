#!/bin/bash
# Profiling recipe (B200_PROFILING.md): plain run, launch list, one --set full
# capture of the two dominant kernels.  Usage: bash tools/profile.sh TAG
TAG=${1:-r1}
set -x
B="python bench.py --steps 2 --warmup 3 --frames 32 --distinct 8 --no-cpu-baseline --latency-runs 5"
$B > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $B > gpurun_out/ncu_l_$TAG.log 2>&1; echo ncu_launches=$?
$B > gpurun_out/plain2_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"census_pairs|match_slots_warp|bm_simd" -s 3 -c 3 -o gpurun_out/prof_$TAG $B > gpurun_out/ncu_f_$TAG.log 2>&1; echo ncu_full=$?
$B > gpurun_out/plain3_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"bm_simd" -s 2 -c 1 -o gpurun_out/prof_bm_$TAG $B > gpurun_out/ncu_bm_$TAG.log 2>&1; echo ncu_bm=$?
