#!/bin/bash
# Round-2 profiling recipe (B200_PROFILING.md): plain bench line, launch list of
# a short bench run, one --set full capture of the K1/K2 kernels of a
# 256-frame rg_range_frames launch.  Each ncu run only after its command ran clean.
set -x
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r2.log 2>&1; echo bench=$?
B="python bench.py --steps 2 --warmup 3 --frames 32 --stream-frames 0 --c3-frames 0 --c1-frames 0 --no-cpu-baseline --latency-runs 5 --no-parity"
$B > gpurun_out/plain_r2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r2.csv $B > gpurun_out/ncu_l_r2.log 2>&1; echo launches=$?
python tools/stage_time.py 256 2 > gpurun_out/st_r2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"census_rowtile|census_rows_kernel|census_cols_kernel|match_slots_warp|sample_slots|plan_frames|occluders|aggregate_warp" -c 8 -o gpurun_out/prof_r2 python tools/stage_time.py 256 1 > gpurun_out/ncu_f_r2.log 2>&1; echo full=$?
