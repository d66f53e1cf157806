# ncu --set full of the matcher (one launch of 32 C2 frames) for RG_MATCH_VARIANT=$V
V=${V:-0}; TAG=${TAG:-r2}
RG_MATCH_VARIANT=$V python tools/stage_time.py 32 3 > gpurun_out/st_$TAG.log 2>&1 && \
RG_MATCH_VARIANT=$V ncu --set full --clock-control none --import-source on -k regex:"match_slots_warp" -s 2 -c 1 -o gpurun_out/prof_match_$TAG python tools/stage_time.py 32 3 > gpurun_out/ncu_match_$TAG.log 2>&1
echo ncu=$?
