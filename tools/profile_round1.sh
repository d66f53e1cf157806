set -x
python -m pytest tests/test_gpu_batch.py -q -x 2>&1 | tail -5
B="python bench.py --steps 2 --warmup 3 --frames 32 --distinct 8 --no-cpu-baseline --latency-runs 5"
$B > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu1.log 2>&1; echo ncu1=$?
$B > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"census_frames|match_slots" -s 2 -c 2 -o gpurun_out/prof1 $B > gpurun_out/ncu2.log 2>&1; echo ncu2=$?
ls -la gpurun_out
