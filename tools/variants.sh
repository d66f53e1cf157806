#!/bin/bash
# A/B of matcher launch variants (RG_MATCH_VARIANT) on the C2 bench.
python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1
for v in ${VARIANTS:-0 1 2 3 4}; do
  RG_MATCH_VARIANT=$v python bench.py --steps 10 --warmup 3 --latency-runs 5 --no-cpu-baseline --stream-frames 0 > gpurun_out/var_$v.json 2>/dev/null
  python -c "
import json,sys
d=json.loads(open('gpurun_out/var_$v.json').read().strip().splitlines()[-1])
print('variant $v', round(d['value']), d['kernels']['stage_ms_per_step'], round(d['kernels']['census']['frac'],3))"
done
