#!/bin/bash
# A/B of BM/autorect library variants (csrc/Makefile VAR=...): C4 offset-search time per frame.
for v in "$@"; do
  if [ "$v" = base ]; then L=paper_2604_07980_b200/lib/libranger_cuda.so; else L=paper_2604_07980_b200/lib/var_$v/libranger_cuda.so; fi
  RG_LIB_PATH=$PWD/$L python -m pytest tests/test_gpu_parity.py -q -x -k "bm or rect" 2>&1 | tail -1
  RG_LIB_PATH=$PWD/$L python bench.py --steps 3 --warmup 3 --frames 32 --distinct 8 --latency-runs 3 --no-cpu-baseline > gpurun_out/bv_$v.json 2>/dev/null
  python -c "
import json
d=json.loads(open('gpurun_out/bv_$v.json').read().strip().splitlines()[-1])
print('$v', round(d['autorect']['ms_per_frame'], 4))"
done
