#!/bin/bash
# A/B of compile-time variants built with `make -C paper_2604_07980_b200/csrc VAR=x VARFLAGS=...`
# Usage: bash tools/lib_variants.sh base x y ...   (base = the default lib)
for v in "$@"; do
  if [ "$v" = base ]; then L=paper_2604_07980_b200/lib/libranger_cuda.so; else L=paper_2604_07980_b200/lib/var_$v/libranger_cuda.so; fi
  RG_LIB_PATH=$PWD/$L python -m pytest tests/test_gpu_parity.py -q -x -k "census_transform_matches or estimate" 2>&1 | tail -1
  RG_LIB_PATH=$PWD/$L python bench.py --steps 20 --warmup 3 --latency-runs 3 --no-cpu-baseline > gpurun_out/lv_$v.json 2>/dev/null
  python -c "
import json
d=json.loads(open('gpurun_out/lv_$v.json').read().strip().splitlines()[-1])
k=d['kernels']
print('$v', round(d['value']), {n: round(x, 4) for n, x in k['stage_ms_per_step'].items()}, round(k['census']['frac'],3))"
done
