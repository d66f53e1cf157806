# matcher A/B: library variants x RG_MATCH_VARIANT
for v in ${VARS:-base}; do
  if [ $v = base ]; then L=""; else L=$PWD/paper_2604_07980_b200/lib/var_$v/libranger_cuda.so; fi
  for mv in ${MVS:-0}; do
    RG_LIB_PATH=$L RG_MATCH_VARIANT=$mv python tools/stage_time.py 256 10 2>&1 | sed "s/^/$v mv$mv /"
  done
done
