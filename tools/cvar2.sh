# census rowtile CTA-size variants (RG_LIB_PATH libraries built with VAR=...)
for v in base ${VARS}; do
  if [ $v = base ]; then L=""; else L=$PWD/paper_2604_07980_b200/lib/var_$v/libranger_cuda.so; fi
  RG_LIB_PATH=$L RG_CENSUS_MODE=1 python tools/stage_time.py 256 10 2>&1 | sed "s/^/$v /"
done
RG_CENSUS_FULL=1 python tools/stage_time.py 256 10 2>&1 | sed "s/^/full /"
