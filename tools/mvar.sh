# matcher variants: parity (GPU batch tests) + stage times per RG_MATCH_VARIANT
for v in ${VARS:-8 9 10 0}; do
  RG_MATCH_VARIANT=$v python tools/stage_time.py 256 10 2>&1 | sed "s/^/v$v /"
done
