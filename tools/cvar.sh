# census A/B: ROI census modes (RG_CENSUS_MODE 0: pair tiles + store masks, 1: warp row tiles) vs full-frame K1
for m in 0 1; do RG_CENSUS_MODE=$m python tools/stage_time.py 256 10 2>&1 | sed "s/^/mode$m /"; done
RG_CENSUS_FULL=1 python tools/stage_time.py 256 10 2>&1 | sed "s/^/full /"
for m in 0 1; do RG_CENSUS_MODE=$m python tools/stage_time.py 4 50 2>&1 | sed "s/^/mode$m /"; done
RG_CENSUS_FULL=1 python tools/stage_time.py 4 50 2>&1 | sed "s/^/full /"
