#!/bin/bash
# compute-sanitizer over a -m gpu subset that reaches every batched kernel
# (census ROI kernels, planner, throughput + latency (cooperative) matchers,
# aggregation, BM/autorect, SGM, renderer, radar refiner).  One log per tool.
SEL="tests/test_gpu_parity.py::test_census_transform_matches_oracle \
tests/test_gpu_parity.py::test_estimate_object_disparities_matches_oracle \
tests/test_gpu_batch.py::test_range_frames_device_and_host \
tests/test_gpu_batch.py::test_latency_and_throughput_matchers_agree \
tests/test_gpu_batch.py::test_large_blocks_fit_the_device_matcher \
tests/test_gpu_parity.py::test_auto_rect_search_matches_oracle \
tests/test_gpu_parity.py::test_auto_rect_search_downscale_on_device \
tests/test_gpu_sgm.py \
tests/test_gpu_render.py \
tests/test_sequence.py::test_dense_radar_refiner_matches_reference_pipeline"
for tool in ${TOOLS:-memcheck racecheck synccheck}; do
  extra=""
  [ $tool = memcheck ] && extra="--leak-check no"
  timeout ${TMO:-1500} compute-sanitizer --tool $tool $extra --print-limit 50 --error-exitcode 9 \
    python -m pytest -q -x -p no:cacheprovider $SEL > gpurun_out/sanitizer_$tool.log 2>&1
  echo "$tool rc=$?" | tee -a gpurun_out/sanitizer_summary.log
  tail -5 gpurun_out/sanitizer_$tool.log >> gpurun_out/sanitizer_summary.log
done
