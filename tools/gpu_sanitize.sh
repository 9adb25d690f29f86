#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over the kernel tests
# (every replay variant on the reference-made fixtures, the segmented replay,
# the tensor-core scorer and its float64 re-score, K2, K7, K8, K9), small
# shapes so the instrumented run stays within minutes.
mkdir -p gpurun_out
SEL="tests/test_score_tc_gpu.py tests/test_parity_gpu.py::test_small_cases tests/test_parity_gpu.py::test_next_use_kernel_matches_numpy tests/test_parity_gpu.py::test_scorer_ranks_match_scores tests/test_segment_gpu.py::test_segmented_windows_and_costs tests/test_kat_gpu.py tests/test_diag_gpu.py tests/test_tracefile_gpu.py"
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 --target-processes all \
    python -m pytest $SEL -q -x -p no:cacheprovider > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_$tool.log
  tail -4 gpurun_out/sanitize_$tool.log
done
