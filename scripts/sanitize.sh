#!/bin/bash
# compute-sanitizer over a GPU parity subset (under gpurun): memcheck, racecheck,
# synccheck.  Logs -> gpurun_out/sanitize_<tool>.log (summaries copied to profiles/).
mkdir -p gpurun_out
SEL="tests/test_gpu_parity.py::test_csr_matches_reference_minibatches tests/test_gpu_edge.py::test_adversarial_records_match_oracle tests/test_gpu_edge.py::test_failure_placement_across_launches tests/test_gpu_stream.py::test_file_run_memory_is_one_slice tests/test_gpu_capi.py tests/test_gpu_sharded.py::test_sharded_run_matches_goldens tests/test_gpu_edge.py::test_basic_view_names_the_first_repeat tests/test_gpu_staged.py::test_staged_edge_cases_match_reference"
for tool in memcheck racecheck synccheck; do
  extra=""
  [ "$tool" = memcheck ] && extra="--leak-check no"
  [ "$tool" = racecheck ] && extra="--racecheck-report analysis"
  timeout 1500 compute-sanitizer --tool $tool $extra --target-processes all --print-limit 50 \
    python -m pytest $SEL -q -m gpu -p no:cacheprovider -k "not (sharded_run_matches_goldens and (lookup_heavy or sign_heavy))" > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/sanitize_$tool.log
done
