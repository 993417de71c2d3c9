#!/bin/bash
# compute-sanitizer over every kernel family (tools/sanitize_cases.py) -> gpurun_out/sanitize_<tool>.log
# memcheck runs with the torch caching allocator off, so each buffer is its own allocation (out-of-bounds accesses
# between neighbouring tensors are caught)
mkdir -p gpurun_out
for tool in ${TOOLS:-memcheck racecheck synccheck initcheck}; do
  extra=""
  # (no --leak-check: the library allocates no device memory of its own on these paths; torch frees its pool
  # at process exit, which the leak checker would report)
  [ "$tool" = "racecheck" ] && extra="--racecheck-report hazard"
  for c in ${CASES:-mesh silhouette softmax points camera_batching}; do
    echo "== $tool $c" >> gpurun_out/sanitize_$tool.log
    PYTORCH_NO_CUDA_MEMORY_CACHING=$([ "$tool" = "memcheck" ] && echo 1 || echo 0) \
      timeout ${TMO:-900} compute-sanitizer --tool $tool $extra --print-limit 20 --target-processes all \
      python tools/sanitize_cases.py $c >> gpurun_out/sanitize_$tool.log 2>&1
    echo "rc=$?" >> gpurun_out/sanitize_$tool.log
  done
  grep -E "^== |SUMMARY|rc=|case .* done" gpurun_out/sanitize_$tool.log
done
