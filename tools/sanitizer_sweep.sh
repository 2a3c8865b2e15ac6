#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over every libsem kernel
# family (tools/sanitize_driver.py), results into gpurun_out/sanitizer_<tool>.log.
# PYTORCH_NO_CUDA_MEMORY_CACHING=1: every tensor is its own cudaMalloc, so an
# out-of-bounds access cannot hide inside the caching allocator's pool.
mkdir -p gpurun_out
export PYTORCH_NO_CUDA_MEMORY_CACHING=1
Ns="${SAN_NS:-3 4 7 10 15}"
for tool in memcheck racecheck synccheck; do
  timeout ${SAN_TIMEOUT:-1500} compute-sanitizer --tool $tool --error-exitcode 99 --print-limit 50 \
      --target-processes all python tools/sanitize_driver.py $Ns > gpurun_out/sanitizer_$tool.log 2>&1
  echo "$tool rc=$? $(grep -c '^ok' gpurun_out/sanitizer_$tool.log) cases ok; $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/sanitizer_$tool.log | tail -1)"
done
