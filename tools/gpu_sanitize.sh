#!/bin/bash
# compute-sanitizer racecheck / synccheck / memcheck / initcheck over tools/sanitize_cases.py (attention
# kernels, both head dims, causal, ragged, GQA, FP16/FP32 accumulation, instrumented variant) and the
# four prepass kernels they launch.  Usage: bash tools/gpu_sanitize.sh tag
tag=${1:-san}
out=gpurun_out/$tag
mkdir -p $out
# no caching allocator: each tensor is its own cudaMalloc, so memcheck sees accesses past its end
export PYTORCH_NO_CUDA_MEMORY_CACHING=1
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ $tool = racecheck ] && extra="--racecheck-report all"
  timeout 900 compute-sanitizer --tool $tool $extra --print-limit 50 --error-exitcode 9 \
    python tools/sanitize_cases.py > $out/$tool.log 2>&1
  echo "$tool rc=$?" >> $out/$tool.log
  tail -3 $out/$tool.log
done
