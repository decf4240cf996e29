#!/bin/bash
# Fast GPU iteration: parity tests + perf sweep (no ncu).  Usage: bash tools/gpu_quick.sh tag [N...]
tag=${1:-quick}; shift
out=gpurun_out/$tag
mkdir -p $out
timeout 180 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
timeout 120 python tools/quick_perf.py ${@:-1024 4096 16384} > $out/quick_perf.log 2>&1
tail -3 $out/pytest_gpu.log; cat $out/quick_perf.log
