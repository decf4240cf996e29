#!/bin/bash
# Quick GPU check: the GPU tests (optionally a -k filter) and one bench line.  Usage: bash tools/gpu_quick.sh tag [pytest -k expr]
tag=${1:-q}; kexpr=${2:-}
out=gpurun_out/$tag
mkdir -p $out
if [ -n "$kexpr" ]; then
  timeout 1200 python -m pytest tests -m gpu -x -q -k "$kexpr" > $out/pytest_gpu.log 2>&1
else
  timeout 1200 python -m pytest tests -m gpu -q --durations=15 > $out/pytest_gpu.log 2>&1
fi
echo "pytest rc=$?" >> $out/pytest_gpu.log
tail -25 $out/pytest_gpu.log
timeout 300 python bench.py --no-e2e --no-cpu > $out/bench.json 2> $out/bench.err
head -c 1500 $out/bench.json; tail -3 $out/bench.err
