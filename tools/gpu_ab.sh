#!/bin/bash
# A/B of the attention kernels (SA2PP_ATTN=v4 vs the default) on the headline bench and the GPU tests.
# Usage: bash tools/gpu_ab.sh tag [pytest -k expr]
tag=${1:-ab}; kexpr=${2:-}
out=gpurun_out/$tag
mkdir -p $out
if [ -n "$kexpr" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q -k "$kexpr" > $out/pytest_gpu.log 2>&1
else
  timeout 900 python -m pytest tests -m gpu -q -x > $out/pytest_gpu.log 2>&1
fi
echo "pytest rc=$?" >> $out/pytest_gpu.log
tail -15 $out/pytest_gpu.log
for impl in default v4; do
  for args in "" "--causal" "--workload cogvideox"; do
    n=$(echo "$impl$args" | tr -d ' -')
    if [ $impl = v4 ]; then export SA2PP_ATTN=v4; else unset SA2PP_ATTN; fi
    timeout 300 python bench.py --no-e2e --no-cpu $args > $out/bench_$n.json 2> $out/bench_$n.err
    python -c "import json,sys; d=json.load(open('$out/bench_$n.json')); print('$n', round(d['value'],1), 'attn', round(d['roofline']['achieved'],1), 'pre ms', round(d['prepass']['ms_per_launch'],3))" 2>/dev/null || tail -3 $out/bench_$n.err
  done
done
