#!/bin/bash
# Bench the default library and every variants/libsa2pp_*.so on the headline + causal + CogVideoX
# workloads (GPU tests on the default first).  Usage: bash tools/gpu_variants.sh tag [pytest -k expr|none]
tag=${1:-var}; kexpr=${2:-}
out=gpurun_out/$tag
mkdir -p $out
if [ "$kexpr" != "none" ]; then
  if [ -n "$kexpr" ]; then
    timeout 900 python -m pytest tests -m gpu -x -q -k "$kexpr" > $out/pytest_gpu.log 2>&1
  else
    timeout 900 python -m pytest tests -m gpu -q -x > $out/pytest_gpu.log 2>&1
  fi
  echo "pytest rc=$?" >> $out/pytest_gpu.log
  tail -4 $out/pytest_gpu.log
fi
for lib in default $(ls variants/libsa2pp_*.so 2>/dev/null); do
  n=$(basename $lib .so)
  if [ $lib = default ]; then unset SA2PP_LIB; else export SA2PP_LIB=$lib; fi
  timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "output_vs_reference or qk_scores or ragged_lengths" > $out/pytest_$n.log 2>&1
  echo "$n parity: $(tail -1 $out/pytest_$n.log)"
  for args in "" "--causal" "--workload cogvideox"; do
    m=$n$(echo "$args" | tr -d ' -')
    timeout 300 python bench.py --no-e2e --no-cpu --steps 5 $args > $out/bench_$m.json 2> $out/bench_$m.err
    python -c "import json; d=json.load(open('$out/bench_$m.json')); print('$m', round(d['value'],1), 'attn', round(d['roofline']['achieved'],1))" 2>/dev/null || tail -3 $out/bench_$m.err
  done
done
