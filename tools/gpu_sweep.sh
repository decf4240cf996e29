#!/bin/bash
# BASELINE configs[1] sweep through bench.py: seq 1K-32K x causal/non-causal x head_dim 128/64, each a
# full bench line (roofline, prepass, e2e, cpu_baseline, clocks), plus the attention kernel's DRAM
# traffic per launch from ncu (one launch per config).  Usage: bash tools/gpu_sweep.sh tag
tag=${1:-sweep}
out=gpurun_out/$tag
mkdir -p $out
for D in 128 64; do
  for c in "" "--causal"; do
    for N in 1024 2048 4096 8192 16384 32768; do
      n=d${D}_n${N}$(echo "$c" | tr -d ' -')
      timeout 300 python bench.py --seq $N --head-dim $D $c > $out/bench_$n.json 2> $out/bench_$n.err
      timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:attn_ws \
        -s 3 -c 1 --csv --log-file $out/traffic_$n.csv \
        python bench.py --seq $N --head-dim $D $c --steps 1 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
      python -c "import json; d=json.load(open('$out/bench_$n.json')); print('$n', round(d['value'],1), 'attn', round(d['roofline']['achieved'],1), 'pre_ms', round(d['prepass']['ms_per_launch'],3), 'e2e', round(d['e2e']['value'],1))" 2>/dev/null || tail -2 $out/bench_$n.err
    done
  done
done
