#!/bin/bash
# North-star A/B: FP16 vs FP32 PV accumulation of the attention kernel at 4x32x16K x128 under ncu
# (tensor-pipe, ALU/FMA/XU pipe, issue and TMEM-load counters).  Usage: bash tools/gpu_acc_ab.sh tag [seq]
tag=${1:-acc_ab}; seq=${2:-16384}
out=gpurun_out/$tag
mkdir -p $out
for acc in fp16 fp32; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 3 -c 1 \
    -o $out/attn_$acc -f python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --seq $seq --pv-accum $acc \
    > $out/ncu_$acc.log 2>&1
  tail -1 $out/ncu_$acc.log
  timeout 300 python bench.py --seq $seq --pv-accum $acc --no-e2e --no-cpu > $out/bench_$acc.json 2> $out/bench_$acc.err
done
