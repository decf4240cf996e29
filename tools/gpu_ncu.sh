#!/bin/bash
# ncu --set full of the attention kernel at the bench shape (one launch).  Usage: bash tools/gpu_ncu.sh tag [seq] [extra bench args]
tag=${1:-ncu}; seq=${2:-16384}; shift; shift
out=gpurun_out/$tag
mkdir -p $out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 3 -c 1 -o $out/attn_full -f \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --seq $seq "$@" > $out/ncu_full.log 2>&1
tail -2 $out/ncu_full.log
