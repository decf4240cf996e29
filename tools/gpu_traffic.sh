#!/bin/bash
# DRAM bytes per attention launch for every bench workload (one ncu-replayed launch each).
# Usage: bash tools/gpu_traffic.sh tag
tag=${1:-tr}
out=gpurun_out/$tag
mkdir -p $out
for args in "" "--causal" "--workload cogvideox" "--workload llama" "--workload longctx"; do
  name=$(echo "w$args" | tr -d ' -')
  timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:attn_fwd -s 3 -c 1 --csv --log-file $out/$name.csv \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu $args > $out/$name.log 2>&1
  tail -1 $out/$name.log | head -c 200; echo
done
