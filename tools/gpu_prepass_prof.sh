#!/bin/bash
# ncu --set full (source-level) of the three prepass kernels of the headline bench command, with summary
# and hot-instruction lists.  Usage: bash tools/gpu_prepass_prof.sh tag [bench args...]
tag=${1:-pp}; shift
out=gpurun_out/$tag
mkdir -p $out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"channel|quantize" -s 3 -c 3 -o $out/prepass_full -f \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu "$@" > $out/ncu_prepass.log 2>&1
tail -2 $out/ncu_prepass.log
python tools/ncu_summary.py $out/prepass_full.ncu-rep $out/prepass_summary.md > /dev/null 2>&1
ncu -i $out/prepass_full.ncu-rep --page source --csv --print-source sass > $out/prepass_source.csv 2>/dev/null
gzip -f $out/prepass_source.csv
grep -E "^## |duration|issue slots|DRAM read|DRAM write|occupancy %|warp instructions|registers" $out/prepass_summary.md
