#!/bin/bash
# ncu --set full of ONE attention launch of the bench command, summarised on the box (the .ncu-rep is
# kept only if small).  Usage: bash tools/gpu_prof.sh tag units [bench args...]
#   units = (query tile, key block) pairs per launch, for the per-tile opcode histogram
tag=${1:-prof}; units=${2:-4194304}; shift; shift
out=gpurun_out/$tag
mkdir -p $out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn -s 3 -c 1 -o $out/attn -f \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu "$@" > $out/ncu.log 2>&1
tail -2 $out/ncu.log
python tools/ncu_summary.py $out/attn.ncu-rep $out/summary.md > /dev/null
python tools/ncu_ophist.py $out/attn.ncu-rep $units 60 > $out/ophist.txt
python tools/ncu_hot.py $out/attn.ncu-rep $units 60 > $out/hot.txt
ncu -i $out/attn.ncu-rep --page source --csv --print-source sass > $out/source.csv 2>/dev/null
gzip -f $out/source.csv
sz=$(stat -c %s $out/attn.ncu-rep); [ $sz -gt 30000000 ] && rm $out/attn.ncu-rep
grep -E "duration|issue slots|tensor pipe|XU|ALU|FMA pipe|LSU|occupancy %|warp instructions" $out/summary.md
sed -n '/Warp stall/,$p' $out/summary.md | head -20
head -40 $out/ophist.txt
