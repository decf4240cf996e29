#!/bin/bash
# Round-2 check in one gpurun call: GPU tests, headline bench line, ncu launch list of the bench
# command and ncu --set full of the attention kernel (attn_ws_kernel) with summaries.
# Usage: bash tools/gpu_r02.sh tag [skip-tests]
tag=${1:-r02}; skip=${2:-}
out=gpurun_out/$tag
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $out/smi.txt 2>&1
if [ -z "$skip" ]; then
  timeout 900 python -m pytest tests -m gpu -q > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
  tail -3 $out/pytest_gpu.log
fi
timeout 300 python bench.py > $out/bench.json 2> $out/bench.err
head -c 600 $out/bench.json; echo
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 0 -c 60 --csv --log-file $out/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > $out/ncu_launch_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn -s 3 -c 1 -o $out/attn_full -f \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > $out/ncu_attn.log 2>&1
python tools/ncu_summary.py $out/attn_full.ncu-rep $out/attn_summary.md > /dev/null 2>&1
python tools/ncu_ophist.py $out/attn_full.ncu-rep 4194304 60 > $out/attn_ophist.txt 2>&1
python tools/ncu_hot.py $out/attn_full.ncu-rep 4194304 80 > $out/attn_hot.txt 2>&1
ncu -i $out/attn_full.ncu-rep --page source --csv --print-source sass > $out/attn_source.csv 2>/dev/null
gzip -f $out/attn_source.csv
sz=$(stat -c %s $out/attn_full.ncu-rep); [ "$sz" -gt 40000000 ] && rm $out/attn_full.ncu-rep
grep -E "duration|issue slots|tensor pipe|XU|ALU|FMA pipe|occupancy %|warp instructions" $out/attn_summary.md
