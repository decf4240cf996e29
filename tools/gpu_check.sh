#!/bin/bash
# One gpurun pass: parity tests, perf sweep, bench line, ncu launch list + full capture of the attention kernel.
# Usage (from the repo root, on the GPU box): bash tools/gpu_check.sh [tag]
tag=${1:-r01}
out=gpurun_out/$tag
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $out/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
timeout 300 python tools/quick_perf.py 1024 4096 16384 > $out/quick_perf.log 2>&1
timeout 600 python bench.py > $out/bench.json 2> $out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $out/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > $out/ncu_launch_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 3 -c 1 -o $out/attn_full -f \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > $out/ncu_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:quantize -s 6 -c 2 -o $out/prepass_full -f \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > $out/ncu_prepass.log 2>&1
echo done
