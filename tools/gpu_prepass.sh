#!/bin/bash
# Prepass kernels at the bench shape: launch-time list (one step) + ncu --set full of each prepass
# kernel (one launch each).  Usage: bash tools/gpu_prepass.sh tag [seq]
tag=${1:-pp}; seq=${2:-16384}
out=gpurun_out/$tag
mkdir -p $out
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 12 --csv --log-file $out/launches.csv \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --seq $seq > $out/launches.log 2>&1
python - $out/launches.csv <<'PY'
import csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
for r in rows[1:]:
    print(f"{r[h.index('Kernel Name')][:60]:60s} {r[h.index('Metric Value')]:>12s} {r[h.index('Metric Unit')]}")
PY
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"channel_sums|quantize" -s 3 -c 3 \
  -o $out/prepass_full -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --seq $seq > $out/ncu_full.log 2>&1
tail -2 $out/ncu_full.log
