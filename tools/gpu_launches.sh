#!/bin/bash
# ncu launch list (device time per kernel, cold-cache serialised) of one bench step.  Usage: bash tools/gpu_launches.sh tag [bench args]
tag=${1:-launch}; shift
out=gpurun_out/$tag
mkdir -p $out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 12 -c 8 --csv --log-file $out/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu "$@" > $out/ncu_launch.log 2>&1
python - "$out/launches.csv" <<'PY'
import csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]; iN = h.index("Kernel Name"); iV = h.index("Metric Value"); iU = h.index("Metric Unit")
for r in rows[1:]:
    print(f"{r[iN][:70]:70s} {r[iV]:>12s} {r[iU]}")
PY
