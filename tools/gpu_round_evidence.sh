#!/bin/bash
# End-of-round evidence in one gpurun call: GPU tests, bench lines for every BASELINE workload (+ the
# reference arm), the ncu launch list of the headline bench command, ncu --set full of the attention
# kernel and of the prepass kernels.  Usage: bash tools/gpu_round_evidence.sh tag
tag=${1:-ev}
out=gpurun_out/$tag
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $out/smi.txt 2>&1
timeout 300 python -m pytest tests -m gpu -q > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
timeout 300 python bench.py > $out/bench.json 2> $out/bench.err
for w in cogvideox llama longctx; do
  timeout 300 python bench.py --workload $w > $out/bench_$w.json 2> $out/bench_$w.err
done
timeout 300 python bench.py --causal > $out/bench_causal.json 2> $out/bench_causal.err
timeout 300 python bench.py --pv-accum fp32 > $out/bench_fp32acc.json 2> $out/bench_fp32acc.err
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > $out/bench_ref.json 2> $out/bench_ref.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 0 -c 60 --csv --log-file $out/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > $out/ncu_launch_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 3 -c 1 -o $out/attn_full -f \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > $out/ncu_attn.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"channel|quantize" -s 12 -c 4 -o $out/prepass_full -f \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > $out/ncu_prepass.log 2>&1
tail -2 $out/pytest_gpu.log
for f in $out/bench*.json; do echo "$f: $(head -c 300 $f)"; done
