#!/bin/bash
# Round evidence in one gpurun call: GPU tests + smoke, bench lines for every BASELINE workload and the
# reference arm, the ncu launch list of the headline bench command, ncu --set full of the attention
# kernel with FP16 and FP32 PV accumulation (the north-star A/B) and of the prepass kernels, the
# configs[1] sweep with per-config DRAM traffic, and the pipe microbenchmark.
# Usage: bash tools/gpu_final.sh tag
tag=${1:-final}
out=gpurun_out/$tag
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $out/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
tail -2 $out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?" >> $out/smoke.log
tail -1 $out/smoke.log
timeout 300 python bench.py > $out/bench.json 2> $out/bench.err
for w in cogvideox llama longctx; do
  timeout 300 python bench.py --workload $w > $out/bench_$w.json 2> $out/bench_$w.err
done
timeout 300 python bench.py --causal > $out/bench_causal.json 2> $out/bench_causal.err
timeout 300 python bench.py --pv-accum fp32 > $out/bench_fp32acc.json 2> $out/bench_fp32acc.err
timeout 300 python bench.py --impl reference --steps 2 --warmup 3 > $out/bench_ref.json 2> $out/bench_ref.err
for f in $out/bench*.json; do python -c "import json,sys; d=json.load(open('$f')); print('$f', round(d['value'],2), d.get('roofline',{}).get('achieved'), d.get('e2e',{}).get('value'))" 2>/dev/null; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 0 -c 60 --csv --log-file $out/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > $out/ncu_launch_bench.log 2>&1
for acc in fp16 fp32; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_ws -s 3 -c 1 -o $out/attn_$acc -f \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --pv-accum $acc > $out/ncu_attn_$acc.log 2>&1
  python tools/ncu_summary.py $out/attn_$acc.ncu-rep $out/attn_${acc}_summary.md > /dev/null 2>&1
  python tools/ncu_ophist.py $out/attn_$acc.ncu-rep 4194304 60 > $out/attn_${acc}_ophist.txt 2>&1
  ncu -i $out/attn_$acc.ncu-rep --page raw --csv > $out/attn_${acc}_raw.csv 2>/dev/null
  gzip -f $out/attn_${acc}_raw.csv
  sz=$(stat -c %s $out/attn_$acc.ncu-rep); [ "$sz" -gt 30000000 ] && rm $out/attn_$acc.ncu-rep
done
timeout 900 ncu --set full --clock-control none -k regex:"channel|quantize" -s 4 -c 4 -o $out/prepass -f \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > $out/ncu_prepass.log 2>&1
python tools/ncu_summary.py $out/prepass.ncu-rep $out/prepass_summary.md > /dev/null 2>&1
bash tools/gpu_sweep.sh $tag/sweep > $out/sweep.log 2>&1
tail -24 $out/sweep.log
./tools/pipe_bench > $out/pipe_bench.txt 2>&1 || (nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/pipe_bench.cu -o /tmp/pb && /tmp/pb > $out/pipe_bench.txt 2>&1)
tail -3 $out/pipe_bench.txt
