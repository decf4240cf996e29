out=gpurun_out/r02final4; mkdir -p $out/sweep
timeout 300 python bench.py --workload cogvideox > $out/bench_cogvideox.json 2> $out/bench_cogvideox.err
D=64
for c in "" "--causal"; do
  for N in 1024 2048 4096 8192 16384 32768; do
    n=d${D}_n${N}$(echo "$c" | tr -d ' -')
    timeout 300 python bench.py --seq $N --head-dim $D $c > $out/sweep/bench_$n.json 2> $out/sweep/bench_$n.err
    timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:attn_ws \
      -s 3 -c 1 --csv --log-file $out/sweep/traffic_$n.csv \
      python bench.py --seq $N --head-dim $D $c --steps 1 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
    python -c "import json; d=json.load(open('$out/sweep/bench_$n.json')); print('$n', round(d['value'],1), 'attn', round(d['roofline']['achieved'],1), d['clocks'])"
  done
done
python -c "import json; d=json.load(open('$out/bench_cogvideox.json')); print('cogvideox', round(d['value'],1), round(d['roofline']['achieved'],1), d['e2e']['value'], d['clocks'])"
