# per-kernel ncu times of the prepass at small N, and a plain bench line per N
out=gpurun_out/r02sn; mkdir -p $out
for n in 1024 2048; do
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"quantize|channel|attn_ws" -s 10 -c 10 --csv --log-file $out/launch_$n.csv python bench.py --seq $n --steps 2 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
  timeout 300 python bench.py --seq $n --no-e2e --no-cpu > $out/b_$n.json 2>/dev/null
  python -c "import json;d=json.load(open('$out/b_$n.json'));print($n, round(d['value'],1), round(d['roofline']['achieved'],1), round(d['prepass']['ms_per_launch'],4), round(d['ms_per_step'],4))"
done
