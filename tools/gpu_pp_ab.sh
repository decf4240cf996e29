out=gpurun_out/r02h; mkdir -p $out
timeout 900 python -m pytest tests -m gpu -q -x > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log; tail -3 $out/pytest_gpu.log
for lib in default variants/libsa2pp_kminb2.so; do
  if [ $lib = default ]; then unset SA2PP_LIB; else export SA2PP_LIB=$lib; fi
  for args in "" "--seq 1024" "--workload cogvideox" "--workload llama"; do
    timeout 300 python bench.py --no-e2e --no-cpu --steps 5 $args > $out/b.json 2>$out/b.err
    python -c "import json; d=json.load(open('$out/b.json')); print('$lib $args', round(d['value'],1), 'attn', round(d['roofline']['achieved'],1), 'pre_ms', round(d['prepass']['ms_per_launch'],4))" || tail -3 $out/b.err
  done
done
unset SA2PP_LIB
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 0 -c 30 --csv --log-file $out/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
grep -E "quantize|channel" $out/launches.csv | awk -F'","' '{print $5, $NF}' | cut -c1-80 | tail -8
