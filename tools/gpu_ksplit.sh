# A/B reduce-scatter bias butterfly in quantize_k (prepass ms, K kernel ncu time), parity tests
out=gpurun_out/r02sp; mkdir -p $out
timeout 900 python -m pytest tests -m gpu -q -x -k "prepass or golden or gqa or llama or bias or means or padded" > $out/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 $out/pytest.log
for i in 1 2; do
  for lib in default variants/libsa2pp_sp0.so; do
    if [ $lib = default ]; then unset SA2PP_LIB; else export SA2PP_LIB=$PWD/$lib; fi
    for a in "" "--workload llama" "--workload cogvideox"; do
      timeout 300 python bench.py --no-cpu --no-e2e $a > $out/b.json 2>/dev/null
      python -c "import json;d=json.load(open('$out/b.json'));print('$lib', '$a', round(d['value'],1), round(d['prepass']['ms_per_launch'],4))"
    done
  done
done
for lib in default variants/libsa2pp_sp0.so; do
  if [ $lib = default ]; then unset SA2PP_LIB; else export SA2PP_LIB=$PWD/$lib; fi
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"quantize_k" -s 2 -c 2 --csv --log-file $out/k_$(basename $lib).csv python bench.py --steps 1 --warmup 2 --no-e2e --no-cpu > /dev/null 2>&1
  grep -o '"[0-9.,]*"$' $out/k_$(basename $lib).csv | tail -2
done
