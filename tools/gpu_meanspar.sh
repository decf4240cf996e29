# A/B parallel certified channel means vs the sequential chain only; GPU tests; e2e chunk check
out=gpurun_out/r02mp; mkdir -p $out
timeout 900 python -m pytest tests -m gpu -q -x > $out/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 $out/pytest.log
grep -E "FAILED|Error" $out/pytest.log | head -5
for i in 1 2; do
  for lib in default variants/libsa2pp_mp0.so; do
    if [ $lib = default ]; then unset SA2PP_LIB; else export SA2PP_LIB=$PWD/$lib; fi
    for a in "" "--seq 1024" "--workload cogvideox" "--workload llama"; do
      timeout 300 python bench.py --no-cpu $a > $out/b.json 2>/dev/null
      python -c "import json;d=json.load(open('$out/b.json'));print('$lib', '$a', round(d['value'],1), round(d['prepass']['ms_per_launch'],4), round(d['e2e']['value'],1))"
    done
  done
done
unset SA2PP_LIB
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"quantize|channel|means" -s 12 -c 6 --csv --log-file $out/launch.csv python bench.py --steps 1 --warmup 2 --no-e2e --no-cpu > /dev/null 2>&1
