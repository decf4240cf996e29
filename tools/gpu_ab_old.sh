# A/B of this build against variants/libsa2pp_old.so (previous commit), alternating, attention TOPS
out=gpurun_out/r02ab; mkdir -p $out
timeout 1200 python -m pytest tests -m gpu -q -x > $out/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $out/pytest.log
for i in 1; do
  for lib in default variants/libsa2pp_old.so; do
    if [ $lib = default ]; then unset SA2PP_LIB; else export SA2PP_LIB=$PWD/$lib; fi
    for a in "" "--causal"; do
      timeout 300 python bench.py --no-cpu --no-e2e $a > $out/b.json 2>/dev/null
      python -c "import json;d=json.load(open('$out/b.json'));print('$lib' , '$a', round(d['value'],1), round(d['roofline']['achieved'],1), round(d['prepass']['ms_per_launch'],3))"
    done
  done
done
