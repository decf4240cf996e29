# parallel certified means only below one chain per SM: every workload and e2e, A/B vs sequential only
out=gpurun_out/r02mp2; mkdir -p $out
timeout 900 python -m pytest tests -m gpu -q -x > $out/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 $out/pytest.log
for lib in default variants/libsa2pp_mp0.so; do
  if [ $lib = default ]; then unset SA2PP_LIB; else export SA2PP_LIB=$PWD/$lib; fi
  for a in "" "--workload cogvideox" "--workload llama" "--workload longctx"; do
    timeout 300 python bench.py --no-cpu $a > $out/b.json 2>/dev/null
    python -c "import json;d=json.load(open('$out/b.json'));print('$lib', '$a', round(d['value'],1), round(d['prepass']['ms_per_launch'],4), round(d['e2e']['value'],1))"
  done
done
