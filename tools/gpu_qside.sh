# A/B of quantize_q beside quantize_k at short N (prepass ms and step ms)
out=gpurun_out/r02qs; mkdir -p $out
timeout 600 python -m pytest tests -m gpu -q -x -k "graph or concurren or golden or prepass" > $out/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 $out/pytest.log
for i in 1 2; do
  for lib in default variants/libsa2pp_qs0.so variants/libsa2pp_qs4096.so; do
    if [ $lib = default ]; then unset SA2PP_LIB; else export SA2PP_LIB=$PWD/$lib; fi
    for n in 1024 2048 4096; do
      timeout 300 python bench.py --no-cpu --no-e2e --seq $n > $out/b.json 2>/dev/null
      python -c "import json;d=json.load(open('$out/b.json'));print('$lib', $n, round(d['value'],1), round(d['prepass']['ms_per_launch'],4), round(d['ms_per_step'],4))"
    done
  done
done
