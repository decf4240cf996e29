# GPU tests (padded head dims 32 / 96 included) and the default + causal bench lines of this build
out=gpurun_out/r02hd; mkdir -p $out
timeout 1200 python -m pytest tests -m gpu -q -x > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
tail -4 $out/pytest_gpu.log
grep -E "FAILED|Error" $out/pytest_gpu.log | head -20
for a in "" "--causal" "--workload cogvideox"; do
  timeout 300 python bench.py --no-cpu $a > $out/b.json 2>/dev/null
  python -c "import json;d=json.load(open('$out/b.json'));print('$a', round(d['value'],1), round(d['roofline']['achieved'],1), round(d['prepass']['ms_per_launch'],3))" 2>&1 | tail -1
done
