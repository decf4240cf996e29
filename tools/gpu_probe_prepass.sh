# per-kernel prepass time, FP64-pipe and issue utilisation for the default library and variants/*.so
out=gpurun_out/r02probe; mkdir -p $out
for lib in default $(ls variants/libsa2pp_*.so 2>/dev/null); do
  n=$(basename $lib .so)
  if [ $lib = default ]; then unset SA2PP_LIB; else export SA2PP_LIB=$lib; fi
  timeout 300 ncu --metrics gpu__time_duration.sum,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"quantize|channel" -s 4 -c 4 --csv --log-file $out/$n.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
done
