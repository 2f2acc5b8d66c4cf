# A/B: K5e2 (two merge slots per thread, default build) vs K5e (libq1slot)
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "fused_round or config4" > gpurun_out/i2_tests.log 2>&1; echo rc=$? >> gpurun_out/i2_tests.log
for v in base q1slot base q1slot; do
  if [ $v = base ]; then L=""; else L="tools/variants/lib$v.so"; fi
  MP_NATIVE_LIB=$L python bench.py --config 4 --steps 50 --warmup 5 --no-e2e --no-cpu-baseline >> gpurun_out/i2_$v.json 2>> gpurun_out/i2_$v.err
done
ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:quad_tile -c 1 python bench.py --config 4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | grep -E "quad_tile|duration|inst_exec|issue|warps_active" > gpurun_out/i2_ncu.log
