# A/B: K5e split searches from a proportional guess (default build) vs plain (libqnopred)
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "fused_round or config4 or mid_size or extreme" > gpurun_out/qp_tests.log 2>&1; echo rc=$? >> gpurun_out/qp_tests.log
for v in base qnopred base qnopred; do
  if [ $v = base ]; then L=""; else L="tools/variants/lib$v.so"; fi
  MP_NATIVE_LIB=$L python bench.py --config 4 --steps 50 --warmup 5 --no-e2e --no-cpu-baseline >> gpurun_out/qp_$v.json 2>> gpurun_out/qp_$v.err
done
ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:quad_tile -c 1 python bench.py --config 4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | grep -E "duration|inst_exec|issue" > gpurun_out/qp_ncu.log
