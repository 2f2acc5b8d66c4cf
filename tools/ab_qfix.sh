# A/B: fixed-step (binary lifting) searches in K5e vs the while-loop searches (libqloop)
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "fused_round or config4" > gpurun_out/qf_tests.log 2>&1; echo rc=$? >> gpurun_out/qf_tests.log
for v in base qloop base qloop; do
  if [ $v = base ]; then L=""; else L="tools/variants/lib$v.so"; fi
  MP_NATIVE_LIB=$L python bench.py --config 4 --steps 50 --warmup 5 --no-e2e --no-cpu-baseline >> gpurun_out/qf_$v.json 2>> gpurun_out/qf_$v.err
done
ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:quad_tile -c 1 python bench.py --config 4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | grep -E "duration|inst_exec|issue" > gpurun_out/qf_ncu.log
