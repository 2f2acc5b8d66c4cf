# A/B: K3w passes' split searches from diag/2 (default build) vs plain (libk3nopred)
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "sort" > gpurun_out/k3p_tests.log 2>&1; echo rc=$? >> gpurun_out/k3p_tests.log
for v in base k3nopred base k3nopred; do
  if [ $v = base ]; then L=""; else L="tools/variants/lib$v.so"; fi
  MP_NATIVE_LIB=$L python bench.py --config 4 --steps 50 --warmup 5 --no-e2e --no-cpu-baseline >> gpurun_out/k3p_$v.json 2>> gpurun_out/k3p_$v.err
done
ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active --clock-control none -k regex:block_sort -c 1 python bench.py --config 4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | grep -E "duration|inst_exec|pipe" > gpurun_out/k3p_ncu.log
