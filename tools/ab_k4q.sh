# A/B: K4q bounds from the proportional guess (default build) vs full-run bisection (libk4qold)
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "fused_round or config4 or mid_size or beyond" > gpurun_out/k4q_tests.log 2>&1; echo rc=$? >> gpurun_out/k4q_tests.log
for v in base k4qold base k4qold; do
  if [ $v = base ]; then L=""; else L="tools/variants/lib$v.so"; fi
  MP_NATIVE_LIB=$L python bench.py --config 4 --steps 50 --warmup 5 --no-e2e --no-cpu-baseline >> gpurun_out/k4q_$v.json 2>> gpurun_out/k4q_$v.err
done
