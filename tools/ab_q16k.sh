# A/B: fused-pass tile 16384 (half the K4q/K4r work) vs 8192
for v in base q16k_640_27 q16k_544_31 base q16k_640_27 q16k_544_31; do
  if [ $v = base ]; then L=""; else L="tools/variants/lib$v.so"; fi
  MP_NATIVE_LIB=$L python bench.py --config 4 --steps 50 --warmup 5 --no-e2e --no-cpu-baseline >> gpurun_out/q16_$v.json 2>> gpurun_out/q16_$v.err
done
MP_NATIVE_LIB=tools/variants/libq16k_640_27.so python -m pytest tests/test_gpu_parity.py -x -q -k "fused_round and warp or config4" > gpurun_out/q16_tests.log 2>&1; echo rc=$? >> gpurun_out/q16_tests.log
MP_NATIVE_LIB=tools/variants/libq16k_640_27.so ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"quad_" -c 3 python bench.py --config 4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | grep -E "quad_|duration" > gpurun_out/q16_ncu.log
