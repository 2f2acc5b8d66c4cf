# A/B: K4r outer probes from the proportional guess (default build) vs midpoints (libk4rold)
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "fused_round or config4 or mid_size" > gpurun_out/k4r_tests.log 2>&1; echo rc=$? >> gpurun_out/k4r_tests.log
for v in base k4rold base k4rold; do
  if [ $v = base ]; then L=""; else L="tools/variants/lib$v.so"; fi
  MP_NATIVE_LIB=$L python bench.py --config 4 --steps 50 --warmup 5 --no-e2e --no-cpu-baseline >> gpurun_out/k4r_$v.json 2>> gpurun_out/k4r_$v.err
done
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:quad_refine -c 2 python bench.py --config 4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | grep -E "duration|dram" > gpurun_out/k4r_ncu.log
