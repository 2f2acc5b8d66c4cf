# A/B with fused round pairs: K3w 512 threads (8192-key runs, 8 pairs + 1 round) vs 1024 (16384-key runs, 8 pairs)
for v in base nt1024 base nt1024; do
  if [ $v = base ]; then L=""; else L="tools/variants/lib$v.so"; fi
  MP_NATIVE_LIB=$L python bench.py --config 4 --steps 50 --warmup 5 --no-e2e --no-cpu-baseline >> gpurun_out/nt2_$v.json 2>> gpurun_out/nt2_$v.err
done
MP_NATIVE_LIB=tools/variants/libnt1024.so python -m pytest tests/test_gpu_parity.py -x -q -k "fused_round and warp or config4" > gpurun_out/nt2_tests.log 2>&1; echo rc=$? >> gpurun_out/nt2_tests.log
