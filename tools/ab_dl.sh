# A/B: K3w merge step with the double-load / FMA-pipe addressing (libdl) vs default
for v in base dl base dl; do
  if [ $v = base ]; then L=""; else L="tools/variants/lib$v.so"; fi
  MP_NATIVE_LIB=$L python bench.py --config 4 --steps 50 --warmup 5 --no-e2e --no-cpu-baseline >> gpurun_out/dl_$v.json 2>> gpurun_out/dl_$v.err
done
for v in base dl; do
  if [ $v = base ]; then L=""; else L="tools/variants/lib$v.so"; fi
  MP_NATIVE_LIB=$L ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active --clock-control none -k regex:block_sort -c 1 python bench.py --config 4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | grep -E "duration|inst_exec|pipe" >> gpurun_out/dl_ncu.log
done
MP_NATIVE_LIB=tools/variants/libdl.so python -m pytest tests/test_gpu_parity.py -x -q -k "fused_round and warp-0-merge" >> gpurun_out/dl_tests.log 2>&1
