# A/B: predicted-search window 2^5 / 2^6 (default) / 2^7
for v in base qpw5 qpw7 base qpw5 qpw7; do
  if [ $v = base ]; then L=""; else L="tools/variants/lib$v.so"; fi
  MP_NATIVE_LIB=$L python bench.py --config 4 --steps 50 --warmup 5 --no-e2e --no-cpu-baseline >> gpurun_out/qw_$v.json 2>> gpurun_out/qw_$v.err
done
