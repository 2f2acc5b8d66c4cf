# A/B: K5e thread shapes at the 16384-output tile
for v in base q16k_576_29 q16k_704_25 base q16k_576_29 q16k_704_25; do
  if [ $v = base ]; then L=""; else L="tools/variants/lib$v.so"; fi
  MP_NATIVE_LIB=$L python bench.py --config 4 --steps 50 --warmup 5 --no-e2e --no-cpu-baseline >> gpurun_out/q162_$v.json 2>> gpurun_out/q162_$v.err
done
