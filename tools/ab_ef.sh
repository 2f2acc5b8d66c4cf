# A/B: bulk copies with an L2 evict_first policy (libef) vs default
for v in base ef base ef; do
  if [ $v = base ]; then L=""; else L="tools/variants/lib$v.so"; fi
  for c in 2 5 4; do
    MP_NATIVE_LIB=$L python bench.py --config $c --steps 100 --warmup 5 --no-e2e --no-cpu-baseline >> gpurun_out/ef_${v}_c$c.json 2>> gpurun_out/ef_$v.err
  done
done
