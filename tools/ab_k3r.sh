# A/B: K3w predicted-search windows (default 32/64)
for v in base k3r16_32 k3r64_128 base k3r16_32 k3r64_128; do
  if [ $v = base ]; then L=""; else L="tools/variants/lib$v.so"; fi
  MP_NATIVE_LIB=$L ncu --metrics gpu__time_duration.sum --clock-control none -k regex:block_sort -c 1 python bench.py --config 4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | grep -E "duration" | sed "s/^/$v /" >> gpurun_out/k3r.log
done
