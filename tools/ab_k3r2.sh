# A/B: K3w predicted-search windows, second sweep
for v in k3r16_32 k3r8_16 k3r16_16 k3r16_24 k3r16_32 k3r8_16 k3r16_16 k3r16_24; do
  MP_NATIVE_LIB=tools/variants/lib$v.so ncu --metrics gpu__time_duration.sum --clock-control none -k regex:block_sort -c 1 python bench.py --config 4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | grep -E "duration" | sed "s/^/$v /" >> gpurun_out/k3r2.log
done
