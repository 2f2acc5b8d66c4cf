# A/B: K3w with 512 threads (8192-key runs) vs 1024 threads (16384-key runs)
for v in base nt1024 base nt1024; do
  if [ $v = base ]; then L=""; else L="tools/variants/lib$v.so"; fi
  MP_NATIVE_LIB=$L python bench.py --config 4 --steps 50 --warmup 5 --no-e2e --no-cpu-baseline >> gpurun_out/nt_$v.json 2>> gpurun_out/nt_$v.err
done
MP_NATIVE_LIB=tools/variants/libnt1024.so ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"block_sort|round_partition|merge_tiles" -c 36 python bench.py --config 4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/nt_ncu.log 2>&1
