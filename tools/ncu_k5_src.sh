# source-level stall sampling of the fused pass (K5e vs K5p)
set -x
for sh in -1 0; do
  MP_QUAD_PERSIST=$sh ncu --set full --import-source on -k regex:"quad_tile_kernel|quad_persist_kernel" -s 3 -c 1 -f -o gpurun_out/k5_src_$sh python bench.py --config 4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-extra > gpurun_out/ncu_k5_$sh.log 2>&1
  ncu -i gpurun_out/k5_src_$sh.ncu-rep --page source --csv --print-source sass > gpurun_out/k5_sass_$sh.csv 2>/dev/null
  ncu -i gpurun_out/k5_src_$sh.ncu-rep --page raw --csv > gpurun_out/k5_raw_$sh.csv 2>/dev/null
  ncu -i gpurun_out/k5_src_$sh.ncu-rep --page details --csv > gpurun_out/k5_details_$sh.csv 2>/dev/null
done
ls -la gpurun_out | tail
