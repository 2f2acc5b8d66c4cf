# source-level stall sampling of the sort's two dominant kernels (K5e, K3w)
set -x
O=gpurun_out/src; mkdir -p $O
for k in quad_tile_kernel block_sort_warp; do
  ncu --set full --import-source on -k regex:$k -s 1 -c 1 -f -o $O/$k python bench.py --config 4 --steps 1 --warmup 2 --no-e2e --no-cpu-baseline --no-extra > $O/ncu_$k.log 2>&1
  ncu -i $O/$k.ncu-rep --page source --csv --print-source sass > $O/${k}_sass.csv 2>/dev/null
  ncu -i $O/$k.ncu-rep --page raw --csv > $O/${k}_raw.csv 2>/dev/null
  rm -f $O/$k.ncu-rep
done
ls -la $O
