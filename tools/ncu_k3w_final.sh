# --set full raw page of the product K3w (and K5e) at the final code
set -x
O=gpurun_out/k3wf; mkdir -p $O
for k in block_sort_warp quad_tile_kernel; do
  skip=1; [ $k = block_sort_warp ] && skip=0  # one K3w launch per sort
  ncu --set full --import-source on -k regex:$k -s $skip -c 1 -f -o $O/$k python tools/sort_once.py > $O/ncu_$k.log 2>&1
  ncu -i $O/$k.ncu-rep --page raw --csv > $O/${k}_raw.csv 2>/dev/null
  rm -f $O/$k.ncu-rep
done
