# source-level capture of the fused pass: K5g (gather outer merge) vs K5e
set -x
O=gpurun_out/k5g; mkdir -p $O
for g in 1 0; do
  MP_QUAD_GATHER=$g ncu --set full --import-source on -k regex:"quad_tile" -s 3 -c 1 -f -o $O/k5_$g python tools/sort_once.py > $O/ncu_$g.log 2>&1
  ncu -i $O/k5_$g.ncu-rep --page source --csv --print-source sass > $O/k5_sass_$g.csv 2>/dev/null
  ncu -i $O/k5_$g.ncu-rep --page raw --csv > $O/k5_raw_$g.csv 2>/dev/null
  rm -f $O/k5_$g.ncu-rep
done
ls -la $O
