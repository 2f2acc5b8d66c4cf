set -x
O=gpurun_out/k5g2; mkdir -p $O
MP_NATIVE_LIB=$GRAFT_REPO_ROOT/paper_1406_2628_b200/libmergepath_b200_g2.so ncu --set full --import-source on -k regex:"quad_tile" -s 3 -c 1 -f -o $O/k5 python tools/sort_once.py > $O/ncu.log 2>&1
ncu -i $O/k5.ncu-rep --page source --csv --print-source sass > $O/k5_sass.csv 2>/dev/null
ncu -i $O/k5.ncu-rep --page raw --csv > $O/k5_raw.csv 2>/dev/null
rm -f $O/k5.ncu-rep
