# ncu DRAM launch lists -> profiles/traffic_config{2,3a,5,4}.json (stamped
# with the kernel sources' hash; bench.py uses them only while it matches)
set -x
O=gpurun_out/tr; mkdir -p $O
for c in 2 3a 5; do
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/dram_config$c.csv python bench.py --config $c --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-extra > $O/ncu_c$c.log 2>&1
  python tools/traffic_from_ncu.py $O/dram_config$c.csv $c "merge_tiles_kernel.*PlainMap"
done
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/dram_config4.csv python bench.py --config 4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-extra > $O/ncu_c4.log 2>&1
python tools/traffic_from_ncu.py $O/dram_config4.csv 4 step 25
cp profiles/traffic_config*.json $O/
python tools/ncu_sum.py $O/dram_config4.csv
