# Round-end evidence: smoke, default bench lines for configs 1-5 (device value,
# e2e, CPU baseline, clocks, launches), the reference arm for configs 2 and 4,
# and the launch lists of the default bench command and of one config-4 sort.
set -x
O=gpurun_out/fs; mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
for c in 2 4 3a 3b 5 1; do
  timeout 900 python bench.py --config $c > $O/bench_c$c.json 2> $O/bench_c$c.err
done
for c in 2 4; do
  timeout 600 python bench.py --impl reference --config $c > $O/bench_ref$c.json 2> $O/bench_ref$c.err
done
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv --log-file $O/launches_bench_default.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_default.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"block_sort|round_partition|merge_tiles" -c 36 --csv --log-file $O/launches_config4.csv python bench.py --config 4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_c4.log 2>&1
