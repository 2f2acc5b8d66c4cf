# Round-2 evidence sweep: smoke; default bench line (config 2 + nested sort);
# every config's line; the reference arm for configs 2 and 4; the launch
# list of the default command; DRAM launch lists of config 2 and one
# config-4 sort (-> profiles/traffic_config*.json, stamped with the kernel
# sources' hash); a --set full capture of config 2's K2.
set -x
O=gpurun_out/sw; mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1200 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "default rc=$?"
for c in 1 3a 3b 5 4; do
  timeout 900 python bench.py --config $c --no-extra > $O/bench_c$c.json 2> $O/bench_c$c.err; echo "c$c rc=$?"
done
for c in 2 4; do
  timeout 600 python bench.py --impl reference --config $c > $O/bench_ref$c.json 2> $O/bench_ref$c.err
done
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_default.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_default.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/dram_config2.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-extra > $O/ncu_c2.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/dram_config4.csv python bench.py --config 4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-extra > $O/ncu_c4.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"PlainMap" -s 2 -c 1 -f -o $O/k2_c2 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-extra > $O/ncu_full.log 2>&1
ncu -i $O/k2_c2.ncu-rep --page raw --csv > $O/k2_c2_raw.csv 2>/dev/null
rm -f $O/k2_c2.ncu-rep
python tools/ncu_sum.py $O/dram_config4.csv > $O/dram_config4_sum.txt
ls -la $O
