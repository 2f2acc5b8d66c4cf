# Round-2 final evidence: traffic capture (stamps profiles/traffic_config*.json
# for the code being measured), smoke, GPU suite, default bench line (config 2
# + nested sort), every config's line, the reference arm for configs 2 and 4,
# the launch list of the default command, a --set full capture of config-2 K2.
set -x
O=gpurun_out/fin; mkdir -p $O
bash tools/capture_traffic.sh > $O/capture_traffic.log 2>&1; echo "traffic rc=$?"
cp profiles/traffic_config*.json $O/
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -2 $O/gpu_tests.log
timeout 1200 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "default rc=$?"
for c in 1 3a 3b 5 4; do
  timeout 900 python bench.py --config $c --no-extra > $O/bench_c$c.json 2> $O/bench_c$c.err; echo "c$c rc=$?"
done
for c in 2 4; do
  timeout 900 python bench.py --impl reference --config $c > $O/bench_ref$c.json 2> $O/bench_ref$c.err
done
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_default.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_default.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"PlainMap" -s 2 -c 1 -f -o $O/k2_c2 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-extra > $O/ncu_full.log 2>&1
ncu -i $O/k2_c2.ncu-rep --page raw --csv > $O/k2_c2_raw.csv 2>/dev/null
rm -f $O/k2_c2.ncu-rep
ls -la $O
