# device-resident bench lines for configs 2, 3a, 4, 5 (no e2e / CPU legs) + the GPU suite
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/sw_tests.log 2>&1; echo rc=$? >> gpurun_out/sw_tests.log
for c in 2 3a 5 4; do
  python bench.py --config $c --steps 100 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/sw_c$c.json 2> gpurun_out/sw_c$c.err
done
ncu --set full --clock-control none --import-source on -k regex:merge_tiles -c 1 -f -o gpurun_out/k2_c2_sent python bench.py --config 2 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/sw_ncu.log 2>&1
