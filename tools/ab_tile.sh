# A/B of the sort's round tile (8192 vs 4096 outputs) on the B200
python -m pytest tests/test_gpu_parity.py -x -q -k "sort" > gpurun_out/abt_tests.log 2>&1; echo rc=$? >> gpurun_out/abt_tests.log
for t in 8192 4096 8192 4096; do
  MP_SORT_TILE=$t python bench.py --config 4 --steps 50 --warmup 5 --no-e2e --no-cpu-baseline >> gpurun_out/abt_c4_$t.json 2>> gpurun_out/abt_c4_$t.err
done
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv python bench.py --config 4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/abt_launches.csv 2>&1
