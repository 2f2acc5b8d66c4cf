# K5f (X/Y in their own smem region, outputs stored as produced) A/B vs K5e
set -x
for sh in 1 2 3; do
  MP_K5F=$sh python -m pytest tests/test_gpu_parity.py -x -q -k "fused_round and warp or config4_sort_full_size and not reference" > gpurun_out/k5f_tests_$sh.log 2>&1; echo "tests $sh rc=$?"; tail -1 gpurun_out/k5f_tests_$sh.log
done
for sh in 0 1 2 3 0 1 2; do
  MP_K5F=$sh python bench.py --config 4 --steps 50 --warmup 5 --no-e2e --no-cpu-baseline --no-extra > gpurun_out/k5f.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/k5f.json'));print('k5f $sh', d['ms_per_step'], d['value'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
for sh in 1 2; do
MP_K5F=$sh ncu --metrics gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:"quad_" python bench.py --config 4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-extra > gpurun_out/k5f_ncu_$sh.csv 2>&1
python tools/ncu_sum.py gpurun_out/k5f_ncu_$sh.csv
done
