set -x
python -m pytest tests/test_gpu_parity.py -x -q -k "fused_round or config4 or sort" > gpurun_out/wide_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/wide_tests.log
for i in 1 2; do
python bench.py --config 4 --steps 50 --warmup 5 --no-e2e --no-cpu-baseline --no-extra > gpurun_out/wide_c4_$i.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/wide_c4_$i.json'));print('wide', d['ms_per_step'], d['value'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
ncu --metrics gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:quad_tile python bench.py --config 4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-extra > gpurun_out/wide_ncu.csv 2>&1
python tools/ncu_sum.py gpurun_out/wide_ncu.csv
