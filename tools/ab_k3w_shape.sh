# K3w shape A/B: correctness of each shape (fused-round sorts) + config-4 sort time
set -x
for sh in 0 1 2; do
  MP_K3W_SHAPE=$sh python -m pytest tests/test_gpu_parity.py -x -q -k "fused_round and warp" > gpurun_out/k3w_tests_$sh.log 2>&1; echo "tests $sh rc=$?"; tail -1 gpurun_out/k3w_tests_$sh.log
  MP_K3W_SHAPE=$sh python bench.py --config 4 --steps 30 --warmup 5 --no-e2e --no-cpu-baseline --no-extra > gpurun_out/k3w_c4_$sh.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/k3w_c4_$sh.json'));print('k3w shape $sh', d['ms_per_step'], d['value'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
  MP_K3W_SHAPE=$sh ncu --metrics gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --csv -k regex:block_sort_warp python bench.py --config 4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-extra > gpurun_out/k3w_ncu_$sh.csv 2>&1
  python tools/ncu_sum.py gpurun_out/k3w_ncu_$sh.csv
done
