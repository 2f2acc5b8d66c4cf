set -x
export MP_NATIVE_LIB=$GRAFT_REPO_ROOT/paper_1406_2628_b200/libmergepath_b200_v64.so
MP_BLOCK_SORT= python -m pytest tests/test_gpu_parity.py -x -q -k "fused_round and warp" > gpurun_out/v64_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/v64_tests.log
for i in 1 2; do
python bench.py --config 4 --steps 50 --warmup 5 --no-e2e --no-cpu-baseline --no-extra > gpurun_out/v64_c4_$i.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/v64_c4_$i.json'));print('v64', d['ms_per_step'], d['value'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
ncu --metrics gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --csv -k regex:block_sort_warp python bench.py --config 4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-extra > gpurun_out/v64_ncu.csv 2>&1
python tools/ncu_sum.py gpurun_out/v64_ncu.csv
