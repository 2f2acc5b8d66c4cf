set -x
python -m pytest tests/test_gpu_parity.py -x -q -k "fused_round or config4" > gpurun_out/ch_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/ch_tests.log
for lib in "" $GRAFT_REPO_ROOT/paper_1406_2628_b200/libmergepath_b200_c1.so "" $GRAFT_REPO_ROOT/paper_1406_2628_b200/libmergepath_b200_c1.so; do
  MP_NATIVE_LIB=$lib python bench.py --config 4 --steps 50 --warmup 5 --no-e2e --no-cpu-baseline --no-extra > gpurun_out/ch.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/ch.json'));print('chains lib=${lib##*/}', d['ms_per_step'], d['value'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
ncu --metrics gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none --csv -k regex:quad_tile python bench.py --config 4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-extra > gpurun_out/ch_ncu.csv 2>&1
python tools/ncu_sum.py gpurun_out/ch_ncu.csv
