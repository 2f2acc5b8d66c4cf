set -x
R=$GRAFT_REPO_ROOT/paper_1406_2628_b200
python -m pytest tests/test_gpu_parity.py -x -q -k "fused_round and warp" > gpurun_out/fma_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/fma_tests.log
for lib in "" $R/libmergepath_b200_alu.so "" $R/libmergepath_b200_alu.so; do
  MP_NATIVE_LIB=$lib python bench.py --config 4 --steps 50 --warmup 5 --no-e2e --no-cpu-baseline --no-extra > gpurun_out/fma.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/fma.json'));print('fma lib=${lib##*/}', d['ms_per_step'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
ncu --metrics gpu__time_duration.sum,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none --csv -k regex:block_sort_warp python bench.py --config 4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-extra > gpurun_out/fma_ncu.csv 2>&1
python tools/ncu_sum.py gpurun_out/fma_ncu.csv
