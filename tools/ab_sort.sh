# A/B of sort engines on the B200 (bench config 4, device-resident, 50 steps)
set -x
python -m pytest tests/test_gpu_parity.py -x -q -k "fused_round or sort" > gpurun_out/ab_tests.log 2>&1; echo rc=$? >> gpurun_out/ab_tests.log
for k in tr merge; do
  MP_K3W=$k python bench.py --config 4 --steps 50 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/ab_c4_$k.json 2> gpurun_out/ab_c4_$k.err
done
MP_K3W=tr ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum --clock-control none -k regex:block_sort -c 2 python bench.py --config 4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ab_ncu_tr.log 2>&1
