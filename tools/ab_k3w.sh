# K3w check: sort parity tests, config-4 bench, block-sort kernel time + instructions
python -m pytest tests/test_gpu_parity.py -x -q -k "sort" > gpurun_out/k3w_tests.log 2>&1; echo rc=$? >> gpurun_out/k3w_tests.log
python bench.py --config 4 --steps 50 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/k3w_c4.json 2> gpurun_out/k3w_c4.err
ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum --clock-control none -k regex:block_sort -c 1 python bench.py --config 4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/k3w_ncu.log 2>&1
