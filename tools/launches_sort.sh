# launch list (ncu duration only) of one 2^30 u32 sort
ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/sort_once.py > gpurun_out/launches_sort.csv 2>&1
python tools/ncu_sum.py gpurun_out/launches_sort.csv
