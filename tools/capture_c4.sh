# config-4 evidence at the final code: per-kernel time + DRAM of one sort, and a --set full capture of K5e
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"block_sort|quad_|round_partition|merge_tiles" -c 27 --csv python bench.py --config 4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/c4_launch_dram.csv 2> gpurun_out/c4_launch_dram.err
ncu --set full --clock-control none --import-source on -k regex:quad_tile -s 1 -c 1 -f -o gpurun_out/k5e_full python bench.py --config 4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/k5e_full.log 2>&1
ncu -i gpurun_out/k5e_full.ncu-rep --page raw --csv > gpurun_out/k5e_full_raw.csv 2>/dev/null
