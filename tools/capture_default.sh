# Launch list of the default bench command (recipe: gpu__time_duration, no clock control)
# and a --set full capture of the config-2 K2 launch (for roofline.traffic)
python bench.py --steps 2 --warmup 3 > gpurun_out/cd_bench.json 2> gpurun_out/cd_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/cd_launches_default.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/cd_ncu.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"PlainMap" -s 2 -c 1 -f -o gpurun_out/cd_k2_c2 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/cd_full.log 2>&1
ncu -i gpurun_out/cd_k2_c2.ncu-rep --page raw --csv > gpurun_out/cd_k2_c2_raw.csv 2>/dev/null
