set -x
export MP_SORT_QUAD=1
python bench.py --config 4 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/quad_bench.json 2> gpurun_out/quad_bench.err
ncu --section SourceCounters --section LaunchStats --section Occupancy --section SchedulerStats --section WarpStateStats --import-source on -k regex:quad_tile_kernel -c 1 -f -o gpurun_out/k5e_src python bench.py --config 4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_k5e.log 2>&1
ncu --section SourceCounters --section LaunchStats --section Occupancy --section SchedulerStats --section WarpStateStats --import-source on -k regex:quad_refine_kernel -c 1 -f -o gpurun_out/k4r_src python bench.py --config 4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_k4r.log 2>&1
unset MP_SORT_QUAD
ncu --section SourceCounters --section LaunchStats --section Occupancy --section SchedulerStats --section WarpStateStats --import-source on -k regex:merge_tiles_kernel -s 2 -c 1 -f -o gpurun_out/k2r_src python bench.py --config 4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_k2r.log 2>&1
ncu --section SourceCounters --section LaunchStats --section Occupancy --section SchedulerStats --section WarpStateStats --import-source on -k regex:block_sort_warp -c 1 -f -o gpurun_out/k3w_src python bench.py --config 4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_k3w.log 2>&1
ls -la gpurun_out
