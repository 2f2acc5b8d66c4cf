# K5p (persistent fused pass) correctness + shape A/B on config 4
set -x
python -m pytest tests/test_gpu_parity.py -x -q -k "fused_round or config4" > gpurun_out/k5p_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/k5p_tests.log
for sh in ${SHAPES:--1 0 1 2}; do
  MP_QUAD_PERSIST=$sh python bench.py --config 4 --steps 30 --warmup 5 --no-e2e --no-cpu-baseline --no-extra > gpurun_out/k5p_c4_$sh.json 2>gpurun_out/k5p_c4_$sh.err
  python -c "import json;d=json.load(open('gpurun_out/k5p_c4_$sh.json'));print('shape $sh', d['ms_per_step'], d['value'], d['clocks'])"
done
MP_QUAD_PERSIST=${NCU_SHAPE:-0} ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none --csv python bench.py --config 4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-extra > gpurun_out/k5p_launches.csv 2>&1
python tools/ncu_sum.py gpurun_out/k5p_launches.csv
