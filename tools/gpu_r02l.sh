set -x
python -m pytest tests/test_gpu_parity.py -x -q -k "sort" > gpurun_out/r02l_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r02l_tests.log
for g in 0 1 0 1; do
MP_QUAD_GATHER=$g python bench.py --config 4 --steps 30 --warmup 5 --no-e2e --no-cpu-baseline --no-extra > gpurun_out/r02l_c4_$g.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/r02l_c4_$g.json'));print('c4 gather=$g', d['ms_per_step'], d['value'], d['clocks'])"
done
