set -x
python -m pytest tests/test_gpu_parity.py -x -q -k "sort" 2>&1 | tail -1
bash tools/launches_sort.sh
for rep in 1 2; do
  python bench.py --config 4 --steps 40 --warmup 5 --no-e2e --no-cpu-baseline --no-extra > gpurun_out/quick.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/quick.json'));print('c4', d['ms_per_step'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
