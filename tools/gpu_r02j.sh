set -x
./tools/bin/k3w_lab > gpurun_out/k3w_lab.log 2>&1; echo "lab rc=$?"; cat gpurun_out/k3w_lab.log
python bench.py --config 4 --steps 30 --warmup 5 --no-e2e --no-cpu-baseline --no-extra > gpurun_out/r02j_c4.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/r02j_c4.json'));print('c4', d['ms_per_step'], d['value'], d['roofline']['frac'], d['clocks'])"
