set -x
python -m pytest tests -m gpu -x -q > gpurun_out/r02m_gputests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r02m_gputests.log
python bench.py --config 4 --steps 50 --warmup 5 --no-e2e --no-cpu-baseline --no-extra > gpurun_out/r02m_c4.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/r02m_c4.json'));print('c4', d['ms_per_step'], d['value'], d['roofline']['frac'], d['clocks'])"
