set -x
for ns in 0 1000 2500 4000 6000; do
  MP_K5E_STAGGER_NS=$ns python bench.py --config 4 --steps 30 --warmup 5 --no-e2e --no-cpu-baseline --no-extra > gpurun_out/stag_$ns.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/stag_$ns.json'));print('stagger $ns', d['ms_per_step'], d['clocks']['sm_mhz'])"
done
