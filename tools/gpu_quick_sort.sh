# sort parity subset + config-4 timing (A/B helper): LIBS="a.so b.so" to compare builds
set -x
python -m pytest tests/test_gpu_parity.py -x -q -k "sort" 2>&1 | tail -1
for rep in 1 2; do
for lib in "" $LIBS; do
  MP_NATIVE_LIB=$lib python bench.py --config 4 --steps 40 --warmup 5 --no-e2e --no-cpu-baseline --no-extra > gpurun_out/quick.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/quick.json'));print('c4 lib=${lib##*/}', d['ms_per_step'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
done
