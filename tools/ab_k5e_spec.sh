# K5e split search: first bisection level(s) probed together with the window's edge probes
set -x
R=$GRAFT_REPO_ROOT/paper_1406_2628_b200
for lib in "" $R/libmergepath_b200_spec1.so $R/libmergepath_b200_spec2.so "" $R/libmergepath_b200_spec1.so $R/libmergepath_b200_spec2.so; do
  MP_NATIVE_LIB=$lib python bench.py --config 4 --steps 40 --warmup 5 --no-e2e --no-cpu-baseline --no-extra > gpurun_out/spec.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/spec.json'));print('spec lib=${lib##*/}', d['ms_per_step'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
for lib in $R/libmergepath_b200_spec1.so $R/libmergepath_b200_spec2.so; do
MP_NATIVE_LIB=$lib python -m pytest tests/test_gpu_parity.py -x -q -k "sort" 2>&1 | tail -1
done
