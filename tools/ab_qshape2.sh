# K5e thread shapes after the granule-copy change (variant builds via MP_NATIVE_LIB)
set -x
R=$GRAFT_REPO_ROOT/paper_1406_2628_b200
for lib in "" $R/libmergepath_b200_q576.so $R/libmergepath_b200_q704.so $R/libmergepath_b200_q672.so "" $R/libmergepath_b200_q576.so $R/libmergepath_b200_q704.so $R/libmergepath_b200_q672.so; do
  MP_NATIVE_LIB=$lib python bench.py --config 4 --steps 50 --warmup 5 --no-e2e --no-cpu-baseline --no-extra > gpurun_out/qs.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/qs.json'));print('qshape ${lib##*/}', d['ms_per_step'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
