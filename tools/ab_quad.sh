# A/B on one box: fused two-round passes (MP_SORT_QUAD=1) vs plain rounds
for q in 1 0 1 0; do
  MP_SORT_QUAD=$q python bench.py --config 4 --steps 50 --warmup 5 --no-e2e --no-cpu-baseline >> gpurun_out/abq_$q.json 2>> gpurun_out/abq_$q.err
done
