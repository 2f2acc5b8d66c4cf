# A/B: programmatic dependent launch on K1->K2 and the sort's K4->K2->K4 chain
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pdl_tests.log 2>&1; echo rc=$? >> gpurun_out/pdl_tests.log
for p in 1 0 1 0; do
  for c in 2 4; do
    MP_PDL=$p python bench.py --config $c --steps 100 --warmup 5 --no-e2e --no-cpu-baseline >> gpurun_out/pdl_${p}_c$c.json 2>> gpurun_out/pdl_$p.err
  done
done
