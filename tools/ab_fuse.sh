# small-merge fusion A/B (config 1) + the whole GPU suite
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/fu_tests.log 2>&1; echo rc=$? >> gpurun_out/fu_tests.log
for f in 592 0 592 0; do
  MP_MERGE_FUSE_TILES=$f python bench.py --config 1 --steps 200 --warmup 10 --no-cpu-baseline >> gpurun_out/fu_c1_$f.json 2>> gpurun_out/fu_c1_$f.err
done
python bench.py --config 2 --steps 100 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/fu_c2.json 2> gpurun_out/fu_c2.err
