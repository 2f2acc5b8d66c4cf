set -x
python -m pytest tests/test_gpu_multi_capi.py -x -q > gpurun_out/r02f_multicapi.log 2>&1; echo "multicapi rc=$?"
tail -3 gpurun_out/r02f_multicapi.log
python -m pytest tests -m gpu -x -q --deselect tests/test_gpu_multi_capi.py > gpurun_out/r02f_gputests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/r02f_gputests.log
python bench.py > gpurun_out/r02f_bench.json 2> gpurun_out/r02f_bench.err; echo "bench rc=$?"
cat gpurun_out/r02f_bench.json
