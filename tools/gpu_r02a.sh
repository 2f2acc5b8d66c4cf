set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
nproc; lscpu | grep -E "Model name|Socket|Thread|Core"; free -g
python -m pytest tests -m gpu -x -q > gpurun_out/r02a_gputests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/r02a_gputests.log
python bench.py > gpurun_out/r02a_bench.json 2> gpurun_out/r02a_bench.err; echo "bench rc=$?"
python bench.py --config 4 > gpurun_out/r02a_bench_c4.json 2> gpurun_out/r02a_bench_c4.err; echo "bench c4 rc=$?"
cat gpurun_out/r02a_bench.json gpurun_out/r02a_bench_c4.json
