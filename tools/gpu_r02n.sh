# last session: randomised parity on the final kernels, then the evidence sweep
set -x
python tools/stress_parity.py 800 7331 > gpurun_out/stress_parity_r02n.log 2>&1; echo "stress rc=$?"; tail -2 gpurun_out/stress_parity_r02n.log
bash tools/final_sweep_r02.sh
